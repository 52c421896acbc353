#!/bin/bash
# One full ncu capture of the fused stage kernel (steady-state RK launch) per config in $CONFIGS, with the
# bench-only library when present; summaries under gpurun_out/.
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
[ -f paper_2002_08110_b200/libhd_bench.so ] && export HD_LIB_PATH=$PWD/paper_2002_08110_b200/libhd_bench.so
for c in ${CONFIGS:-6d}; do
  op=${OP:-rk}
  tag=${TAG:-cur}_${op}_$c
  timeout 300 python tools/prof_driver.py --config $c --op $op --reps 2 > $O/plain_$tag.log 2>&1 || { echo "plain $c failed"; tail -5 $O/plain_$tag.log; continue; }
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s ${SKIP:-6} -c 1 \
     -o $O/ncu_$tag python tools/prof_driver.py --config $c --op $op --reps 2 > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
  python tools/ncu_lines.py $O/ncu_$tag.ncu-rep 45 > $O/ncu_${tag}_lines.txt 2>&1
  head -40 $O/ncu_$tag.txt
done
