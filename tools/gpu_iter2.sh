#!/bin/bash
# tests + quick bench of variants + ncu of the 6D RK stage kernel (summarised on the box; reports > 25 MB dropped)
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
fi
: > $O/quick.txt
for v in ${VARIANTS:-libhd.so}; do
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v CONFIGS="${CONFIGS:-5d 6d}" STEPS=${STEPS:-3} bash tools/quick_bench.sh $v >> $O/quick.txt 2>&1
done
cat $O/quick.txt
for v in ${NCU_VARIANTS}; do
  for c in ${NCU_CONFIGS:-6d}; do
    export HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v
    tag=${v%.so}_$c
    timeout 300 python tools/prof_driver.py --config $c --op ${NCU_OP:-rk} --reps 2 > $O/plain_$tag.log 2>&1 && \
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s ${NCU_SKIP:-6} -c 1 \
       -o $O/ncu_$tag python tools/prof_driver.py --config $c --op ${NCU_OP:-rk} --reps 2 > $O/ncu_$tag.log 2>&1
    python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
    sz=$(stat -c %s $O/ncu_$tag.ncu-rep 2>/dev/null || echo 0)
    if [ "$sz" -gt 25000000 ]; then rm -f $O/ncu_$tag.ncu-rep; fi
  done
done
du -sh $O
