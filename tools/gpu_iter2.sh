#!/bin/bash
# tests + quick bench of variants + ncu of the 6D RK stage kernel for each variant
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
: > $O/quick.txt
for v in ${VARIANTS:-libhd.so}; do
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v CONFIGS="${CONFIGS:-5d 6d}" STEPS=${STEPS:-3} bash tools/quick_bench.sh $v >> $O/quick.txt 2>&1
done
cat $O/quick.txt
for v in ${NCU_VARIANTS}; do
  for c in ${NCU_CONFIGS:-6d}; do
    export HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v
    timeout 300 python tools/prof_driver.py --config $c --op rk --reps 2 > $O/plain_$v_$c.log 2>&1 && \
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s 6 -c 1 \
       -o $O/ncu_${v%.so}_$c python tools/prof_driver.py --config $c --op rk --reps 2 > $O/ncu_${v%.so}_$c.log 2>&1
  done
done
