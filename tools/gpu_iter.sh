#!/bin/bash
# Iteration run: GPU parity tests, then quick benches of the library variants given in $VARIANTS.
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
: > $O/quick.txt
for v in ${VARIANTS:-libhd.so}; do
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v CONFIGS="${CONFIGS:-5d 6d}" STEPS=${STEPS:-3} bash tools/quick_bench.sh $v >> $O/quick.txt 2>&1
done
cat $O/quick.txt
