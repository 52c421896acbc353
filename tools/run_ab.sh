#!/bin/bash
# A/B of experiment libraries: LIBS="a.so b.so" CONFIGS="6d 5d" bash tools/run_ab.sh
for L in ${LIBS}; do
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$L CONFIGS="${CONFIGS:-6d 5d}" bash tools/quick_bench.sh $L | tee -a gpurun_out/ab.txt
done
