#!/bin/bash
# A/B quick benches: $VARIANTS = list of libraries in paper_2002_08110_b200/ (default build first)
O=gpurun_out
: > $O/quick.txt
for v in ${VARIANTS:-libhd.so}; do
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v CONFIGS="${CONFIGS:-5d 6d}" STEPS=3 bash tools/quick_bench.sh $v >> $O/quick.txt 2>&1
done
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2; fi
