#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
: > $O/quick.txt
CONFIGS="4d 5d 6d" STEPS=3 bash tools/quick_bench.sh v8 >> $O/quick.txt 2>&1
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh v8-skew3 HD_SKEW=3 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
