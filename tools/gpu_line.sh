#!/bin/bash
O=gpurun_out
: > $O/quick.txt
CONFIGS="4d 5d 6d" STEPS=3 bash tools/quick_bench.sh tile >> $O/quick.txt 2>&1
CONFIGS="4d 5d 6d" STEPS=3 bash tools/quick_bench.sh line HD_LINE=1 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
HD_LINE=1 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
