#!/bin/bash
O=gpurun_out
: > $O/quick.txt
for dbg in 0 1 2 3; do CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh dbg$dbg HD_DBG=$dbg >> $O/quick.txt 2>&1; done
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh notrace HD_TRACE=0 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
