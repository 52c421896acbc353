#!/bin/bash
O=gpurun_out
: > $O/quick.txt
for m in 0 1 2; do CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh pub$m HD_PUBMODE=$m >> $O/quick.txt 2>&1; done
CONFIGS="6d" STEPS=3 bash tools/quick_bench.sh nodiscard HD_DISCARD=0 >> $O/quick.txt 2>&1
CONFIGS="6d" STEPS=3 bash tools/quick_bench.sh skew3 HD_SKEW=3 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
