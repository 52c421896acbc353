#!/bin/bash
O=gpurun_out
: > $O/quick.txt
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh line2 HD_LINE=1 >> $O/quick.txt 2>&1
HD_LIB_PATH=$PWD/paper_2002_08110_b200/libhd_l3.so CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh line3 HD_LINE=1 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
