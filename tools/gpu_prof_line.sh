#!/bin/bash
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
export HD_LINE=1
tag=line_5d
timeout 300 python tools/prof_driver.py --config 5d --op rk --reps 2 > $O/plain_$tag.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:line_kernel -s 6 -c 1 \
   -o $O/ncu_$tag python tools/prof_driver.py --config 5d --op rk --reps 2 > $O/ncu_$tag.log 2>&1
python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
