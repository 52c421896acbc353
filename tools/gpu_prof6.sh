#!/bin/bash
# full ncu capture of one 6D RK-stage launch of the tile kernel, SASS + CUDA-line summaries
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
tag=${TAG:-6d}
cfg=${CFG:-6d}
timeout 300 python tools/prof_driver.py --config $cfg --op rk --reps 2 > $O/plain_$tag.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s 6 -c 1 \
   -o $O/ncu_$tag python tools/prof_driver.py --config $cfg --op rk --reps 2 > $O/ncu_$tag.log 2>&1
python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
ncu -i $O/ncu_$tag.ncu-rep --page source --csv --print-source cuda > $O/ncu_${tag}_cuda.csv 2>&1
ls -la $O
