#!/bin/bash
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
# 6D source-level stall profile (application replay: no 140 GB save/restore per pass)
timeout 300 python tools/prof_driver.py --config 6d --op rk --reps 1 > $O/plain_6d.log 2>&1 && \
timeout 1500 ncu --replay-mode application --section SourceCounters --section WarpStateStats --section SpeedOfLight \
   --import-source on --clock-control none -k regex:cell_kernel -s 3 -c 1 \
   -o $O/ncu_src_6d python tools/prof_driver.py --config 6d --op rk --reps 1 > $O/ncu_src_6d.log 2>&1
ls -la $O
