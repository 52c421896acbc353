#!/bin/bash
O=gpurun_out
for env in "HD_DISCARD=1" "HD_DISCARD=0" "HD_TRACE=0" "HD_SKEW=0"; do
  echo "== $env" >> $O/dbg2.txt
  env $env timeout 120 python tools/prof_driver.py --config 6d --op rk --reps 2 >> $O/dbg2.txt 2>&1
  tail -2 $O/dbg2.txt
done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
