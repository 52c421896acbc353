#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the small kernel-path driver (logs in gpurun_out/)
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_driver.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/sanitize_$tool.log
  tail -4 $O/sanitize_$tool.log
done
