#!/bin/bash
# trace-source counts per launch (HD_COUNT experiment builds)
O=gpurun_out
for L in ${LIBS:-libhd_basec.so libhd_leanc.so}; do for c in ${CFGS:-6d 5d}; do for op in ${OPS:-rk adv}; do
  echo "== $L $c $op"
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$L timeout 300 python tools/prof_driver.py --config $c --op $op --reps 2 2>&1 | grep HDCOUNT | tail -3
done; done; done
