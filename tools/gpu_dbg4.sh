#!/bin/bash
O=gpurun_out
for v in libhd.so libhd_nohint.so libhd_r232.so libhd_minb2.so; do
  echo "== $v" >> $O/dbg4.txt
  HD_LIB_PATH=$PWD/paper_2002_08110_b200/$v timeout 120 python tools/prof_driver.py --config 6d --cells 4,4,4,4,4,4 --op rk --reps 2 >> $O/dbg4.txt 2>&1; tail -1 $O/dbg4.txt
done
