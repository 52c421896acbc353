#!/bin/bash
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "d6 or d5k3" > $O/dbg3_par.txt 2>&1; tail -5 $O/dbg3_par.txt
echo "== default 6d" >> $O/dbg3.txt
timeout 120 python tools/prof_driver.py --config 6d --op rk --reps 2 >> $O/dbg3.txt 2>&1; tail -1 $O/dbg3.txt
echo "== adv 6d" >> $O/dbg3.txt
timeout 120 python tools/prof_driver.py --config 6d --op adv --reps 2 >> $O/dbg3.txt 2>&1; tail -1 $O/dbg3.txt
echo "== minb2 6d" >> $O/dbg3.txt
HD_LIB_PATH=$PWD/paper_2002_08110_b200/libhd_minb2.so timeout 120 python tools/prof_driver.py --config 6d --op rk --reps 2 >> $O/dbg3.txt 2>&1; tail -1 $O/dbg3.txt
echo "== small 6d cells 4" >> $O/dbg3.txt
timeout 120 python tools/prof_driver.py --config 6d --cells 4,4,4,4,4,4 --op rk --reps 2 >> $O/dbg3.txt 2>&1; tail -1 $O/dbg3.txt
