#!/bin/bash
O=gpurun_out
: > $O/quick.txt
CONFIGS="4d 5d 6d" STEPS=3 bash tools/quick_bench.sh jouter >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_mesh_operators or config_full" -p no:cacheprovider 2>&1 | tail -2
