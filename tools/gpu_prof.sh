#!/bin/bash
# ncu captures of the fused stage kernel + knob comparison. Output under gpurun_out/.
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh base > $O/knobs.txt 2>&1
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh notrace HD_TRACE=0 >> $O/knobs.txt 2>&1
for c in 5d 6d; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s 6 -c 1 \
     -o $O/ncu_rk_$c python tools/prof_driver.py --config $c --op rk --reps 2 > $O/ncu_rk_$c.log 2>&1
done
