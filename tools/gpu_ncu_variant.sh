#!/bin/bash
# full ncu capture of one experiment library: LIB=libhd_lean.so CFG=6d OP=adv bash tools/gpu_ncu_variant.sh
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
L=$PWD/paper_2002_08110_b200/${LIB:-libhd_lean.so}; c=${CFG:-6d}; op=${OP:-adv}; tag=${TAG:-var}_${c}_$op
HD_LIB_PATH=$L timeout 300 python tools/prof_driver.py --config $c --op $op --reps 3 > $O/plain_$tag.log 2>&1 || { echo plain failed; tail $O/plain_$tag.log; exit 1; }
HD_LIB_PATH=$L timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s 2 -c 1 \
   -o $O/ncu_$tag python tools/prof_driver.py --config $c --op $op --reps 3 > $O/ncu_$tag.log 2>&1
python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
python tools/ncu_lines.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_${tag}_lines.txt 2>&1
ncu -i $O/ncu_$tag.ncu-rep --page raw --csv > $O/ncu_${tag}_raw.csv 2>&1
sz=$(stat -c %s $O/ncu_$tag.ncu-rep 2>/dev/null || echo 0); [ "$sz" -gt 30000000 ] && rm -f $O/ncu_$tag.ncu-rep
head -30 $O/ncu_$tag.txt
