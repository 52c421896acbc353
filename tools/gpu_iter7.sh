#!/bin/bash
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
: > $O/quick.txt
CONFIGS="4d 5d 6d" STEPS=3 bash tools/quick_bench.sh v5 >> $O/quick.txt 2>&1
CONFIGS="5d 6d" STEPS=3 bash tools/quick_bench.sh v5-skew1 HD_SKEW=1 >> $O/quick.txt 2>&1
grep -v "^ \|Trace\|File\|json\|^$" $O/quick.txt
for c in 5d; do
  tag=v5_$c
  timeout 300 python tools/prof_driver.py --config $c --op rk --reps 2 > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s 6 -c 1 \
     -o $O/ncu_$tag python tools/prof_driver.py --config $c --op rk --reps 2 > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
  sz=$(stat -c %s $O/ncu_$tag.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 50000000 ]; then rm -f $O/ncu_$tag.ncu-rep; fi
done
du -sh $O
