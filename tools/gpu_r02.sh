#!/bin/bash
# Round-2 measurement set (outputs in gpurun_out/, summaries copied into profiles/ by hand):
#  bench lines (6D default, 5D, 4D with L2 flush, the CPU-oracle reference arm), the ncu launch list of the
#  bench command, DRAM traffic per launch of the fused stage kernel in RK and A modes (6D, 5D) and of the
#  mass kernel, and one full ncu capture of the RK and A kernels (6D) and the RK kernel (5D).
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_6d.json 2> $O/bench_6d.err; echo "bench 6d rc=$?"
timeout 600 python bench.py --config 5d > $O/bench_5d.json 2> $O/bench_5d.err; echo "bench 5d rc=$?"
timeout 600 python bench.py --config 4d --no-cpu --l2-flush > $O/bench_4d.json 2> $O/bench_4d.err; echo "bench 4d rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_6d.json 2> $O/bench_ref.err; echo "ref rc=$?"
# launch list of the bench command (same command, fewer steps; cold-cache serialised times: shares only)
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_6d.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_6d.csv > $O/launches_6d_summary.txt 2>&1
# DRAM traffic per launch (steady state)
for c in 6d 5d; do
  for op in rk adv mass; do
    k=cell_kernel; [ $op = mass ] && k=mass_kernel
    timeout 300 python tools/prof_driver.py --config $c --op $op --reps 3 > $O/plain_traffic_${c}_$op.log 2>&1 && \
    timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:$k -s 2 -c 1 --csv --log-file $O/traffic_${c}_$op.csv \
      python tools/prof_driver.py --config $c --op $op --reps 3 > $O/ncu_traffic_${c}_$op.log 2>&1
    echo "traffic $c $op rc=$?"
  done
done
# full captures
for spec in "6d rk 6" "6d adv 2" "5d rk 6"; do
  set -- $spec
  c=$1; op=$2; skip=$3; tag=full_${c}_$op
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cell_kernel -s $skip -c 1 \
     -o $O/ncu_$tag python tools/prof_driver.py --config $c --op $op --reps 3 > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_$tag.txt 2>&1
  python tools/ncu_lines.py $O/ncu_$tag.ncu-rep 40 > $O/ncu_${tag}_lines.txt 2>&1
  sz=$(stat -c %s $O/ncu_$tag.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 30000000 ]; then rm -f $O/ncu_$tag.ncu-rep; fi
done
du -sh $O
