#!/bin/bash
# Round-2 closing run: GLL basis-change tests first, the whole GPU suite + smoke, bench lines (6D default, 5D, the
# reference arm), the ncu launch list of the bench command, DRAM traffic and one full capture of basis_kernel.
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_gll.py -m gpu -q -p no:cacheprovider --durations=5 > $O/pytest_gll.log 2>&1; echo "pytest gll rc=$?" | tee -a $O/pytest_gll.log
tail -15 $O/pytest_gll.log
timeout 900 python bench.py > $O/bench_6d.json 2> $O/bench_6d.err; echo "bench 6d rc=$?"
timeout 600 python bench.py --config 5d > $O/bench_5d.json 2> $O/bench_5d.err; echo "bench 5d rc=$?"
for c in 6d 5d; do
  timeout 300 python tools/prof_driver.py --config $c --op basis --reps 3 > $O/plain_traffic_${c}_basis.log 2>&1 && \
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:basis_kernel -s 2 -c 1 --csv --log-file $O/traffic_${c}_basis.csv \
    python tools/prof_driver.py --config $c --op basis --reps 3 > $O/ncu_traffic_${c}_basis.log 2>&1
  echo "traffic $c basis rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:basis_kernel -s 2 -c 1 \
   -o $O/ncu_full_6d_basis python tools/prof_driver.py --config 6d --op basis --reps 3 > $O/ncu_full_6d_basis.log 2>&1
python tools/ncu_summary.py $O/ncu_full_6d_basis.ncu-rep 40 > $O/ncu_full_6d_basis.txt 2>&1
python tools/ncu_lines.py $O/ncu_full_6d_basis.ncu-rep 30 > $O/ncu_full_6d_basis_lines.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_6d.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_6d.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_6d.csv > $O/launches_6d_summary.txt 2>&1
du -sh $O
