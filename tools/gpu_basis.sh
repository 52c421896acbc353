#!/bin/bash
# quick check of the basis-change kernel: parity tests, CUDA-event timing, one full ncu capture (6D)
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_gll.py -m gpu -q -p no:cacheprovider --durations=5 > $O/pytest_gll.log 2>&1; echo "pytest gll rc=$?" | tee -a $O/pytest_gll.log
tail -8 $O/pytest_gll.log
for c in 6d 5d 4d; do timeout 300 python tools/prof_driver.py --config $c --op basis --reps 3 --time 2>&1 | tee -a $O/basis_time.txt; done
timeout 300 python tools/prof_driver.py --config 6d --op mass --reps 3 --time 2>&1 | tee -a $O/basis_time.txt
for c in 6d 5d; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:basis_kernel -s 2 -c 1 --csv --log-file $O/traffic_${c}_basis.csv \
    python tools/prof_driver.py --config $c --op basis --reps 3 > $O/ncu_traffic_${c}_basis.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:basis_kernel -s 2 -c 1 \
   -o $O/ncu_full_6d_basis python tools/prof_driver.py --config 6d --op basis --reps 3 > $O/ncu_full_6d_basis.log 2>&1
python tools/ncu_summary.py $O/ncu_full_6d_basis.ncu-rep 40 > $O/ncu_full_6d_basis.txt 2>&1
python tools/ncu_lines.py $O/ncu_full_6d_basis.ncu-rep 30 > $O/ncu_full_6d_basis_lines.txt 2>&1
