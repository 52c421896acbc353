#!/bin/bash
# FCL comparison path: its GPU tests, the 5D bench line (ECL and FCL timed on the same workload), the DRAM
# traffic of each FCL pass (5D) and one full ncu capture of the FCL cell pass. Outputs in gpurun_out/.
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_fcl.py -q -p no:cacheprovider > $O/pytest_fcl.log 2>&1; echo "pytest fcl rc=$?" >> $O/pytest_fcl.log
tail -5 $O/pytest_fcl.log
timeout 600 python bench.py --config 5d --no-cpu > $O/bench_5d_fcl.json 2> $O/bench_5d_fcl.err; echo "bench 5d rc=$?"
timeout 300 python tools/prof_driver.py --config 5d --op fcl --reps 3 > $O/plain_fcl.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:fcl_ -s 3 -c 3 --csv --log-file $O/traffic_5d_fcl.csv \
  python tools/prof_driver.py --config 5d --op fcl --reps 3 > $O/ncu_traffic_5d_fcl.log 2>&1; echo "traffic fcl rc=$?"
