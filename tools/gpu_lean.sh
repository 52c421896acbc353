#!/bin/bash
# A/B of the lean (2 CTAs/SM) experiment build against the base build + its parity tests + DRAM traffic
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
L=$PWD/paper_2002_08110_b200/${LEANLIB:-libhd_lean.so}
HD_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
  -k "(config_full_parity and not 2d) or config_6d or 6d_full or reuse_flags" > $O/lean_tests.log 2>&1; tail -3 $O/lean_tests.log
VARIANTS="${VARIANTS:-libhd_base.so ${LEANLIB:-libhd_lean.so}}" CONFIGS="6d 5d" bash tools/gpu_ab.sh
for op in ${OPS:-rk adv}; do
HD_LIB_PATH=$L timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,sass__inst_executed_local_loads \
      --clock-control none -k regex:cell_kernel -s 2 -c 1 --csv --log-file $O/lean_traffic_6d_$op.csv \
      python tools/prof_driver.py --config 6d --op $op --reps 3 > /dev/null 2>&1
python - $O/lean_traffic_6d_$op.csv <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    print(r[h.index("Metric Name")], r[h.index("Metric Value")], r[h.index("Metric Unit")])
PY
done
