#!/bin/bash
# quick comparison runs: tools/quick_bench.sh "<label>" [env...] ; prints config, RK GDoF/s, A GDoF/s, frac
label=$1; shift
for c in ${CONFIGS:-5d 6d}; do
  env "$@" timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.loads(open('/tmp/b.json').read()); print('$label $c', round(d['value'],1), 'A', round(d['apply_advection']['gdofs'],1), 'frac', round(d['roofline']['frac'],3), 'mhz', d['clocks']['sm_mhz'])" || tail -3 /tmp/b.err
done
