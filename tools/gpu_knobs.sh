#!/bin/bash
# env-knob A/B on the 6D/5D benches (each twice): KNOBS="HD_X=0 HD_SKEW=3 ..." bash tools/gpu_knobs.sh
for rep in 1 2; do
  for kv in ${KNOBS:-"HD_X=0"}; do CONFIGS="${CONFIGS:-6d 5d}" bash tools/quick_bench.sh "$kv" $kv; done
done
