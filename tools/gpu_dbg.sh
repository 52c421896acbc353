#!/bin/bash
O=gpurun_out
for kv in ws base; do
  HD_KERNEL=$kv timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -k "$KSEL" > $O/dbg_$kv.log 2>&1
  grep -E "passed|failed|FAILED" $O/dbg_$kv.log | head -40
done
