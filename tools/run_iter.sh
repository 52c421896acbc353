#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=5 > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -8 gpurun_out/pytest_iter.log
LIBS="${LIBS:-libhd_bench.so}" bash tools/run_ab.sh
[ -n "$PROF" ] && CONFIGS="$PROF" bash tools/gpu_prof.sh
true
