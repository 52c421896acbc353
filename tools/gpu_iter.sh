#!/bin/bash
# Iteration run on the GPU box: GPU parity tests (stop at first failure), then quick 6D/5D bench.
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_iter.log 2>&1; echo "pytest rc=$?" >> $O/pytest_iter.log
tail -25 $O/pytest_iter.log
if [ "${BENCH:-1}" = "1" ]; then CONFIGS="${CONFIGS:-6d 5d}" bash tools/quick_bench.sh iter > $O/quick_iter.txt 2>&1; cat $O/quick_iter.txt; fi
