#!/bin/bash
# Round-2 closing evidence at the final commit: bench lines (6D default, 5D), the whole GPU suite, smoke.
O=gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > $O/bench_6d.json 2> $O/bench_6d.err; echo "bench 6d rc=$?"
timeout 600 python bench.py --config 5d > $O/bench_5d.json 2> $O/bench_5d.err; echo "bench 5d rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
