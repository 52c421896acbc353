#!/bin/bash
# GPU parity tests (+ smoke) on the box; output under gpurun_out/
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -12 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; cat $O/smoke.log
