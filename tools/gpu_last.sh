#!/bin/bash
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log; tail -3 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_gll.py -m gpu -q -p no:cacheprovider > $O/pytest_gll.log 2>&1; echo "pytest gll rc=$?" | tee -a $O/pytest_gll.log
tail -8 $O/pytest_gll.log
