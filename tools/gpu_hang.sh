#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -v --timeout 100 -p no:cacheprovider > $O/pytest_v.log 2>&1; echo "rc=$?" >> $O/pytest_v.log
grep -E "PASSED|FAILED|ERROR|Timeout|rc=" $O/pytest_v.log | tail -60
