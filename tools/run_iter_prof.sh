timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=8 > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -15 gpurun_out/pytest_iter.log
HD_LIB_PATH=$PWD/paper_2002_08110_b200/libhd_bench.so CONFIGS="6d 5d" bash tools/quick_bench.sh bench
CONFIGS=6d bash tools/gpu_prof.sh
