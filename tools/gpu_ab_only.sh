VARIANTS="$1" CONFIGS="6d 5d" bash tools/gpu_ab.sh
