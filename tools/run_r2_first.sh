O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
./tools/mb2 > $O/mb2.jsonl 2>&1
CONFIGS="6d 5d" bash tools/quick_bench.sh base > $O/quick_base.txt 2>&1
cat $O/mb2.jsonl $O/quick_base.txt
