timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "P2" 2>&1 | tail -2
: > gpurun_out/c3.jsonl
for w in 8 16 32; do
PM_STRIP_W=$w timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"W$w\"/" >> gpurun_out/c3.jsonl
done
python tools/summarize.py gpurun_out/c3.jsonl
