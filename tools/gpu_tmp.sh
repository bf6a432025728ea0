timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "P2" 2>&1 | tail -1
: > gpurun_out/c3b.jsonl
for b in 1 0; do for w in 8 16 32; do
PM_STRIP_BULKRED=$b PM_STRIP_W=$w timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"B${b}W$w\"/" >> gpurun_out/c3b.jsonl
done; done
python tools/summarize.py gpurun_out/c3b.jsonl
