timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shard.py -m gpu -x -q -k "strip or host or VP1 or shard" 2>&1 | tail -1
: > gpurun_out/v.jsonl
for c in C5b C4-VP1-rcm-L50 C4-VP1-rcm-L100; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/v.jsonl
done
python tools/summarize.py gpurun_out/v.jsonl
