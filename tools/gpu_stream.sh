: > gpurun_out/stream.jsonl
for cfg in 1 0 2 3; do
 for c in C2 C4-DG1xDG1-rcm-L100; do
  PM_STREAM_CFG=$cfg timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"cfg$cfg\"/" >> gpurun_out/stream.jsonl
 done
done
PM_STREAM_CFG=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C2 or DG1xDG1 or DG0xDG1" 2>&1 | tail -2
PM_STREAM_CFG=3 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C2 or DG1xDG1 or DG0xDG1" 2>&1 | tail -2
python tools/summarize.py gpurun_out/stream.jsonl
