PM_STRIP_BULK=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stripred or sharded or smoke" 2>&1 | tail -3
: > gpurun_out/bulk.jsonl
for c in C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L256; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bulk.jsonl
  PM_STRIP_BULK=1 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed 's/"schedule": "auto"/"schedule": "bulk"/' >> gpurun_out/bulk.jsonl
done
python tools/summarize.py gpurun_out/bulk.jsonl
