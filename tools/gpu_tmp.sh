: > gpurun_out/e2e.jsonl
for mb in 40 16 8 4; do
PM_HOST_CHUNK_MB=$mb timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"mb$mb\"/" >> gpurun_out/e2e.jsonl
done
python tools/summarize.py gpurun_out/e2e.jsonl
