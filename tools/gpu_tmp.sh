timeout 600 python -m pytest tests/test_edge_cases.py -m gpu -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
: > gpurun_out/dg.jsonl
for c in C2 C2 C4-DG1xDG1-rcm-L20 C4-DG1xDG1-rcm-L100 C3 C1; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/dg.jsonl
done
python tools/summarize.py gpurun_out/dg.jsonl
