timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_quadrature_rules.py -m gpu -x -q -k "strip or P2 or smoke or host or custom or VP1 or CG1" 2>&1 | tail -2
: > gpurun_out/cg.jsonl
for c in C5a C5b C4-CG1xCG1-rcm-L100 C4-VP1-rcm-L50 C4-CG1xDG1-rcm-L50; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/cg.jsonl
done
python tools/summarize.py gpurun_out/cg.jsonl
