# CG strip-REDG check: parity tests of the strip kernels + C3/C5a/C5b/C4 lines.
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strip or P2 or smoke or host" 2>&1 | tail -5 > gpurun_out/pytest_cg.log
: > gpurun_out/cg.jsonl
for c in C3 C5a C5b C4-CG1xCG1-rcm-L100 C4-VP1-rcm-L50; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/cg.jsonl
done
cat gpurun_out/pytest_cg.log
python tools/summarize.py gpurun_out/cg.jsonl
