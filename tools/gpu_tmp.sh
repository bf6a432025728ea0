timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strip or host" 2>&1 | tail -1
: > gpurun_out/g.jsonl
for c in C2 C1 C3 C5a C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100 C4-CG1xDG1-rcm-L50 C4-DG1xDG1-rcm-L20; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>gpurun_out/g_$c.err | tail -1 >> gpurun_out/g.jsonl
done
python tools/summarize.py gpurun_out/g.jsonl
tail -3 gpurun_out/g_C2.err
