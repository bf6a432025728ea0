# Full round measurement: tests, smoke, every config's bench line.
set -x
[ "$1" = quick ] || timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
: > gpurun_out/all.jsonl
for c in C1 C3 C4-CG1xCG1-rcm-L1 C4-CG1xCG1-rcm-L10 C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L256 \
         C4-CG1xCG1-random-L1 C4-CG1xCG1-random-L20 C4-CG1xCG1-random-L100 \
         C4-DG1xDG1-rcm-L1 C4-DG1xDG1-rcm-L20 C4-DG1xDG1-rcm-L100 C4-DG1xDG1-random-L1 C4-DG1xDG1-random-L100; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
done
timeout 900 python bench.py --config C5a --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
timeout 900 python bench.py --config C5b --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
python tools/summarize.py gpurun_out/bench_C2.json gpurun_out/all.jsonl
