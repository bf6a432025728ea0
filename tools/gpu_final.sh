# Round measurement pass: tests, smoke, headline + reference arm, every
# config's bench line, ncu of the C3 kernel.  bash tools/gpu_final.sh [quick]
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
[ "$1" = quick ] || timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
: > gpurun_out/all.jsonl
for c in C1 C2 C3 C4-CG1xCG1-rcm-L1 C4-CG1xCG1-rcm-L2 C4-CG1xCG1-rcm-L5 C4-CG1xCG1-rcm-L10 C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L256 \
         C4-CG1xCG1-random-L1 C4-CG1xCG1-random-L20 C4-CG1xCG1-random-L100 C4-CG1xCG1-random-L256 \
         C4-DG1xDG1-rcm-L1 C4-DG1xDG1-rcm-L2 C4-DG1xDG1-rcm-L5 C4-DG1xDG1-rcm-L10 C4-DG1xDG1-rcm-L20 C4-DG1xDG1-rcm-L50 C4-DG1xDG1-rcm-L100 C4-DG1xDG1-rcm-L256 \
         C4-DG1xDG1-random-L1 C4-DG1xDG1-random-L20 C4-DG1xDG1-random-L100 C4-DG1xDG1-random-L256 C5a C5b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
done
timeout 600 bash tools/ncu_one.sh C3 auto k_strip_red_e C3
# the run-strip kernel (C5a, auto): ncu --set full summary, opcode histogram, top stall sites
CFG=C5a TAG=final timeout 600 bash tools/gpu_tma_ncu.sh
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
python tools/summarize.py gpurun_out/bench_C5.json gpurun_out/all.jsonl
