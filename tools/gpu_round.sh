# One GPU session: tests, smoke, bench sweep.  Usage: bash tools/gpu_round.sh [quick]
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ "$1" = quick ] || timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
: > gpurun_out/sweep.jsonl
for cs in "C2 auto"; do
  set -- $cs
  timeout 300 python bench.py --config $1 --schedule $2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sweep.jsonl
done
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
python tools/summarize.py gpurun_out/sweep.jsonl gpurun_out/bench_C2.json
