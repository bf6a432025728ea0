# Re-entry sanity pass: GPU tests, smoke, default bench line, the CG configs.
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C3 C5a C5b; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$c.json
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
python tools/summarize.py gpurun_out/bench_C2.json gpurun_out/bench_C3.json gpurun_out/bench_C5a.json gpurun_out/bench_C5b.json
