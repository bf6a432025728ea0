set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2>&1
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.json 2>&1
timeout 600 python bench.py --config C3 --schedule colored --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_col.json 2>&1
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_C2.json gpurun_out/bench_C2.err | tail -5
