set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "sharded or halo" 2>&1 | tail -5 > gpurun_out/pytest_shard.log
timeout 900 python bench.py --config C5a --steps 10 --warmup 3 > gpurun_out/bench_C5a.json 2> gpurun_out/bench_C5a.err
timeout 900 python bench.py --config C5b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5b.json 2> gpurun_out/bench_C5b.err
python bench.py --config C4-CG1xCG1-rcm-L50 --schedule column --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_column -s 1 -c 1 -o gpurun_out/prof_C4P1_column -f \
  python bench.py --config C4-CG1xCG1-rcm-L50 --schedule column --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_p1.log 2>&1
cat gpurun_out/pytest_shard.log
python tools/summarize.py gpurun_out/bench_C5a.json gpurun_out/bench_C5b.json
tail -3 gpurun_out/bench_C5a.err
