# ncu captures of the top kernels (run after the plain commands exit 0).
set -x
python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/plain_C2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dg_stream -s 2 -c 1 \
    -o gpurun_out/prof_C2_stream -f python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_C2.log 2>&1
python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_C3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_column -s 1 -c 1 \
    -o gpurun_out/prof_C3_column -f python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_C3.log 2>&1
python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/plain_C2b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
