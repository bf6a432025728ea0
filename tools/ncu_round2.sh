set -x
python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/plain_C2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dg_stream -s 2 -c 1 \
    -o gpurun_out/prof_C2_stream2 -f python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_C2.log 2>&1
python bench.py --config C3 --schedule patch --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_C3p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_patch -s 1 -c 1 \
    -o gpurun_out/prof_C3_patch -f python bench.py --config C3 --schedule patch --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_C3p.log 2>&1
ls gpurun_out
