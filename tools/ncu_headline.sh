set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_head.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_head2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dg_stream -s 4 -c 1 \
    -o gpurun_out/prof_C2_stream_final -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_head.log 2>&1
python bench.py --config C5a --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_strip_red -s 1 -c 1 \
    -o gpurun_out/prof_C5a_stripred -f python bench.py --config C5a --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1
ls gpurun_out/*.ncu-rep
