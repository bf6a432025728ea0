for c in C5a C5b; do
ncu --set full --clock-control none --import-source on -k k_strip_red -s 1 -c 1 \
    -o gpurun_out/prof_${c}_stripred -f python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_${c}_stripred.ncu-rep > gpurun_out/prof_${c}_stripred.txt 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_strip_red -s 1 -c 1 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "__" > gpurun_out/traffic_C3.txt
