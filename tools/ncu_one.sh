# usage: bash tools/ncu_one.sh <config> <schedule> <kernel-regex> <tag>
set -x
python bench.py --config $1 --schedule $2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o gpurun_out/prof_$4 -f \
  python bench.py --config $1 --schedule $2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$4.log 2>&1
tail -2 gpurun_out/ncu_$4.log
