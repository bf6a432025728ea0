# Round-end measurement pass: GPU tests, smoke, headline bench line (with
# CPU baseline) and the reference arm, every config, the config-4 sweep,
# the launch list and one ncu --set full capture per dominant kernel.
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
: > gpurun_out/all.jsonl
for c in C1 C3 C5a C5b; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
done
for lay in CG1xCG1 DG1xDG1; do for o in rcm random; do for L in 1 2 5 10 20 50 100 256; do
  timeout 300 python bench.py --config C4-$lay-$o-L$L --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/all.jsonl
done; done; done
python tools/summarize.py gpurun_out/bench_C2.json gpurun_out/all.jsonl > gpurun_out/all.txt
# launch list of the default bench command
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dg_stream -s 4 -c 1 \
    -o gpurun_out/prof_C2_stream -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_strip_red_e -s 1 -c 1 \
    -o gpurun_out/prof_C3_stripred_e -f python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k k_strip_red -s 1 -c 1 \
    -o gpurun_out/prof_C5a_stripred -f python bench.py --config C5a --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c5a.log 2>&1
for r in gpurun_out/prof_C2_stream gpurun_out/prof_C3_stripred_e gpurun_out/prof_C5a_stripred; do
  python tools/ncu_summary.py $r.ncu-rep > $r.txt 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/all.txt | head -60
ncu --set full --clock-control none --import-source on -k k_strip_red -s 1 -c 1 \
    -o gpurun_out/prof_C5b_stripred -f python bench.py --config C5b --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c5b.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_C5b_stripred.ncu-rep > gpurun_out/prof_C5b_stripred.txt 2>&1
