: > gpurun_out/wsweep.jsonl
for cfg in C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L100 C3; do
 for w in 8 16 32; do
  PM_COLUMN_W=$w timeout 300 python bench.py --config $cfg --schedule column --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"column\"/\"schedule\": \"colW$w\"/" >> gpurun_out/wsweep.jsonl
 done
 timeout 300 python bench.py --config $cfg --schedule strip --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/wsweep.jsonl
done
timeout 600 python bench.py --config C5b --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/wsweep.jsonl
python tools/summarize.py gpurun_out/wsweep.jsonl
