: > gpurun_out/sw.jsonl
for c in C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L256 C1; do
 for w in 8 16 32; do
  PM_STRIP_W=$w timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"W$w\"/" >> gpurun_out/sw.jsonl
 done
done
timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sw.jsonl
python tools/summarize.py gpurun_out/sw.jsonl
