# levels-per-lane experiment for the strip-REDG kernel
for L in 1 2; do
  PM_STRIP_L=$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strip or host" 2>&1 | tail -2 > gpurun_out/pytest_L$L.log
done
: > gpurun_out/sl.jsonl
for c in C5a C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L256 C1; do
 for L in 1 2; do
  for w in 8 16; do
  PM_STRIP_W=$w PM_STRIP_L=$L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | sed "s/\"schedule\": \"auto\"/\"schedule\": \"L${L}W$w\"/" >> gpurun_out/sl.jsonl
  done
 done
done
cat gpurun_out/pytest_L*.log
python tools/summarize.py gpurun_out/sl.jsonl
