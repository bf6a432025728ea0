PM_DG_RING=1 timeout 900 python -m pytest tests -m gpu -q -x -k "DG or dg or stream or smoke" 2>&1 | tail -2
for r in 0 1 2 3 4; do
  echo "ring $r: $(PM_DG_RING=$r timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["value"], d["roofline"]["frac"])')"
done
for c in C4-DG1xDG1-rcm-L20 C4-DG1xDG1-rcm-L256 C4-DG1xDG1-random-L100; do for r in 0 1; do
  echo "$c ring $r: $(PM_DG_RING=$r timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["value"], d["roofline"]["frac"])')"
done; done
