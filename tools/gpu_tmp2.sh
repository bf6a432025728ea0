PM_STREAM_WS=1 timeout 900 python -m pytest tests -m gpu -q -x -k "DG1xDG1 or stream or host_pipelined" 2>&1 | tail -1
for r in 0 1 2 3 0; do
  echo "ws $r: $(PM_STREAM_WS=$r timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["value"], d["roofline"]["frac"])')"
done
for c in C4-DG1xDG1-rcm-L20 C4-DG1xDG1-rcm-L256; do for r in 0 1; do
  echo "$c ws $r: $(PM_STREAM_WS=$r timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["value"], d["roofline"]["frac"])')"
done; done
