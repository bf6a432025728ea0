PM_STREAM_CFG=7 timeout 600 python -m pytest tests -m gpu -q -k "DG1xDG1 or stream or host_pipelined" 2>&1 | tail -1
for r in 1 7 8 9 1 7 8 9; do
  echo "cfg $r: $(PM_STREAM_CFG=$r timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],5), round(d["roofline"]["kernel_ms"],5), round(d["value"]), round(d["roofline"]["frac"],4))')"
done
