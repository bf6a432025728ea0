timeout 900 python -m pytest tests -m gpu -q -x -k "patch_strips or pstrip" 2>&1 | tail -1
for c in C5b C3; do
  timeout 600 python tools/ab_sched.py $c stripred pstrip 2>&1 | grep -v Warn
  for P in 64 128 256 1024; do echo "P=$P $(PM_PATCH_CELLS=$P timeout 600 python tools/ab_sched.py $c pstrip 2>&1 | grep -v Warn)"; done
done
