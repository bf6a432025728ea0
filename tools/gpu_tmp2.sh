for c in C3 C5a; do
  timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn
  for o in morton rcm; do for P in 32 64 128 256; do
    echo "order $o P $P: $(PM_PATCH_ORDER=$o PM_PATCH_CELLS=$P timeout 600 python tools/ab_sched.py $c pstrip 2>&1 | grep -v Warn)"
  done; done
done
