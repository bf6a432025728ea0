for c in C3 C5a C5b; do
  for m in 128 256 512 4096; do echo "maxlen $m $(PM_STRIP_MAXLEN=$m timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn)"; done
done
