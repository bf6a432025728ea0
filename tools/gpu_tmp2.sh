for L in 1 2 5 10 20 50 100 256; do
  for w in 8 16 32; do echo "L=$L W=$w $(PM_STRIP_W=$w timeout 600 python tools/ab_sched.py C4-CG1xCG1-rcm-L$L stripred 2>&1 | grep -v Warn | awk '{print $3}')"; done
done
