for L in 10 20 50 100; do for it in 3000 6000 12000; do for w in 16 32; do
  echo "L=$L items=$it W=$w $(PM_STRIP_ITEMS=$it PM_STRIP_W=$w timeout 600 python tools/ab_sched.py C4-CG1xCG1-rcm-L$L stripred 2>&1 | grep -v Warn | awk '{print $3}')"
done; done; done
for it in 3000 6000 12000; do echo "C3 items=$it $(PM_STRIP_ITEMS=$it timeout 600 python tools/ab_sched.py C3 stripred 2>&1 | grep -v Warn | awk '{print $3}')"; done
