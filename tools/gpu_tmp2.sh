for c in C5b C5a C3; do for w in 16 32; do echo "W=$w $(PM_STRIP_W=$w timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done; done
