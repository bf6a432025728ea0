timeout 900 python -m pytest tests -m gpu -q -x -k "stripred or strip_red or VP1 or CG1xCG1 or halo" 2>&1 | tail -1
for c in C5a C5b C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L20; do timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn; done
