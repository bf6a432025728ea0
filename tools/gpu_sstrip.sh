# stacked store-first strips: parity, then A/B against the global strips
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "sstrip or stacked" > gpurun_out/pytest_sstrip.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_sstrip.log
for c in C5a C5b C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100; do
  timeout 300 python tools/ab_sched.py $c stripred sstrip
  PM_STACK_DEPTH=2 timeout 300 python tools/ab_sched.py $c sstrip
  PM_STACK_DEPTH=8 PM_STACK_MAXLEN=64 timeout 300 python tools/ab_sched.py $c sstrip
  PM_STACK_DEPTH=4 PM_STACK_MAXLEN=256 timeout 300 python tools/ab_sched.py $c sstrip
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_sstrip.txt
