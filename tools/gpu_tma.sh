# TMA-ring strip kernel (PM_STRIP_TMA=1): parity, then A/B against the cp.async ring
set -x
PM_STRIP_TMA=1 timeout 600 python tools/time_op.py C5a tma_smoke
PM_STRIP_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "stripred or CG1xCG1 or VP1 or long" > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_tma.log
for m in 0 1 0 1; do
  for c in C5a C5b C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100; do PM_STRIP_TMA=$m timeout 300 python tools/time_op.py $c tma$m; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_tma.txt
