# run-strip kernel (schedule "striptma"): parity first (bounded by timeouts:
# a deadlocked mbarrier wait must not hang the box), then A/B against the
# cp.async strip kernel
set -x
timeout 600 python -m pytest tests/test_strip_tma.py -m gpu -q -x -p no:cacheprovider --timeout 120 > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_tma.log
for c in ${CONFIGS:-C5a C5b C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100}; do
  PM_SCHED=auto timeout 300 python tools/time_op.py $c base
  for lib in "" ${VARIANTS}; do
  for g in 2 4; do for ns in 2 3; do
    PM_NATIVE_LIB=$lib PM_SCHED=striptma PM_TMA_G=$g PM_TMA_NS=$ns timeout 300 python tools/time_op.py $c tma_g${g}_ns${ns}_$(basename "$lib" .so)
  done; done; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_tma.txt
