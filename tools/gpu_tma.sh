# run-strip kernel (schedule "striptma") A/B against the cp.async strip
# kernel; every run bounded by a timeout (a deadlocked mbarrier wait must
# not hang the box)
for c in ${CONFIGS:-C5a C5b C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100}; do
  PM_SCHED=auto timeout 120 python -u tools/time_op.py $c base
  for lib in "" ${VARIANTS}; do
  for nq in 2 1; do for ns in 2 3; do
    PM_NATIVE_LIB=$lib PM_SCHED=striptma PM_TMA_NQ=$nq PM_TMA_NS=$ns timeout 120 python -u tools/time_op.py $c tma_nq${nq}_ns${ns}_$(basename "$lib" .so)
  done; done; done
done 2>&1 | tee gpurun_out/ab_tma.txt
