# deferred staged-row REDs (PM_SR_DEFER): parity on the staged layouts, A/B
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py tests/test_fused_halo.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "VP1 or P2 or stripred or long or fused" > gpurun_out/pytest_defer.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_defer.log
for lib in default df0; do
  if [ $lib = default ]; then unset PM_NATIVE_LIB; else export PM_NATIVE_LIB=build/var/$lib.so; fi
  for c in C5b C3 C5a; do timeout 300 python tools/time_op.py $c $lib; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_defer.txt
