set -x
for lib in default idpf late both default both; do
  if [ $lib = default ]; then unset PM_NATIVE_LIB; else export PM_NATIVE_LIB=build/var/$lib.so; fi
  for c in C5b C5a C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100; do timeout 300 python tools/time_op.py $c $lib; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab5.txt
export PM_NATIVE_LIB=build/var/both.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "stripred or VP1 or CG1 or long" > gpurun_out/pytest_both.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_both.log
