# A/B of native-library variants (build/var/*.so) on the CG strip kernels
set -x
for lib in default os3 os6; do
  if [ $lib = default ]; then unset PM_NATIVE_LIB; else export PM_NATIVE_LIB=build/var/$lib.so; fi
  for c in C5a C5b C3 C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100; do timeout 300 python tools/time_op.py $c $lib; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab2.txt
