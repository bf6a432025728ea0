set -x
for lib in default sr16 default sr16; do
  if [ $lib = default ]; then unset PM_NATIVE_LIB; else export PM_NATIVE_LIB=build/var/$lib.so; fi
  for c in C5b C5a C4-CG1xCG1-rcm-L20 C4-CG1xCG1-rcm-L100; do timeout 300 python tools/time_op.py $c $lib; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_sr16.txt
