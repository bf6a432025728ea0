set -x
for lib in tm8 tm12; do
  export PM_NATIVE_LIB=build/var/$lib.so
  for c in C5a C5b C4-CG1xCG1-rcm-L100; do PM_STRIP_TMA=1 timeout 300 python tools/time_op.py $c $lib; done
done 2>&1 | grep -v "^+" | tee gpurun_out/ab_tma2.txt
