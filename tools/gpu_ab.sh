# A/B of the strip ring copy width: 8-byte cp.async.ca (default) vs 16-byte cp.async.cg (PM_SR16=1)
CF="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -I include -I paper_1604_05937_b200/csrc"
for v in 8 16; do
  if [ $v = 16 ]; then
    /usr/local/cuda/bin/nvcc $CF -DPM_SR16=1 -c paper_1604_05937_b200/csrc/strip_red.cu -o build/obj/strip_red.cu.o && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1604_05937_b200/_native/libprismesh_cuda.so build/obj/*.o
    timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -m gpu -q -k "strip or CG1 or VP1 or long" > gpurun_out/pt16.log 2>&1; tail -1 gpurun_out/pt16.log
  fi
  for c in C5a C5b C4-CG1xCG1-rcm-L100 C4-CG1xCG1-rcm-L20 C4-VP1-rcm-L50 C4-CG1xDG1-rcm-L50; do python tools/time_op.py $c sr$v; done
done
