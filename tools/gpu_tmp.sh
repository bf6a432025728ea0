for c in C5a C4-CG1xCG1-rcm-L100; do python tools/time_op.py $c new; done
timeout 600 python -m pytest tests/test_fused_halo.py tests/test_gpu_parity.py -m gpu -q -k "fused or strip or host" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
