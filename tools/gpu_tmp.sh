timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -m gpu -q -k "P2" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for w in 8 16 32; do PM_STRIP_W=$w python tools/time_op.py C3 W$w; done
