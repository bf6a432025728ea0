timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -v 2>&1 | tail -40 > gpurun_out/pytest_crash.log
