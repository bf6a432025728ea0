# CLI harness on the GPU: its tests, verify, stream, and the paper's
# layout x ordering x layers sweep at ~15M cell-layers (PAPER 4.1.3)
timeout 900 python -m pytest tests/test_cli.py -m gpu -x -q 2>&1 | tail -3
python -m paper_1604_05937_b200 verify 2>&1 | tail -3
python -m paper_1604_05937_b200 stream
rm -f gpurun_out/layout_sweep.csv
timeout 2400 python -m paper_1604_05937_b200 bench --horiz CG1,DG0,DG1 --vert CG1,DG0,DG1 \
  --ordering rcm,random --layers 1,2,5,10,20,50,100 --target-cells 15000000 \
  --repeats 10 --out gpurun_out/layout_sweep.csv 2> gpurun_out/layout_sweep.err
tail -3 gpurun_out/layout_sweep.err; wc -l gpurun_out/layout_sweep.csv
