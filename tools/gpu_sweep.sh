# The paper's layout x ordering x layers sweep (~15M cell-layers per point)
rm -f gpurun_out/layout_sweep.csv
timeout 2400 python -m paper_1604_05937_b200 bench --horiz CG1,DG0,DG1 --vert CG1,DG0,DG1 \
  --ordering rcm,random --layers 1,2,5,10,20,50,100 --target-cells 15000000 \
  --repeats 10 --out gpurun_out/layout_sweep.csv 2> gpurun_out/layout_sweep.err
wc -l gpurun_out/layout_sweep.csv; tail -2 gpurun_out/layout_sweep.err
