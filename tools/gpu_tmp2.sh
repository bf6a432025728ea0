L=paper_1604_05937_b200/_native/libprismesh_cuda.so
cp build/exp/d6.so $L
timeout 900 python -m pytest tests -m gpu -q -x -k "stripred or strip_red or pstrip or patch_strips" 2>&1 | tail -2
for v in base d6; do
  cp build/exp/$v.so $L
  for c in C3 C5a C5b C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L20; do
    echo "$v $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn)"
  done
done
