L=paper_1604_05937_b200/_native/libprismesh_cuda.so
cp build/exp/pack.so $L
timeout 900 python -m pytest tests -m gpu -q -k "stripred or strip_red or VP1 or CG1xCG1 or CG1xDG or halo or pstrip or patch_strips" 2>&1 | tail -1
for v in nopack pack nopack pack; do
  cp build/exp/$v.so $L
  for c in C5a C5b C4-CG1xCG1-rcm-L50 C4-CG1xCG1-rcm-L20; do echo "$v $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done
done
