L=paper_1604_05937_b200/_native/libprismesh_cuda.so
for v in st256 st128 st512 st256 st128; do
  cp build/exp/$v.so $L
  for c in C5a C4-CG1xCG1-rcm-L50; do echo "$v $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done
done
cp build/exp/st256.so $L
