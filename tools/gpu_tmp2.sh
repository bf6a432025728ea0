L=paper_1604_05937_b200/_native/libprismesh_cuda.so
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in pack fold pack fold; do
  cp build/exp/$v.so $L
  for c in C3 C5a C5b; do echo "$v $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done
done
cp build/exp/fold.so $L
