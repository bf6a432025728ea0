L=paper_1604_05937_b200/_native/libprismesh_cuda.so
cp build/exp/cslow.so $L
timeout 900 python -m pytest tests -m gpu -q -k "stripred or P2 or VP1" 2>&1 | tail -1
for v in cfast cslow cfast cslow; do
  cp build/exp/$v.so $L
  for c in C5a C5b C3; do echo "$v $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done
done
