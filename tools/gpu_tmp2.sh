L=paper_1604_05937_b200/_native/libprismesh_cuda.so
for v in sre0 sre1 sre0 sre1; do
  cp build/exp/$v.so $L
  echo "$v $(timeout 600 python tools/ab_sched.py C3 stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"
done
cp build/exp/sre1.so $L; timeout 900 python -m pytest tests -m gpu -q -k "P2" 2>&1 | tail -1
