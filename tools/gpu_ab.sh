set -e
(cd ab_old && python paper_1604_05937_b200/build_native.py > /dev/null 2>&1)
for c in C5a C4-CG1xCG1-rcm-L100; do
  python tools/time_op.py $c new
  (cd ab_old && python tools/time_op.py $c old)
done
