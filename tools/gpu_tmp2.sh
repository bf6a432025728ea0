L=paper_1604_05937_b200/_native/libprismesh_cuda.so
cp build/exp/nocopy.so $L
for c in C5a C4-CG1xCG1-rcm-L50; do echo "nocopy $(timeout 600 python tools/ab_sched.py $c stripred 2>&1 | grep -v Warn | awk '{print $1, $3}')"; done
ncu --clock-control none --metrics gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum -k regex:k_strip_red -s 3 -c 1 python tools/ab_sched.py C5a stripred 2>&1 | grep "__"
