bash tools/ncu_one.sh C5a auto "k_strip_red" C5a_sr_r2
python tools/ncu_summary.py gpurun_out/prof_C5a_sr_r2.ncu-rep > gpurun_out/ncu_C5a_sr_r2.txt 2>&1
cat gpurun_out/ncu_C5a_sr_r2.txt
ncu -i gpurun_out/prof_C5a_sr_r2.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]; v=r[2] if len(r)>2 else r[1]
for name,val in zip(h,v):
    if 'warp_issue_stalled' in name and 'pct' in name and 'not_issued' not in name:
        try:
            if float(val)>2: print(name,val)
        except: pass
" > gpurun_out/stalls_C5a.txt
cat gpurun_out/stalls_C5a.txt
