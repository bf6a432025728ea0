python tools/time_op.py C4-DG1xCG1-rcm-L100 x overwrite > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cell_stream -s 2 -c 1 -o gpurun_out/prof_cell -f python tools/time_op.py C4-DG1xCG1-rcm-L100 x overwrite > gpurun_out/ncu_cell.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_cell.ncu-rep | head -22 | tail -18
ncu -i gpurun_out/prof_cell.ncu-rep --page source --csv --print-source sass 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[1]; rows=r[2:]
cols=[c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot={c:0 for c in cols}
for x in rows:
    for c in cols:
        v=x[h.index(c)]
        if v.replace('.','').isdigit(): tot[c]+=float(v)
T=sum(tot.values())
for c,v in sorted(tot.items(), key=lambda kv:-kv[1])[:6]: print(f'{c:28s} {100*v/T:5.1f}%')
i_s=h.index('Warp Stall Sampling (All Samples)')
for k in sorted(range(len(rows)),key=lambda k:-int(rows[k][i_s]) if rows[k][i_s].isdigit() else 0)[:6]:
    print('----', rows[k][i_s])
    for y in rows[max(0,k-6):k+2]: print(y[i_s].rjust(6), y[1][:90])
"
