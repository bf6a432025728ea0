"""Top stall sites of an ncu report's source page (SASS):
ncu_top.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_src = h.index("Source")
i_ex = h.index("Instructions Executed")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
val = [int(r[i_s]) if r[i_s].isdigit() else 0 for r in data]
tot = sum(val)
print("total samples", tot)
for j in sorted(range(len(data)), key=lambda j: -val[j])[:n]:
    r = data[j]
    print(f"{r[0][-5:]} {100 * val[j] / tot:5.1f}% {r[i_ex]:>10} "
          f"{r[i_src][:60]:60s} <- {data[j - 1][i_src][:45]}")
