"""Executed warp instructions by opcode from an ncu report's SASS page:
ncu_ophist.py report.ncu-rep [steps]  (per-step counts when `steps` given)"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
c = collections.Counter()
for r in rows[2:]:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[i_src])
    if m and r[i_ex].isdigit():
        c[m.group(2)] += int(r[i_ex])
tot = sum(c.values())
print("total", tot, "per step", round(tot / steps, 1))
for k, v in c.most_common(40):
    print(f"{k:10s} {v / steps:10.2f} {100 * v / tot:5.1f}%")
