"""Stall reasons of an ncu report summed over SASS address ranges; the
ranges are the loops (backward branches) containing a marker mnemonic:
ncu_region.py report.ncu-rep [marker=REDG]"""
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
data = rows[2:]
marker = sys.argv[2] if len(sys.argv) > 2 else "REDG"
addr = [int(r[0], 16) for r in data]
base = addr[0]
src = [r[h.index("Source")] for r in data]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
i_ex = h.index("Instructions Executed")
# innermost loop containing the marker
loops = []
for j, s in enumerate(src):
    m = re.search(r"BRA\S*\s+(0x[0-9a-f]+)", s)
    if m and "@" not in s.split("BRA")[0][-3:]:
        pass
    if m:
        tgt = int(m.group(1), 16)
        if tgt < addr[j]:
            loops.append((tgt, addr[j]))
cand = [(a, b) for a, b in loops
        if any(marker in src[k] for k in range(len(src)) if a <= addr[k] <= b)]
cand.sort(key=lambda ab: ab[1] - ab[0])
lo, hi = cand[0]


def summ(sel):
    tot = {c: 0 for c in reasons}
    ins = 0
    for j in sel:
        for c in reasons:
            v = data[j][idx[c]]
            tot[c] += int(v) if v.isdigit() else 0
        ins += int(data[j][i_ex]) if data[j][i_ex].isdigit() else 0
    return tot, ins


inside = [j for j in range(len(data)) if lo <= addr[j] <= hi]
outside = [j for j in range(len(data)) if not lo <= addr[j] <= hi]
for name, sel in (("loop", inside), ("rest", outside)):
    tot, ins = summ(sel)
    s = sum(tot.values())
    print(f"{name} {lo - base:#x}..{hi - base:#x} ({len(sel)} instr, "
          f"{ins} executed): {s} samples")
    for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
        print(f"   {c:22s} {v:8d} {100 * v / max(s, 1):5.1f}%")
