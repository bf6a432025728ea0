"""Opcode histogram of the main loop (third backward branch) of one or two
kernels' SASS (cuobjdump -sass of one function):  sass_hist.py a.sass [b.sass]"""
import collections
import re
import subprocess
import sys


def loop(f):
    out = subprocess.run([sys.executable, __file__.replace("sass_hist", "sass_loops"), f],
                         capture_output=True, text=True).stdout.splitlines()
    a, b = re.findall(r"0x[0-9a-f]+", out[2])[:2]
    return int(a, 16), int(b, 16)


def hist(f):
    lo, hi = loop(f)
    c = collections.Counter()
    for line in open(f):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and lo <= int(m.group(1), 16) <= hi:
            c[m.group(3)] += 1
    return c


hs = [hist(f) for f in sys.argv[1:]]
keys = sorted(set().union(*hs), key=lambda k: -(hs[-1][k] - hs[0][k]))
for k in keys:
    print(f"{k:12s} " + " ".join(f"{h[k]:5d}" for h in hs) +
          (f" {hs[-1][k] - hs[0][k]:+d}" if len(hs) > 1 else ""))
