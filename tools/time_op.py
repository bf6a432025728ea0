"""Time MassOperator.apply for a workload without bench.py (A/B helper)."""
import sys
import time

import os
sys.path.insert(0, os.getcwd())
import torch

from paper_1604_05937_b200 import configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator

w = configs.workload(sys.argv[1])
fs, quad, x_np, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
sched = os.environ.get("PM_SCHED", "auto")   # e.g. striptma
op = MassOperator(fs, quad, schedule=sched)
x = torch.from_numpy(x_np).cuda()
y = torch.zeros_like(x)
acc = "overwrite" not in sys.argv
for _ in range(3):
    op.apply(x, coords, y, accumulate=acc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    op.apply(x, coords, y, accumulate=acc)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
op.apply(x, coords, y)          # overwrite: a checksum across builds
torch.cuda.synchronize()
print(sys.argv[2] if len(sys.argv) > 2 else "", sys.argv[1], round(t, 4),
      "ms", "sum %.15e" % float(y.sum()), "l2 %.15e" % float(y.norm()),
      flush=True)
