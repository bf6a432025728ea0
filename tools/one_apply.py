"""One workload, one schedule, a few applies (for ncu captures):
one_apply.py C5a tile [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1604_05937_b200 import configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator

name, sched = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = configs.workload(name)
fs, q, x, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
op = MassOperator(fs, q)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
for _ in range(reps):
    op.apply(xd, coords, y, schedule=sched)
torch.cuda.synchronize()
print("ok", name, sched, float(y.sum()))
