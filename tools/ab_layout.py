"""A/B of schedules for any layout on the split-square RCM mesh:
    python tools/ab_layout.py LAYOUT N LAYERS sched1 sched2 ...
(CUDA events, 10 overwrite applies after 3 warm-up, valuable GB/s)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1604_05937_b200 import configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator
from paper_1604_05937_b200.perfbench import valuable_volume

lname, n, layers = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
quad = {"P2xP2": (6, 6)}.get(lname, (2, 2))
w = configs.Workload("ab", n, layers, lname, quad,
                     ordering=os.environ.get("AB_ORDERING", "rcm"))
fs, q, x_np, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
x = torch.from_numpy(x_np).cuda()
ref = None
for sched in sys.argv[4:]:
    op = MassOperator(fs, q, schedule=sched)
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply(x, coords, y)
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    for _ in range(10):
        op.apply(x, coords, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    diff = 0.0 if ref is None else float((y - ref).abs().max() / ref.abs().max())
    if ref is None:
        ref = y.clone()
    print(f"{lname} n={n} L={layers} {sched:8s} {ms:8.4f} ms "
          f"{valuable_volume(fs) / (ms * 1e-3) / 1e9:8.1f} GB/s "
          f"rel diff {diff:.1e}", flush=True)
