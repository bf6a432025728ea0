"""A/B of MassOperator schedules on one workload (overwrite mode, CUDA
events, 10 applies after 3 warm-up), with the max relative difference of
each schedule's result against the first one.

    python tools/ab_sched.py C3 stripred pstrip
"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_1604_05937_b200 import configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator

w = configs.workload(sys.argv[1])
fs, quad, x_np, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
x = torch.from_numpy(x_np).cuda()
ref = None
for sched in sys.argv[2:]:
    op = MassOperator(fs, quad, schedule=sched)
    y = torch.zeros_like(x)
    t0 = time.perf_counter()
    op.apply(x, coords, y)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for _ in range(3):
        op.apply(x, coords, y)
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    for _ in range(10):
        op.apply(x, coords, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if ref is None:
        ref, diff = y.clone(), 0.0
    else:
        diff = float((y - ref).abs().max() / ref.abs().max())
    from paper_1604_05937_b200.perfbench import valuable_volume
    gbs = valuable_volume(fs) / (ms * 1e-3) / 1e9
    print(f"{w.name} {sched:10s} {ms:8.4f} ms  {gbs:7.1f} GB/s  "
          f"rel diff {diff:.2e}  first call {setup:.2f} s", flush=True)
    del op

# accumulate-mode timing of the last schedule (every residency adds; y
# zeroed by a memset outside the timed op)
if os.environ.get("AB_ACC"):
    op = MassOperator(fs, quad, schedule=sys.argv[-1])
    y = torch.zeros_like(x)
    for _ in range(3):
        op.apply(x, coords, y, accumulate=True)
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    for _ in range(10):
        y.zero_()
        op.apply(x, coords, y, accumulate=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{w.name} {sys.argv[-1]} memset+accumulate "
          f"{e0.elapsed_time(e1) / 10:8.4f} ms")
