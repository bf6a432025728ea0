"""Quick GPU check of the band-tile schedule: parity against the oracle on
small meshes and against the strip-REDG schedule on C5-size meshes, then
timings (ms per apply, CUDA events, graph of K applies)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1604_05937_b200 import configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator
from paper_1604_05937_b200.perfbench import valuable_volume
from paper_1604_05937_b200.quadrature import element_for_layout

FAM = {"CG1xCG1": ("P1", "P1", 1), "VP1": ("P1", "P1", 3),
       "CG1xDG0": ("P1", "P0", 1), "CG1xDG1": ("P1", "P1", 1)}


def parity(n, layers, layout, ordering="rcm", quad=(2, 2)):
    w = configs.Workload("t", n, layers, layout, quad, ordering)
    fs, q, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    op = MassOperator(fs, q)
    xd = torch.from_numpy(x).cuda()
    y = torch.full_like(xd, float("nan"))
    op.apply(xd, coords, y, schedule="tile")
    y2 = op.apply(xd, coords, schedule="tile")   # second launch: epoch path
    el = element_for_layout(fs.layout)
    prob = oracle.Problem(m.base, m.layers, fs.layout.counts, el.tri, el.line,
                          el.ncomp, *quad)
    ref = prob.assemble(x) if n <= 64 else prob.assemble_colored(x)
    yh, y2h = y.cpu().numpy(), y2.cpu().numpy()
    err = np.abs(yh - ref).max() / np.abs(ref).max()
    err2 = np.abs(y2h - ref).max() / np.abs(ref).max()
    print(f"parity {layout:8s} n={n:4d} L={layers:3d} {ordering}: rel err "
          f"{err:.2e} / {err2:.2e}  tiles {op._tiles['n_tiles']} smem "
          f"{op._tiles['smem']}", flush=True)
    assert err < 1e-10 and err2 < 1e-10


def timing(name, schedules, reps=10):
    w = configs.workload(name)
    fs, q, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    op = MassOperator(fs, q)
    xd = torch.from_numpy(x).cuda()
    V = valuable_volume(fs)
    ys = {}
    for s in schedules:
        t0 = time.perf_counter()
        y = op.apply(xd, coords, schedule=s)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        g = op.graph(xd, coords, y, schedule=s, repeat=reps)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        best = 1e9
        for _ in range(3):
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps)
        ys[s] = y.clone()
        print(f"{name} {s:9s}: {best:.4f} ms/apply = {V / best / 1e6:.0f} GB/s "
              f"({100 * V / best / 1e6 / 6441.6:.1f} % of measured HBM); "
              f"first call {setup:.2f} s", flush=True)
    base = ys[schedules[0]]
    for s in schedules[1:]:
        err = (ys[s] - base).abs().max().item() / base.abs().max().item()
        print(f"  {s} vs {schedules[0]}: rel diff {err:.2e}")


if __name__ == "__main__":
    what = sys.argv[1:] or ["parity", "C5a", "C5b"]
    if "parity" in what:
        for layout in ("CG1xCG1", "VP1", "CG1xDG0", "CG1xDG1"):
            for n, L in ((8, 3), (16, 10), (24, 33), (32, 64)):
                parity(n, L, layout)
        parity(32, 20, "CG1xCG1", "random")
        parity(256, 50, "CG1xCG1")
        parity(256, 20, "VP1")
    scheds = os.environ.get("PM_SCHEDS", "stripred,tile").split(",")
    for name in what:
        if name.startswith("C"):
            timing(name, scheds)
