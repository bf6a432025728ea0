"""Per-round timeline of the tile kernel from a PM_TILE_TRACE build:
PM_NATIVE_LIB=build/var/trace.so python tools/tile_trace.py C5a"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1604_05937_b200 import _lib, configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator

name = sys.argv[1] if len(sys.argv) > 1 else "C5a"
w = configs.workload(name)
fs, q, x, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
op = MassOperator(fs, q)
xd = torch.from_numpy(x).cuda()
y = torch.empty_like(xd)
for _ in range(2):
    op.apply(xd, coords, y, schedule="tile")
torch.cuda.synchronize()
L = _lib.host_lib()
L.pm_tile_trace.restype = ctypes.c_int
ns = 8
buf = np.zeros(8 * (ns + 2) * 256 * 4, dtype=np.uint64)
ns = L.pm_tile_trace(buf.ctypes.data_as(ctypes.c_void_p))
assert ns > 0
tr = buf[:8 * (ns + 2) * 256 * 4].reshape(8, ns + 2, 256, 4).astype(np.int64)
pl = op._tiles
print("tiles", pl["n_tiles"], "data_bytes", pl["data_bytes"], "stages", ns)
for cta in (0, 3):
    sys.stdout.flush()
    t0 = tr[cta][tr[cta] > 0].min()
    print(f"CTA {cta}: producer rounds (us): start, empty-wait, issue, prefetch")
    for b in range(ns):
        p = tr[cta, b]
        ok = (p[:, 3] > 0)
        r = np.nonzero(ok)[0][5:60]
        if len(r) == 0:
            continue
        ew = (p[r, 1] - p[r, 0]) / 1e3
        iss = (p[r, 2] - p[r, 1]) / 1e3
        pf = (p[r, 3] - p[r, 2]) / 1e3
        per = np.diff(p[r, 0]) / 1e3
        print(f"  stage {b}: round period {np.median(per):6.2f}  empty-wait "
              f"{np.median(ew):6.2f}  issue {np.median(iss):6.2f}  prefetch "
              f"{np.median(pf):6.2f}")
    c = tr[cta, ns]
    ok = c[:, 2] > 0
    i = np.nonzero(ok)[0][5:200]
    fw = (c[i, 1] - c[i, 0]) / 1e3
    wk = (c[i, 2] - c[i, 1]) / 1e3
    per = np.diff(c[i, 0]) / 1e3
    print(f"  consumer warp 0: per tile {np.median(per):6.2f} us, full-wait "
          f"{np.median(fw):6.2f} (mean {fw.mean():6.2f}), walk "
          f"{np.median(wk):6.2f} (mean {wk.mean():6.2f})")
    z = tr[cta, ns + 1]
    j = np.nonzero(z[:, 3] > 0)[0][3:60]
    if len(j):
        print(f"  zero warp per batch: period {np.median(np.diff(z[j, 0])) / 1e3:6.2f}"
              f" throttle {np.median(z[j, 1] - z[j, 0]) / 1e3:6.2f} stores "
              f"{np.median(z[j, 2] - z[j, 1]) / 1e3:6.2f} fence "
              f"{np.median(z[j, 3] - z[j, 2]) / 1e3:6.2f}")
    print("  first 12 consumer stamps (us from start):",
          np.round((c[:12, 0] - t0) / 1e3, 1).tolist())
