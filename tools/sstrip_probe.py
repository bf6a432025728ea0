"""Stacked store-first strips probe (experiment; needs a library built with
PM_EXPERIMENTAL=1 for the patch-strip kernel): chains of global strips that
share vertex rows, walked by the patch-strip (stream-mode) kernel.
    PM_NATIVE_LIB=build/var/exp.so python tools/sstrip_probe.py C5a [depth] [maxlen] [reps]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_1604_05937_b200 import _lib, configs
from paper_1604_05937_b200.extrusion import extrude_coordinates
from paper_1604_05937_b200.kernels import MassOperator, strip_chunk_width
from paper_1604_05937_b200.schedule import morton_order


def stack(base, max_len, depth):
    sp, st = _lib.build_global_strips(base, max_len=max_len, order="creation")
    ns = sp.shape[0] - 1
    nv = base.num_vertices
    lens = np.diff(sp).astype(np.int64)
    sid = np.repeat(np.arange(ns, dtype=np.int64), lens)
    u = np.unique(st.astype(np.int64) * ns + sid)
    v, s = u // ns, u % ns
    pa, pb = [], []
    for d in range(1, 8):
        ok = np.flatnonzero(v[d:] == v[:-d])
        if ok.size == 0:
            break
        pa.append(s[ok])
        pb.append(s[ok + d])
    succ = np.full(ns, -1, dtype=np.int64)
    pk, cnt = np.unique(np.concatenate(pa) * ns + np.concatenate(pb),
                        return_counts=True)
    a, b = pk // ns, pk % ns
    o = np.lexsort((b, -cnt, a))
    a, b, cnt = a[o], b[o], cnt[o]
    first = np.flatnonzero(np.r_[True, a[1:] != a[:-1]])
    good = cnt[first] * 8 >= lens[a[first]]
    succ[a[first][good]] = b[first][good]
    group = np.full(ns, -1, dtype=np.int64)
    chains = []
    for s0 in range(ns):
        if group[s0] >= 0:
            continue
        ch = [s0]
        group[s0] = len(chains)
        while len(ch) < depth:
            t = succ[ch[-1]]
            if t < 0 or group[t] >= 0:
                break
            group[t] = len(chains)
            ch.append(int(t))
        chains.append(ch)
    xy = np.asarray(base.coords)[st]
    gsum = np.zeros((len(chains), 2))
    gcnt = np.zeros(len(chains))
    np.add.at(gsum, group[sid], xy)
    np.add.at(gcnt, group[sid], 1)
    gorder = morton_order(gsum / np.maximum(gcnt, 1)[:, None])
    strips = [t for g in gorder for t in chains[g]]
    item_ptr = np.zeros(len(chains) + 1, dtype=np.int64)
    np.cumsum([len(chains[g]) for g in gorder], out=item_ptr[1:])
    strip_ptr = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(lens[strips], out=strip_ptr[1:])
    idx = np.concatenate([np.arange(sp[t], sp[t + 1]) for t in strips])
    steps = st[idx].astype(np.int64)
    gv = group[sid[idx]]
    gmin = np.full(nv, np.iinfo(np.int64).max)
    gmax = np.full(nv, -1)
    np.minimum.at(gmin, steps, gv)
    np.maximum.at(gmax, steps, gv)
    private = gmin == gmax
    _, fst = np.unique(steps, return_index=True)
    flags = np.zeros(steps.shape[0], dtype=np.int64)
    flags[fst[private[steps[fst]]]] |= _lib.STEP_STORE
    flags[strip_ptr[:-1]] |= _lib.STEP_NOCELL
    flags[strip_ptr[:-1] + 1] |= _lib.STEP_NOCELL
    zero = np.flatnonzero(~private).astype(np.int32)
    return (item_ptr.astype(np.int32), strip_ptr.astype(np.int32),
            (steps | flags).astype(np.int32), zero)


name = sys.argv[1]
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 4
max_len = int(sys.argv[3]) if len(sys.argv) > 3 else 128
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
w = configs.workload(name)
fs, quad, x_np, _ = configs.build(w)
m = fs.mesh
coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
op = MassOperator(fs, quad)
plan = tuple(torch.from_numpy(a).cuda() for a in stack(m.base, max_len, depth))
plan = plan[:3] + (None,) + plan[3:]
x = torch.from_numpy(x_np).cuda()
y = torch.zeros_like(x)
W = strip_chunk_width(m.layers)


def run(acc=False):
    _lib.column_mass_patch_strips(fs.layout, op.k, m.layers, coords, op.mref,
                                  x, y, fs.total_dofs, plan, op.kron, W,
                                  accumulate=acc,
                                  n_vertices=m.base.num_vertices)


ref = op.apply(x, coords).clone()
run()
torch.cuda.synchronize()
err = float((y - ref).abs().max() / ref.abs().max())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
print(f"sstrip {name} depth {depth} maxlen {max_len}: "
      f"{e0.elapsed_time(e1) / reps:.4f} ms (overwrite), rel err {err:.2e}",
      flush=True)
