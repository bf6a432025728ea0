"""Patch-owner schedule for CG column loops (host planner).

Shared (vertex / edge) DoFs are the reason the reference's coloured
schedule exists.  On the GPU the race-free alternative
used here is *owner computes*:

1. cells are cut into compact patches (Morton / Z order of the cell
   centroids, ``target`` cells each);
2. every DoF-carrying base entity is owned by the lowest-numbered patch
   touching it;
3. patch p visits every cell incident to one of its entities (its own
   cells plus a halo ring), accumulates the cell-layer contributions of a
   W-layer chunk in shared memory (cells grouped by the global greedy
   colouring, so one colour never writes an accumulator twice), and then
   writes its owned entity columns with plain, coalesced stores.

Every DoF is written exactly once, by one CTA, in a fixed order: the
result is bitwise deterministic and needs no zeroing and no atomics.  The
price is the recomputed halo cells (reported as ``redundancy``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class PatchPlan:
    n_patches: int
    n_colors: int
    ent_positions: int          # 3 (vertices) or 6 (vertices + edges)
    cell_ptr: np.ndarray        # int32 [n_patches+1] into `cells`
    cells: np.ndarray           # int32 global cell ids, by colour per patch
    color_ptr: np.ndarray       # int32 [n_patches, n_colors+1] (absolute)
    ent_ptr: np.ndarray         # int32 [n_patches+1] into `ents`
    owned: np.ndarray           # int32 [n_patches] owned entities (first)
    ents: np.ndarray            # int32 entity codes: v, or n_vertices + e
    lents: np.ndarray           # uint16 [len(cells), ent_positions]
    max_local: int              # max entities of one patch
    max_owned: int
    redundancy: float           # cell-visits / cells

    def device(self, dev):
        import torch
        return {k: torch.from_numpy(np.ascontiguousarray(getattr(self, k)))
                .to(dev) for k in ("cell_ptr", "cells", "color_ptr",
                                   "ent_ptr", "owned", "ents", "lents")}


def morton_order(points):
    """Argsort of 2-D points along the Z curve (16 bits per axis)."""
    lo = points.min(axis=0)
    span = max(float((points.max(axis=0) - lo).max()), 1e-300)
    q = np.floor((points - lo) / span * 65535.0).astype(np.uint64)

    def spread(v):
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
    return np.argsort(code, kind="stable")


def build_patch_plan(base, with_edges: bool, target: int,
                     colors: np.ndarray, n_colors: int) -> PatchPlan:
    cv = np.asarray(base.cell_vertices, dtype=np.int64)
    n_cells = cv.shape[0]
    n0 = base.num_vertices
    if with_edges:
        ce = np.asarray(base.cell_edges, dtype=np.int64)
        ents = np.concatenate([cv, n0 + ce], axis=1)
        n_ent = n0 + base.num_edges
    else:
        ents = cv
        n_ent = n0
    E = ents.shape[1]

    coords = np.asarray(base.coords)
    cent = coords[cv].mean(axis=1)
    order = morton_order(cent)
    patch_of = np.empty(n_cells, dtype=np.int64)
    patch_of[order] = np.arange(n_cells) // target
    n_p = int(patch_of.max()) + 1 if n_cells else 0

    flat_e = ents.ravel()
    flat_c = np.repeat(np.arange(n_cells, dtype=np.int64), E)
    owner = np.full(n_ent, n_p, dtype=np.int64)
    np.minimum.at(owner, flat_e, patch_of[flat_c])

    # (patch, cell) visits: every cell incident to an owned entity
    pk = np.unique(owner[flat_e] * n_cells + flat_c)
    vp, vc = pk // n_cells, pk % n_cells
    col = np.asarray(colors, dtype=np.int64)[vc]
    o2 = np.lexsort((vc, col, vp))
    vp, vc, col = vp[o2], vc[o2], col[o2]
    cell_ptr = np.zeros(n_p + 1, dtype=np.int64)
    np.cumsum(np.bincount(vp, minlength=n_p), out=cell_ptr[1:])
    cc = np.bincount(vp * n_colors + col, minlength=n_p * n_colors)
    color_ptr = np.zeros((n_p, n_colors + 1), dtype=np.int64)
    np.cumsum(cc.reshape(n_p, n_colors), axis=1, out=color_ptr[:, 1:])
    color_ptr += cell_ptr[:-1, None]

    # local entities per patch: owned first (ascending), then halo
    pe_p = np.repeat(vp, E)
    pe_e = ents[vc].ravel()
    halo = (owner[pe_e] != pe_p).astype(np.int64)
    key = (pe_p * 2 + halo) * n_ent + pe_e
    ukey, inv = np.unique(key, return_inverse=True)
    up = ukey // (2 * n_ent)
    uhalo = (ukey // n_ent) % 2
    ue = ukey % n_ent
    ent_ptr = np.zeros(n_p + 1, dtype=np.int64)
    np.cumsum(np.bincount(up, minlength=n_p), out=ent_ptr[1:])
    owned = np.bincount(up[uhalo == 0], minlength=n_p)
    local = np.arange(ukey.shape[0]) - ent_ptr[up]
    lents = local[inv].reshape(-1, E)
    max_local = int(np.diff(ent_ptr).max()) if n_p else 0
    if max_local >= 65536:
        raise ValueError("patch too large for 16-bit local entity ids")
    return PatchPlan(
        n_patches=n_p, n_colors=n_colors, ent_positions=E,
        cell_ptr=cell_ptr.astype(np.int32), cells=vc.astype(np.int32),
        color_ptr=color_ptr.astype(np.int32), ent_ptr=ent_ptr.astype(np.int32),
        owned=owned.astype(np.int32), ents=ue.astype(np.int32),
        lents=lents.astype(np.uint16), max_local=max_local,
        max_owned=int(owned.max()) if n_p else 0,
        redundancy=float(vc.shape[0]) / max(n_cells, 1))


def smem_bytes(max_local, max_owned, channels, W):
    """Accumulator A[local][ch][W+1] + carry[owned][ch] (doubles)."""
    return 8 * (max_local * channels * (W + 1) + max_owned * channels)


def plan_for(base, layout, layers, colors, n_colors, smem_budget=100 * 1024,
             W=None, n_sm=148):
    """Pick the chunk width W and the patch size for a layout and build the
    plan: the largest patch whose accumulator fits ``smem_budget``, capped
    so that there are at least ~2 patches per SM."""
    d = layout.delta6()
    with_edges = bool(d[2] or d[3])
    ch = max(int(d[0] + d[1]), int(d[2] + d[3]))
    # local entities per visited cell: ~0.6 (vertices) / ~2.2 (+ edges)
    per_cell = 2.2 if with_edges else 0.62
    n_cells = base.num_cells
    cap = max(16, n_cells // (2 * n_sm))

    def target_for(w):
        t = int(smem_budget / (8 * ch * (w + 1) * per_cell))
        return max(16, min(t, 4096, cap))

    def cost(w):
        chunks = -(-layers // w)
        lanes = chunks * w / layers
        redundancy = 1.0 + 3.8 / np.sqrt(target_for(w))
        return redundancy * lanes * (1.0 + 0.04 * chunks)

    if W is None:
        W = min((8, 16, 32), key=cost)
    target = target_for(W)
    for _ in range(8):
        plan = build_patch_plan(base, with_edges, target, colors, n_colors)
        need = smem_bytes(plan.max_local, plan.max_owned, ch, W)
        if need <= smem_budget or target <= 16:
            return plan, W, ch, need
        target = max(16, int(target * smem_budget / need * 0.95))
    return plan, W, ch, need


# ---------------------------------------------------------------------------
# strip-patch schedule (csrc/strip.cu): vertex-column layouts
# ---------------------------------------------------------------------------
@dataclass
class StripPlan:
    patch: PatchPlan
    W: int
    threads: int
    strip_ptr: np.ndarray      # int32 [n_patches+1] into strip_step_ptr
    step_ptr: np.ndarray       # int32 [n_strips+1] into steps
    step_v: np.ndarray         # uint16 local vertex entering the window
    step_slot: np.ndarray      # uint8 window slot it replaces
    step_flags: np.ndarray     # uint8 bit0: apply the cell kernel
    step_y: np.ndarray         # int32 Y slot of the new residency or -1
    y_count: np.ndarray        # int32 [n_patches]
    own_base: np.ndarray       # int32 [n_patches] prefix of owned counts
    own_y_ptr: np.ndarray      # int32 [total_owned+1]
    own_y: np.ndarray          # int32
    max_y: int
    smem: int
    max_steps: int = 0
    max_strips: int = 0
    max_oy: int = 0

    def device(self, dev):
        import torch
        d = self.patch.device(dev)
        for k in ("strip_ptr", "step_ptr", "step_v", "step_slot",
                  "step_flags", "step_y", "y_count", "own_base", "own_y_ptr",
                  "own_y"):
            d[k] = torch.from_numpy(np.ascontiguousarray(getattr(self, k))) \
                .to(dev)
        return d


def strip_smem(max_local, max_y, max_owned, ch, lv, W, max_steps=0,
               max_strips=0, max_oy=0):
    return (8 * (max_local * (W * ch + lv + 3 * (W + 1)) +
                 max_y * ch * (W + 1) + max_owned * max(lv, 1)) +
            8 * max_steps + 4 * (max_strips + 1 + max_owned + 1 + max_oy +
                                 max_local))


def build_strip_plan(base, layout, layers, colors, n_colors,
                     smem_budget=110 * 1024, W=None, n_sm=148,
                     max_strip=None):
    """Patch plan (vertex entities) + strips, sized to the smem budget."""
    import ctypes
    from . import _lib
    d = layout.delta6()
    if d[2] or d[3] or d[4] or d[5]:
        raise ValueError("the strip schedule handles vertex-column layouts")
    lv, ch = int(d[0]), int(d[0] + d[1])
    threads = 256
    if ch > 2:                 # one CTA per SM (register-bound window)
        smem_budget = max(smem_budget, 200 * 1024)
    if W is None:
        W = min((8, 16, 32), key=lambda w: (-(-layers // w) * w / layers
                                             + 0.05 * (-(-layers // w)), -w))
    n_cells = base.num_cells
    cap = max(16, n_cells // (2 * n_sm))
    # bytes per visited cell: ~0.62 local vertices, ~1.1 Y residencies
    per_cell = 8 * (0.62 * (W * ch + lv + 3 * (W + 1)) + 1.1 * ch * (W + 1))
    target = max(16, min(int(smem_budget / per_cell), cap, 4096))
    for _ in range(10):
        plan = build_patch_plan(base, False, target, colors, n_colors)
        n_visit = plan.cells.shape[0]
        n_p = plan.n_patches
        strip_ptr = np.zeros(n_p + 1, np.int32)
        step_ptr = np.zeros(n_visit + 1, np.int32)
        cap_steps = 3 * n_visit
        step_v = np.zeros(cap_steps, np.uint16)
        step_slot = np.zeros(cap_steps, np.uint8)
        step_flags = np.zeros(cap_steps, np.uint8)
        step_y = np.zeros(cap_steps, np.int32)
        y_count = np.zeros(n_p, np.int32)
        own_total = int(plan.owned.sum())
        own_y_ptr = np.zeros(own_total + 1, np.int32)
        own_y = np.zeros(cap_steps, np.int32)
        totals = np.zeros(3, np.int64)
        ce = np.ascontiguousarray(base.cell_edges, dtype=np.int32)
        mlen = max_strip or 24
        P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
        i32, u16, u8, i64 = (ctypes.c_int32, ctypes.c_uint16, ctypes.c_uint8,
                             ctypes.c_int64)
        _lib.check(_lib.host_lib().pm_build_strips(
            n_p, P(plan.cell_ptr, i32), P(plan.cells, i32), P(ce, i32),
            P(np.ascontiguousarray(plan.lents), u16), P(plan.owned, i32),
            P(plan.ent_ptr, i32), mlen, P(strip_ptr, i32), P(step_ptr, i32),
            P(step_v, u16), P(step_slot, u8), P(step_flags, u8),
            P(step_y, i32), P(y_count, i32), P(own_y_ptr, i32),
            P(own_y, i32), P(totals, i64)))
        n_strips, n_steps, n_oy = (int(v) for v in totals)
        own_base = np.zeros(n_p, np.int32)
        np.cumsum(plan.owned[:-1], out=own_base[1:])
        max_y = int(y_count.max()) if n_p else 0
        steps_pp = step_ptr[strip_ptr[1:]] - step_ptr[strip_ptr[:-1]]
        max_steps = int(steps_pp.max()) if n_p else 0
        max_strips = int(np.diff(strip_ptr).max()) if n_p else 0
        oy_pp = own_y_ptr[own_base + plan.owned] - own_y_ptr[own_base]
        max_oy = int(oy_pp.max()) if n_p else 0
        need = strip_smem(plan.max_local, max_y, plan.max_owned, ch, lv, W,
                          max_steps, max_strips, max_oy)
        if need <= smem_budget or target <= 16:
            break
        target = max(16, int(target * smem_budget / need * 0.95))
    return StripPlan(plan, W, threads, strip_ptr, step_ptr[:n_strips + 1],
                     step_v[:n_steps], step_slot[:n_steps],
                     step_flags[:n_steps], step_y[:n_steps], y_count,
                     own_base, own_y_ptr, own_y[:n_oy], max_y, need,
                     max_steps, max_strips, max_oy)
