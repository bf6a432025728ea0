"""Element kernels on triangle x interval prisms, executed on the GPU.

Drop-in for the SPEC's ``kernels`` module:

* ``prism_quadrature(tri_degree, line_degree)``   (``quadrature.py``)
* ``assemble_residual(fs, f, coords)``  -- ``b_j = int f v_j dx`` with ``f``
  in ``fs``: the mass-matrix action ``b = M f`` (SPEC.md:412-420,
  PAPER.md:629-642 integral I_1)
* ``count_flops(layout, quadrature)``   -- analytic profile

plus the device operator ``MassOperator`` (prepared maps, reusable) that
the benchmark and the sharded driver call, and the probe kernels used to
check the par-loop's addressing.

Fields are flat float64 arrays in the space's global numbering.  Numpy in
-> numpy out (host<->device copies happen inside the call); CUDA tensor in
-> CUDA tensor out.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .fspace import COORDS_LAYOUT, FunctionSpace, number_dofs
from .quadrature import (PrismElement, QuadratureRule, element_for_layout,
                         kronecker_factors, prism_quadrature,
                         reference_mass_matrix, sharing_class)

__all__ = ["Field", "KernelProfile", "MassKernel", "MassOperator",
           "CountingKernel", "ListProbeKernel", "assemble_residual",
           "mass_action", "count_flops", "prism_quadrature",
           "default_quadrature"]


@dataclass
class Field:
    """Values of one function space."""

    space: FunctionSpace
    values: object

    def __post_init__(self):
        if len(self.values) != self.space.total_dofs:
            raise ValueError(
                f"field has {len(self.values)} values, space has "
                f"{self.space.total_dofs}")


@dataclass(frozen=True)
class KernelProfile:
    adds: int
    muls: int
    fmas: int
    vector_flops: int

    @property
    def total_flops(self) -> int:
        return self.adds + self.muls + 2 * self.fmas


def count_flops(layout, quadrature: QuadratureRule) -> KernelProfile:
    """Per cell-layer: per point k muls + (k-1) adds (f . phi), 1 mul
    (w|detJ|), k muls + k adds (scatter) -- SPEC.md:425."""
    from .fspace import slot_table
    k = len(slot_table(layout))
    q = quadrature.num_points
    return KernelProfile(adds=q * (2 * k - 1), muls=q * (2 * k + 1), fmas=0,
                         vector_flops=0)


def default_quadrature(element: PrismElement) -> QuadratureRule:
    """SPEC default (2,2), raised to the exact degree for P2 elements."""
    deg = {"P0": 0, "P1": 1, "P2": 2}
    return prism_quadrature(max(2, 2 * deg[element.tri]),
                            max(2, 2 * deg[element.line]))


def tri_permutation_invariant(mtri) -> bool:
    """``Mtri[p(i), p(j)] == Mtri[i, j]`` for every permutation p of the
    three vertices (edges, NH = 6, follow: edge e is opposite vertex e)."""
    from itertools import permutations
    mtri = np.asarray(mtri)
    nh = mtri.shape[0]
    tol = 1e-14 * max(float(np.abs(mtri).max()), 1e-300)
    for p in permutations(range(3)):
        idx = list(p) + ([3 + q for q in p] if nh == 6 else [])
        if nh not in (3, 6):
            return False
        if np.abs(mtri[np.ix_(idx, idx)] - mtri).max() > tol:
            return False
    return True


def kron_reproduces(element: PrismElement, kron, mref) -> bool:
    """``Mref[j,j'] == δ(comp) Mtri[h,h'] Mline[v,v']`` to round-off?"""
    if kron is None:
        return False
    mtri, mline = kron
    h = np.asarray(element.slot_h)
    v = np.asarray(element.slot_v)
    c = np.asarray(element.slot_comp)
    rebuilt = (mtri[h[:, None], h[None, :]] * mline[v[:, None], v[None, :]] *
               (c[:, None] == c[None, :]))
    scale = max(float(np.abs(mref).max()), 1e-300)
    return bool(np.abs(rebuilt - mref).max() <= 1e-13 * scale)


def _as_device(a, dev):
    import torch
    if isinstance(a, Field):
        a = a.values
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64:
            raise ValueError(f"fields are float64, got {a.dtype}")
        if a.device.type != "cuda":
            return a.to(dev, non_blocking=a.is_pinned()), True
        return a.contiguous(), False
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return torch.from_numpy(arr).to(dev, non_blocking=False), True


class MassOperator:
    """``y = |det J| M_ref x`` over every cell-layer of ``fs`` (device).

    Holds the device-resident bottom-layer maps (K0), the coordinate
    space's maps and the pre-integrated reference matrix.
    """

    def __init__(self, fs: FunctionSpace, quadrature: QuadratureRule = None,
                 element: PrismElement = None, schedule: str = "auto"):
        if not fs.fits_int32:
            raise ValueError(
                f"{fs!r}: {fs.total_dofs} DoFs overflow the int32 cell map")
        self.fs = fs
        self.coord_fs = number_dofs(fs.mesh, COORDS_LAYOUT)
        self.element = element or element_for_layout(fs.layout)
        self.quadrature = quadrature or default_quadrature(self.element)
        self.mref = reference_mass_matrix(self.element, self.quadrature)
        self.kron = kronecker_factors(self.element, self.quadrature)
        # the compiled column / patch kernels assume the layout's default
        # element (their slot -> basis map is a compile-time table)
        default = element_for_layout(fs.layout) if element is not None \
            else self.element
        # ... and factors whose tensor product is Mref (a rule that is not
        # the tensor rule of its degrees would get the dense generic kernel)
        self.kron_ok = default == self.element and \
            kron_reproduces(self.element, self.kron, self.mref)
        self.share = sharing_class(fs.layout)
        self.k = fs.num_slots
        self.schedule = schedule
        self._coloring = None
        self._patch = None
        self._strip = None
        self._gstrips = None
        self._rstrips = None
        self._tma_auto = None
        self._dgstrips = None
        self._pstrips = None
        self._tiles = None
        self._tile_tmp = None
        self._strip_inv = None
        self._hbuf = None
        self.last_schedule = None   # the schedule the last apply resolved
        self._dev = _lib.cuda_device()
        self.cmap = fs.device_cell_map()
        self.offs = fs.device_offsets()
        if self.dg_only:
            # the DG stream kernel addresses the field densely (cell, layer,
            # slot), which is what Alg. 1 gives cell-only layouts
            # (fspace.py:134-149); a space numbered otherwise must not
            # reach it (include/prismesh_cuda.h, PM_VARIANT_STREAM)
            cm = np.asarray(fs.cell_map, dtype=np.int64)
            k, L = cm.shape[1], fs.mesh.layers
            dense = (np.array_equal(np.asarray(fs.offsets), np.full(k, k)) and
                     np.array_equal(cm, (np.arange(cm.shape[0])[:, None] * k * L
                                         + np.arange(k)[None, :])))
            if not dense:
                raise ValueError("cell-only layout with a non-Alg. 1 cell map")
        self.xmap = self.coord_fs.device_cell_map()
        self.xoffs = self.coord_fs.device_offsets()

    @property
    def launches_per_apply(self) -> int:
        """Column-loop kernel launches one ``apply`` issues."""
        if self.schedule in ("colored", "sequential") and self.share == 2:
            return self._color_lists()[1].shape[0] - 1
        d = self.fs.layout.delta6()
        if self.stripdg_ok and d[4] and self.schedule in ("auto", "stripdg") \
                and self.layers > strip_chunk_width(self.layers):
            return 2    # chunk-boundary level zeroing + the strip kernel
        if self.schedule in ("auto", "patch", "stripred", "strip",
                             "pstrip") and \
                self.share == 2:
            return 1
        return 1

    @property
    def n_cells(self):
        return self.fs.mesh.base.num_cells

    @property
    def layers(self):
        return self.fs.mesh.layers

    @property
    def patch_ok(self) -> bool:
        """DoFs only on vertex / edge columns (the patch schedule's case)."""
        d = self.fs.layout.delta6()
        return d[4] == 0 and d[5] == 0 and tuple(d) in _PATCH_LAYOUTS

    @property
    def strip_ok(self) -> bool:
        d = tuple(self.fs.layout.delta6())
        return d in _STRIP_LAYOUTS and self.strip_invariant

    @property
    def stripred_ok(self) -> bool:
        d = tuple(self.fs.layout.delta6())
        return d in _STRIPRED_LAYOUTS and self.strip_invariant

    @property
    def strip_invariant(self) -> bool:
        """The strip kernels place a cell's vertices by window slot, not by
        the cell's local vertex order: valid when the triangle factor is
        invariant under the vertex permutations (every symmetric rule).
        Evaluated once per operator (apply() is on the timed path)."""
        if self._strip_inv is None:
            self._strip_inv = bool(self.kron_ok and
                                   tri_permutation_invariant(self.kron[0]))
        return self._strip_inv

    @property
    def tile_ok(self) -> bool:
        """Layouts of the band-tile kernel (csrc/tile.cu): vertex columns
        only, vertex-permutation invariant triangle factor."""
        d = tuple(self.fs.layout.delta6())
        return d in _STRIP_LAYOUTS and self.strip_invariant

    def _tile_plan(self):
        """Band tiles (cached): host plan (pm_tiles_build), its per-tile
        records on the device and the plan's ticket / epoch words."""
        if self._tiles is None:
            import os
            import torch
            L = self.layers
            d = self.fs.layout.delta6()
            colf = 8 * (int(d[0]) * (L + 1) + int(d[1]) * L)
            colc = 24 * (L + 1)
            W = strip_chunk_width(L)
            # one CTA of PM_TILE_THREADS threads per SM (228 KB of shared
            # memory, 1 KB reserved), `stages` tile buffers in it;
            # PM_TILE_BUDGET overrides the bytes per buffer
            cap = 233472 - 1024
            off, stages, threads = _lib.tile_smem_layout(self.fs.layout,
                                                         1024, 128, W)
            budget = int(os.environ.get("PM_TILE_BUDGET", "0")) or \
                (cap - off) // stages - 256
            nchunks = -(-L // W)
            # walking warps take items from several staged tiles at once:
            # no strip splitting needed for parallelism
            min_strips = int(os.environ.get("PM_TILE_MIN_STRIPS", "1"))
            while True:
                plan = _lib.build_tiles(self.fs.mesh.base, colf, colc, budget,
                                        max_cells=256, min_strips=min_strips)
                area_c = (plan["max_fa"] + 127) // 128 * 128
                data = (area_c + plan["max_ca"] + 127) // 128 * 128
                off, stages, _ = _lib.tile_smem_layout(
                    self.fs.layout, plan["max_words"], plan["max_slots"], W)
                if off + stages * data <= cap or \
                        budget < 3 * (colf + colc + 32) + 4096:
                    break
                budget -= (off + stages * data - cap) // stages + 256
            dev = {k: torch.from_numpy(np.resize(plan[k], max(1, plan[k].size))
                                       ).to(self._dev)
                   for k in ("blob", "off", "zero_ptr", "zero_v0", "zero_n")}
            dev.update({
                   "ctl": torch.tensor([0, 0, 1, 0], dtype=torch.int32,
                                       device=self._dev),
                   "flags": torch.zeros(max(1, plan["n_tiles"]),
                                        dtype=torch.int32, device=self._dev)})
            dev.update(n_tiles=plan["n_tiles"], area_c=area_c,
                       data_bytes=data, max_slots=plan["max_slots"],
                       max_words=plan["max_words"],
                       max_cells=plan["max_cells"], width=W, budget=budget,
                       smem=off + stages * data, stages=stages)
            self._tiles = dev
        return self._tiles

    @property
    def dg_only(self) -> bool:
        d = self.fs.layout.delta6()
        return not (d[0] or d[1] or d[2] or d[3] or d[4])

    def apply_host(self, x_host, coords, y_host, chunks=None):
        """``y_host = M x_host`` for pinned host tensors, with the copies
        pipelined against the compute: for DG (2,1) fields the cell columns
        are contiguous, so chunk j+1 goes up, chunk j is computed and chunk
        j-1 comes down at the same time (three streams).  Other layouts:
        one copy each way around the device call."""
        import torch
        n = self.fs.total_dofs
        if self._hbuf is None:
            self._hbuf = (torch.empty(n, dtype=torch.float64, device=self._dev),
                          torch.empty(n, dtype=torch.float64, device=self._dev),
                          torch.cuda.Stream(self._dev),
                          torch.cuda.Stream(self._dev),
                          torch.cuda.Stream(self._dev))
        xd, yd, s_up, s_cmp, s_down = self._hbuf
        cur = torch.cuda.current_stream()
        pinned = x_host.is_pinned() and y_host.is_pinned()
        if pinned and self.stripred_ok and self._bands() is not None:
            return self._apply_host_bands(x_host, coords, y_host)
        if not (self.dg_only and self.kron_ok and pinned):
            xd.copy_(x_host, non_blocking=True)
            self.apply(xd, coords, yd)
            y_host.copy_(yd, non_blocking=True)
            cur.synchronize()
            return y_host
        L, nc = self.layers, self.n_cells
        if chunks is None:  # ~16 MB per chunk: pipeline fill/drain ~1/chunks
            import os
            mb = float(os.environ.get("PM_HOST_CHUNK_MB", "16"))
            chunks = int(min(64, max(4, n * 8 / (mb * 2**20))))
        # chunk boundaries on whole DG stream units (256 cell-layers)
        q = 256 // np.gcd(256, L)
        per = max(q, -(-nc // chunks // q) * q)
        bounds = list(range(0, nc, per)) + [nc]
        dpl = self.k * L                       # DoFs per cell column
        for s_ in (s_up, s_cmp, s_down):
            s_.wait_stream(cur)
        for c0, c1 in zip(bounds[:-1], bounds[1:]):
            r = slice(c0 * dpl, c1 * dpl)
            with torch.cuda.stream(s_up):
                xd[r].copy_(x_host[r], non_blocking=True)
            s_cmp.wait_stream(s_up)
            _lib.column_mass_dg_range(self.fs.layout, self.k, c0, c1, L,
                                      self.cmap, self.offs, self.xmap,
                                      self.xoffs, coords, self.mref, xd, yd,
                                      stream=s_cmp)
            s_down.wait_stream(s_cmp)
            with torch.cuda.stream(s_down):
                y_host[r].copy_(yd[r], non_blocking=True)
        cur.wait_stream(s_down)
        cur.synchronize()
        return y_host

    def _bands(self):
        """Chunking of the host-buffer path for vertex / edge column layouts
        (cached): cells in index order are cut into chunks; chunk j needs
        the entity columns below up[j] and completes those below done[j],
        per family (vertices; edges, numbered by their sorted vertex pair,
        mesh.py:33-84) -- the cells are sorted by their lowest vertex, as
        apply_ordering leaves them (ordering.py:147-152).  None otherwise.
        """
        if getattr(self, "_band_plan", 0) == 0:
            self._band_plan = None
            import os
            base = self.fs.mesh.base
            d6 = self.fs.layout.delta6()
            cv = np.asarray(base.cell_vertices)
            vmin = cv.min(axis=1)
            if base.num_cells == 0 or d6[4] or d6[5] or \
                    np.any(np.diff(vmin) < 0):
                return None
            n2, n0 = base.num_cells, base.num_vertices
            mb = float(os.environ.get("PM_HOST_CHUNK_MB", "64"))
            nch = int(min(256, max(2, self.fs.total_dofs * 8 / (mb * 2**20))))
            cb = np.unique(np.linspace(0, n2, nch + 1).astype(np.int64))
            fams = []   # (origin, column, up[j], done[j]) per family
            vmax = np.maximum.accumulate(cv.max(axis=1))
            fams.append((0, [int(vmax[c - 1]) + 1 for c in cb[1:]],
                         [int(vmin[c]) if c < n2 else n0 for c in cb[1:]]))
            if d6[2] or d6[3]:
                ce = np.asarray(base.cell_edges)
                emax = np.maximum.accumulate(ce.max(axis=1))
                e_lo = np.asarray(base.edge_vertices)[:, 0]
                fams.append((1, [int(emax[c - 1]) + 1 for c in cb[1:]],
                             [int(np.searchsorted(e_lo, vmin[c]))
                              if c < n2 else base.num_edges
                              for c in cb[1:]]))
            fams = [(int(self.fs.origin_starts[d]),
                     int(self.fs.column_sizes[d]), up, done)
                    for d, up, done in fams]
            chunks = [self._global_strips(
                cells=np.arange(cb[j], cb[j + 1], dtype=np.int32))
                for j in range(len(cb) - 1)]
            self._band_plan = (fams, chunks)
        return self._band_plan

    def _apply_host_bands(self, x_host, coords, y_host):
        """Host buffers, vertex / edge column layouts: the upload of the
        next entity band, the strip kernel over cell chunk j and the
        download of the columns chunk j completed overlap (three streams,
        events between)."""
        import torch
        xd, yd, s_up, s_cmp, s_down = self._hbuf
        cur = torch.cuda.current_stream()
        fams, chunks = self._bands()
        for s_ in (s_up, s_cmp, s_down):
            s_.wait_stream(cur)
        with torch.cuda.stream(s_cmp):
            yd.zero_()
        up0 = [0] * len(fams)
        dn0 = [0] * len(fams)
        n = self.fs.total_dofs
        for j, (strips, W) in enumerate(chunks):
            with torch.cuda.stream(s_up):
                for f, (org, col, up, _done) in enumerate(fams):
                    if up[j] > up0[f]:
                        a, b = org + up0[f] * col, org + up[j] * col
                        xd[a:b].copy_(x_host[a:b], non_blocking=True)
                        up0[f] = up[j]
            s_cmp.wait_stream(s_up)
            _lib.column_mass_strip_red(self.fs.layout, self.k, self.layers,
                                       coords, self.mref, xd, yd, n, strips,
                                       self.kron, W, accumulate=True,
                                       stream=s_cmp,
                                       n_vertices=self.fs.mesh.base.num_vertices)
            s_down.wait_stream(s_cmp)
            with torch.cuda.stream(s_down):
                for f, (org, col, _up, done) in enumerate(fams):
                    if done[j] > dn0[f]:
                        a, b = org + dn0[f] * col, org + done[j] * col
                        y_host[a:b].copy_(yd[a:b], non_blocking=True)
                        dn0[f] = done[j]
        cur.wait_stream(s_down)
        cur.synchronize()
        return y_host

    def _global_strips(self, cells=None):
        """Sequential strips over the mesh (cached) or over ``cells``."""
        if self._gstrips is None or cells is not None:
            import torch
            n = self.n_cells if cells is None else len(cells)
            edges = bool(self.fs.layout.dofs(1, 0) or self.fs.layout.dofs(1, 1))
            import os
            res = _lib.build_global_strips(
                self.fs.mesh.base, max_len=strip_max_len(n, self.layers),
                cells=cells, edges=edges,
                # PM_STRIP_RUNS=1 (tuning knob): strips along the vertex-id
                # bands (pm_build_run_strips) for the cp.async kernels too
                runs=os.environ.get("PM_STRIP_RUNS", "0") == "1")
            g = (tuple(torch.from_numpy(a).to(self._dev) for a in res),
                 strip_chunk_width(self.layers))
            if cells is not None:
                return g
            self._gstrips = g
        return self._gstrips

    @property
    def striptma_ok(self) -> bool:
        """Layouts and sizes the run-strip kernel takes: P1 / 3-vector P1
        columns of at most 128 layers (P1 with two chunks per warp: 256)."""
        d = tuple(int(v) for v in self.fs.layout.delta6())
        two = d[0] == 1 and self.layers > 32 and (self.layers - 1) % 64 >= 32
        return d in ((1, 0, 0, 0, 0, 0), (3, 0, 0, 0, 0, 0)) and \
            self.strip_invariant and self.layers <= (256 if two else 128)

    @property
    def striptma_auto(self) -> bool:
        """``auto`` takes the run-strip kernel where it measured faster than
        the cp.async strips (C5a 2.91 -> 2.34 ms, profiles/README.md):
        scalar P1 columns in whole 32-layer chunks, two per warp (64, 128,
        192 or 256 layers: no predicated RED in the strip loop; config 4 at
        256 layers 0.217 -> 0.178 ms), on a mesh whose strips
        follow vertex-id runs and are long enough to hide the ring's cold
        start per strip.  PM_STRIPTMA=0 keeps the cp.async strips."""
        if self._tma_auto is None:
            import os
            ok = False
            d = tuple(int(v) for v in self.fs.layout.delta6())
            if d == (1, 0, 0, 0, 0, 0) and self.striptma_ok and \
                    self.layers % 64 == 0 and \
                    os.environ.get("PM_STRIPTMA", "1") != "0":
                (sp, st), frac = self._run_strips()
                mean = st.shape[0] / max(1, sp.shape[0] - 1)
                ok = frac >= 0.9 and mean >= 128
            self._tma_auto = ok
        return self._tma_auto

    def _run_strips(self):
        """Strips along the vertex-id bands (pm_build_run_strips, cached)
        and the fraction of steps whose vertex continues its side's id run:
        (device (strip_ptr, steps), fraction)."""
        if self._rstrips is None:
            import numpy as np
            import torch
            sp, st = _lib.build_global_strips(
                self.fs.mesh.base, runs=True,
                max_len=run_strip_max_len(self.n_cells, self.layers))
            d2 = st[2:] == st[:-2] + 1
            # (pairs across a strip boundary: 2 of each strip's steps)
            frac = float(d2.sum()) / max(1, len(st) - 2 * (len(sp) - 1))
            self._rstrips = (tuple(torch.from_numpy(a).to(self._dev)
                                   for a in (sp, st)), frac)
        return self._rstrips

    @property
    def stripdg_ok(self) -> bool:
        """Cell-only layouts the DG strip kernel compiles: DoFs on (2,1)
        only (1, 2, 3 or 6 per cell-layer) or on (2,0) only (1 or 3 per
        cell level)."""
        d = self.fs.layout.delta6()
        if d[0] or d[1] or d[2] or d[3]:
            return False
        if not d[4]:
            return d[5] in (1, 2, 3, 6)
        return not d[5] and d[4] in (1, 3)

    def _dg_strips(self):
        """Global strips + the cell of every step (cached), for the DG
        strip kernel."""
        if self._dgstrips is None:
            import torch
            base = self.fs.mesh.base
            sp, st = _lib.build_global_strips(
                base, max_len=strip_max_len(self.n_cells, self.layers))
            sc = _lib.strip_step_cells(base, sp, st)
            self._dgstrips = (tuple(torch.from_numpy(a).to(self._dev)
                                    for a in (sp, st, sc)),
                              strip_chunk_width(self.layers))
        return self._dgstrips

    def _patch_strips(self):
        """Store-first patch strips (cached): Morton patches of the cells,
        sequential strips inside each (pm_build_patch_strips)."""
        if self._pstrips is None:
            import torch
            from .schedule import morton_order
            base = self.fs.mesh.base
            cv = np.asarray(base.cell_vertices)
            cent = np.asarray(base.coords)[cv].mean(axis=1)
            order = morton_order(cent).astype(np.int32)
            W = strip_chunk_width(self.layers)
            P = patch_strip_size(self.n_cells, self.layers)
            ptr = np.arange(0, self.n_cells + P, P, dtype=np.int64)
            ptr[-1] = self.n_cells
            ptr = np.unique(ptr).astype(np.int32)
            import os
            if os.environ.get("PM_PATCH_ORDER", "rcm") == "rcm":
                # patches in order of their mean vertex id: on RCM-ordered
                # meshes the running patches sweep the mesh along the RCM
                # front, like the global strips
                key = np.add.reduceat(cv[order].astype(np.float64).sum(1),
                                      ptr[:-1]) / np.diff(ptr)
                porder = np.argsort(key, kind="stable")
                lens = np.diff(ptr)[porder]
                order = np.concatenate([order[ptr[p]:ptr[p + 1]]
                                        for p in porder]).astype(np.int32)
                ptr = np.zeros(len(lens) + 1, dtype=np.int32)
                np.cumsum(lens, out=ptr[1:])
            edges = bool(self.fs.layout.dofs(1, 0) or
                         self.fs.layout.dofs(1, 1))
            res = _lib.build_patch_strips(base, order, ptr, edges=edges)
            if not edges:
                res = res[:3] + (None,) + res[3:]
            dev = tuple(None if a is None else torch.from_numpy(a).to(self._dev)
                        for a in res)
            self._pstrips = (dev, W)
        return self._pstrips

    def _strip_plan(self):
        if self._strip is None:
            from .schedule import build_strip_plan
            col = _color(self.fs.mesh)
            plan = build_strip_plan(self.fs.mesh.base, self.fs.layout,
                                    self.layers, col.color_of,
                                    col.num_colors)
            self._strip = (plan, plan.device(self._dev))
        return self._strip

    def _patch_plan(self):
        if self._patch is None:
            from .schedule import plan_for
            col = _color(self.fs.mesh)
            plan, W, _ch, _need = plan_for(self.fs.mesh.base, self.fs.layout,
                                           self.layers, col.color_of,
                                           col.num_colors)
            self._patch = (plan, plan.device(self._dev), W)
        return self._patch

    def _color_lists(self):
        if self._coloring is None:
            import torch
            col = _color(self.fs.mesh)
            order, ptr = col.cells_by_color()
            d_order = torch.from_numpy(order).to(self._dev)
            self._coloring = (d_order, ptr)
        return self._coloring

    def graph(self, x, coords, y, accumulate=False, schedule=None, repeat=1,
              overlap=False):
        """``repeat`` back-to-back ``apply`` calls on fixed device buffers
        captured as one CUDA graph (``torch.cuda.CUDAGraph``; ``.replay()``
        re-runs them on the current stream): repeated application without
        per-call host work, for launch-bound sizes and solver loops.

        ``overlap``: programmatic dependent launch between the captured DG
        stream kernels — each starts its prologue, loads and gathers while
        the previous one drains and waits for it only before its first
        store (the captured calls share their inputs, so this is safe)."""
        import torch
        self.apply(x, coords, y, accumulate=accumulate, schedule=schedule)
        torch.cuda.synchronize()        # plans and kernel attributes ready
        g = torch.cuda.CUDAGraph()
        prev = _lib.set_launch_overlap(overlap)
        try:
            with torch.cuda.graph(g):
                for _ in range(repeat):
                    self.apply(x, coords, y, accumulate=accumulate,
                               schedule=schedule)
        finally:
            _lib.set_launch_overlap(prev)
        torch.cuda.synchronize()
        return g

    def apply(self, x, coords, y=None, accumulate=False, schedule=None,
              stream=None):
        """Device tensors in/out; returns ``y``."""
        import torch
        sched = schedule or self.schedule
        n = self.fs.total_dofs
        if x.shape[0] != n:
            raise ValueError(f"x has {x.shape[0]} values, space has {n}")
        if coords.shape[0] != self.coord_fs.total_dofs:
            raise ValueError("coordinate field does not match the mesh")
        if y is None:
            y = torch.empty(n, dtype=torch.float64, device=x.device)
            accumulate = False
        if not self.kron_ok and sched not in ("stream", "stripdg"):
            sched = "atomic"   # dense Mref in the generic kernel
        if sched == "auto" and self.stripdg_ok and \
                not (self.dg_only and self.k == 6):
            # cell-only layouts with few DoFs per cell-layer: walking the
            # cells along strips loads each vertex's coordinates once per
            # strip instead of gathering six prism vertices per cell-layer
            # (measured at 100 layers: DG0xDG0 +54 %, DG0xDG1 +20 %,
            # DG1xDG0 +6 % over the stream kernel, DG0xCG1 +44 %, DG1xCG1
            # +12 % over the cell-stream kernel; DG1xDG1 keeps the stream
            # kernel, profiles/README.md)
            sched = "stripdg"
        if sched == "auto" and self.share == 2:
            # measured fastest (profiles/): global strips for vertex-column
            # layouts (run strips with bulk-copied columns where they apply),
            # the warp-per-column kernel otherwise
            if self.striptma_auto and x.data_ptr() % 16 == 0 and \
                    coords.data_ptr() % 16 == 0:
                sched = "striptma"
            else:
                sched = "stripred" if self.stripred_ok else "column"
        self.last_schedule = sched
        if sched == "stripred":
            if not self.stripred_ok:
                raise ValueError(
                    f"the strip schedule needs a vertex-column layout and a "
                    f"vertex-permutation invariant triangle factor, got "
                    f"{self.fs.layout.name}")
            strips, W = self._global_strips()
            _lib.column_mass_strip_red(self.fs.layout, self.k, self.layers,
                                       coords, self.mref, x, y, n, strips,
                                       self.kron, W, accumulate=accumulate,
                                       stream=stream,
                                       n_vertices=self.fs.mesh.base.num_vertices)
            return y
        if sched == "striptma":
            if not self.striptma_ok:
                raise ValueError(
                    f"the run-strip schedule takes P1 / 3-vector P1 columns "
                    f"of at most 128 layers, got {self.fs.layout.name} with "
                    f"{self.layers} layers")
            strips, _ = self._run_strips()
            _lib.column_mass_strip_tma(self.fs.layout, self.k, self.layers,
                                       coords, x, y, n, strips, self.kron,
                                       accumulate=accumulate, stream=stream,
                                       n_vertices=self.fs.mesh.base.num_vertices)
            return y
        if sched == "stripdg":
            if not self.stripdg_ok:
                raise ValueError(
                    f"the DG strip schedule needs DoFs on the prism cells "
                    f"only (1, 2, 3 or 6 per cell-layer, or 1 or 3 per "
                    f"cell level), got {self.fs.layout.name}")
            strips, W = self._dg_strips()
            out = torch.empty_like(y) if accumulate else y
            _lib.column_mass_strip_dg(self.fs.layout, self.k, self.n_cells,
                                      self.layers, coords, self.mref, x,
                                      out, strips, W, stream=stream)
            if accumulate:
                y += out
            return y
        if sched == "tile":
            if not self.tile_ok:
                raise ValueError(
                    f"the tile schedule needs a vertex-column layout (P1, "
                    f"3-vector P1, CG1xDG0, CG1xDG1) and a vertex-permutation "
                    f"invariant triangle factor, got {self.fs.layout.name}")
            plan = self._tile_plan()
            out = y
            if accumulate:
                if self._tile_tmp is None or self._tile_tmp.shape != y.shape:
                    self._tile_tmp = torch.empty_like(y)
                out = self._tile_tmp
            _lib.column_mass_tile(self.fs.layout, self.layers, coords, x, out,
                                  n, plan, self.kron, plan["width"],
                                  stream=stream)
            if accumulate:
                y += out
            return y
        if sched == "pstrip":
            if not self.stripred_ok:
                raise ValueError(
                    f"the patch-strip schedule needs a vertex-column layout "
                    f"and a vertex-permutation invariant triangle factor, got "
                    f"{self.fs.layout.name}")
            plan, W = self._patch_strips()
            _lib.column_mass_patch_strips(
                self.fs.layout, self.k, self.layers, coords, self.mref, x, y,
                n, plan, self.kron, W, accumulate=accumulate, stream=stream,
                n_vertices=self.fs.mesh.base.num_vertices)
            return y
        if sched == "strip":
            if not self.strip_ok:
                raise ValueError(
                    f"the strip schedule needs a vertex-column layout and a "
                    f"vertex-permutation invariant triangle factor, got "
                    f"{self.fs.layout.name}")
            plan, dplan = self._strip_plan()
            out = torch.empty_like(y) if accumulate else y
            _lib.column_mass_strip(self.fs.layout, self.k, self.layers,
                                   coords, self.mref, x, out, plan, dplan,
                                   self.kron, stream=stream)
            if accumulate:
                y += out
            return y
        if sched == "patch":
            if not self.patch_ok:
                raise ValueError(
                    f"the patch schedule needs a vertex/edge-only layout, "
                    f"got {self.fs.layout.name}")
            plan, dplan, W = self._patch_plan()
            if accumulate:
                tmp = torch.empty_like(y)
                _lib.column_mass_patch(self.fs.layout, self.k,
                                       self.fs.mesh.base, self.layers,
                                       self.cmap, self.xmap, coords,
                                       self.mref, x, tmp, plan, dplan, W,
                                       stream=stream, kron=self.kron)
                y += tmp
            else:
                _lib.column_mass_patch(self.fs.layout, self.k,
                                       self.fs.mesh.base, self.layers,
                                       self.cmap, self.xmap, coords,
                                       self.mref, x, y, plan, dplan, W,
                                       stream=stream, kron=self.kron)
            return y
        if sched not in _VARIANTS:
            raise ValueError(f"unknown schedule {sched!r}")
        if sched in ("colored", "sequential") and self.share == 2:
            # one launch per colour: no two columns of a launch share a DoF
            if not accumulate:
                y.zero_()
            order, ptr = self._color_lists()
            for c in range(len(ptr) - 1):
                _lib.column_mass(self.fs.layout, self.k, self.n_cells,
                                 self.layers, self.cmap, self.offs, self.xmap,
                                 self.xoffs, coords, self.mref, x, y, n,
                                 accumulate=True,
                                 variant=_lib.VARIANT_COLORED,
                                 cells=order[ptr[c]:ptr[c + 1]],
                                 stream=stream, kron=self.kron)
            return y
        if sched == "stream" and self.share != 0:
            raise ValueError("the stream schedule needs a DG (2,1) layout")
        _lib.column_mass(self.fs.layout, self.k, self.n_cells, self.layers,
                         self.cmap, self.offs, self.xmap, self.xoffs, coords,
                         self.mref, x, y, n, accumulate=accumulate,
                         variant=_VARIANTS[sched], stream=stream,
                         kron=self.kron)
        return y


#: layouts compiled into the patch kernel (csrc/patch.cu)
_PATCH_LAYOUTS = {(1, 0, 0, 0, 0, 0), (0, 1, 0, 0, 0, 0), (0, 2, 0, 0, 0, 0),
                  (1, 1, 1, 1, 0, 0), (3, 0, 0, 0, 0, 0)}

#: layouts compiled into the strip kernels (csrc/strip.cu, strip_red.cu)
_STRIP_LAYOUTS = {(1, 0, 0, 0, 0, 0), (0, 1, 0, 0, 0, 0), (0, 2, 0, 0, 0, 0),
                  (3, 0, 0, 0, 0, 0)}
_STRIPRED_LAYOUTS = _STRIP_LAYOUTS | {(1, 1, 1, 1, 0, 0)}

_VARIANTS = {"auto": _lib.VARIANT_AUTO, "atomic": _lib.VARIANT_ATOMIC,
             "column": _lib.VARIANT_COLUMN, "stream": _lib.VARIANT_STREAM,
             # deterministic schedules for layouts without horizontal
             # sharing: the column kernel writes every DoF exactly once
             "colored": _lib.VARIANT_COLUMN,
             "sequential": _lib.VARIANT_COLUMN}


def strip_chunk_width(layers: int) -> int:
    """Lanes per layer chunk for the strip kernel (least lane waste, a
    small per-chunk charge); PM_STRIP_W overrides (tuning knob)."""
    import os
    forced = int(os.environ.get("PM_STRIP_W", "0"))
    if forced in (8, 16, 32):
        return forced
    # lane slots (chunks x W) weighted by a per-slot cost that grows as the
    # segments narrow (more lines touched per warp instruction): fitted to
    # the config-4 P1 sweep over W in {8, 16, 32} and λ in {1 .. 256}
    # (e.g. λ = 256: 0.458 / 0.272 / 0.249 ms) and C3 (P2, λ = 100: W = 32
    # 5 % faster than 16), profiles/README.md
    cost = {8: 1.6, 16: 1.15, 32: 1.0}
    return min((8, 16, 32), key=lambda w: (-(-layers // w) * w * cost[w], -w))


def patch_strip_size(n_cells: int, layers: int) -> int:
    """Cells per patch of the store-first patch strips: large patches share
    fewer entities (zeroed, added), small ones give enough (patch, chunk)
    items to fill 148 SMs; PM_PATCH_CELLS overrides (tuning knob)."""
    import os
    forced = int(os.environ.get("PM_PATCH_CELLS", "0"))
    if forced > 0:
        return forced
    chunks = -(-layers // strip_chunk_width(layers))
    return int(max(32, min(512, n_cells * chunks // (148 * 64))))


def strip_max_len(n_cells: int, layers: int) -> int:
    """Strip length cap: long strips amortise the 3-vertex fill, the final
    flushes and the per-strip setup, but small meshes need enough (strip,
    chunk) items to fill 148 SMs.  Measured (profiles/README.md): cap 512
    vs 32 takes C5a 3.78 -> 3.35 ms, C5b 9.41 -> 8.66, C3 1.66 -> 1.60;
    4096 is slower again (too few items).  PM_STRIP_MAXLEN overrides."""
    import os
    cap = int(os.environ.get("PM_STRIP_MAXLEN", "512"))
    items = int(os.environ.get("PM_STRIP_ITEMS", "12000"))  # tuning knob
    chunks = -(-layers // strip_chunk_width(layers))
    return int(max(4, min(cap, n_cells * chunks // items)))


def run_strip_max_len(n_cells: int, layers: int) -> int:
    """Strip length cap of the run strips (csrc/strip_tma.cu): its warp
    groups own whole columns, so a few hundred strips fill the GPU and long
    strips pay the ring's cold start least (config 4, P1, 256 layers: 0.178
    ms at 512 against 0.23-0.26 at 64-256).  PM_STRIP_MAXLEN overrides."""
    import os
    return int(os.environ.get("PM_STRIP_MAXLEN", "512"))


_COLORINGS = {}


def _color(mesh):
    from .iterate import color_base_cells
    key = id(mesh.base)
    hit = _COLORINGS.get(key)
    if hit is None or hit[0] is not mesh.base:
        hit = (mesh.base, color_base_cells(mesh))
        _COLORINGS[key] = hit
    return hit[1]


class MassKernel:
    """Stencil kernel ``I_1``: arity (k of the field space, 18 coords)."""

    def __init__(self, fs: FunctionSpace, quadrature=None, element=None):
        self.fs = fs
        self.element = element or element_for_layout(fs.layout)
        self.quadrature = quadrature or default_quadrature(self.element)
        self.arity = (fs.num_slots, 18)
        self._op = None

    def launch(self, fs_list, fields, schedule, stream=None):
        if len(fields) != 3:
            raise ValueError("mass kernel fields are [f, coords, out]")
        if fs_list[1].layout.counts != COORDS_LAYOUT.counts:
            raise ValueError("second space must be the coordinate space")
        if self._op is None or self._op.fs is not fs_list[0]:
            self._op = MassOperator(fs_list[0], self.quadrature, self.element)
        f, coords, out = fields
        self._op.apply(f, coords, out, accumulate=True, schedule=schedule,
                       stream=stream)


class CountingKernel:
    """Adds 1 to every output DoF a cell-layer touches."""

    def __init__(self, fs):
        self.arity = (fs.num_slots,)

    def launch(self, fs_list, fields, schedule, stream=None):
        (out,) = fields
        _lib.column_probe(1, fs_list[0], out, stream=stream)


class ListProbeKernel:
    """Writes each cell-layer's DoF list (N2, layers, k) int64: the
    materialised maps of verification.py:47-75, produced by the loop."""

    def __init__(self, fs):
        self.arity = (fs.num_slots,)

    def launch(self, fs_list, fields, schedule, stream=None):
        (out,) = fields
        _lib.column_probe(0, fs_list[0], out, stream=stream)


def _coords_device(fs, coords, dev):
    import torch
    if coords is None:
        from .extrusion import extrude_coordinates
        m = fs.mesh
        return extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    c, _ = _as_device(coords, dev)
    return c


def mass_action(fs, x, coords=None, quadrature=None, schedule="auto",
                operator: MassOperator = None, out=None):
    """``y = M x`` on ``fs``.

    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out; a host torch
    tensor ``out`` (ideally pinned) receives the result in place.
    """
    import torch
    op = operator or MassOperator(fs, quadrature)
    if op.fs is not fs:
        raise ValueError("operator was prepared for another space")
    dev = op._dev
    d_c = _coords_device(fs, coords, dev)
    if (out is not None and isinstance(x, torch.Tensor) and
            x.device.type == "cpu" and out.device.type == "cpu" and
            schedule == "auto"):
        # host in, host out: copies pipelined with the compute
        return op.apply_host(x, d_c, out)
    d_x, x_host = _as_device(x, dev)
    y = op.apply(d_x, d_c, schedule=schedule)
    if out is not None:
        out.copy_(y, non_blocking=out.device.type == "cpu" and out.is_pinned())
        torch.cuda.current_stream().synchronize()
        return out
    if x_host:
        return y.cpu().numpy()
    return y


def assemble_residual(fs, f, coords=None, quadrature=None, schedule="auto",
                      operator: MassOperator = None):
    """``b_j = sum_{c,l} sum_q w_q |det J| phi_j(q) f(q)``.

    ``coords`` is the extruded coordinate field (default: built on the
    device from the base mesh).  Returns a Field if ``f`` is a Field.
    """
    vals = f.values if isinstance(f, Field) else f
    if isinstance(f, Field) and f.space is not fs:
        raise ValueError("f does not live on fs")
    out = mass_action(fs, vals, coords, quadrature, schedule, operator)
    return Field(fs, out) if isinstance(f, Field) else out
