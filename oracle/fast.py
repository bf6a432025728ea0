"""CPU baseline arm -- TEST INFRASTRUCTURE ONLY (bench.py's reference arm and
cpu_baseline, tests/test_cpu_baseline.py).

``FastMass`` runs ``cpu_fast.c`` (the reference's coloured column loop with
a pre-integrated element matrix, SPEC.md:333-364 + 412-420) on every host
core.  The library is compiled on the machine that runs it (``-O3
-march=native -ffast-math``, the paper's flags) into a
private temporary directory.  Everything it needs -- mesh, maps, extruded
coordinates, the element matrix, the colouring -- comes from the oracle
(``oracle/``), never from the product library.
"""
from __future__ import annotations

import ctypes
import os
import platform
import subprocess
import tempfile
import time

import numpy as np

from . import HERE, Problem, _f64p, _i32p, _i64p, _p, cell_map, extrude, \
    greedy_color

_fast = None


def _build():
    global _fast
    if _fast is None:
        out = os.path.join(tempfile.mkdtemp(prefix="pm_cpu_fast_"),
                           "libcpufast.so")
        flags = ["-O3", "-march=native", "-ffast-math", "-fPIC", "-shared",
                 "-std=gnu11"]
        r = subprocess.run(["gcc", *flags, os.path.join(HERE, "cpu_fast.c"),
                            "-o", out, "-lm", "-lpthread"],
                           capture_output=True, text=True)
        if r.returncode:   # no -march=native support: portable build
            flags[1] = "-march=x86-64-v2"
            subprocess.run(["gcc", *flags, os.path.join(HERE, "cpu_fast.c"),
                            "-o", out, "-lm", "-lpthread"], check=True)
        L = ctypes.CDLL(out)
        L.cf_mass.restype = ctypes.c_int
        L.cf_mass.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                              _i32p, _i32p, _i32p, _i32p, _f64p, _f64p, _f64p,
                              _f64p, ctypes.c_int64, _i32p, _i64p,
                              ctypes.c_int32, ctypes.c_int32]
        L.cf_threads.restype = ctypes.c_int
        L.cf_threads.argtypes = []
        _fast = (L, " ".join(flags))
    return _fast


def reference_matrix(counts, tri, line, ncomp, tri_deg, line_deg):
    """The element matrix M_ref (k x k, slot order) by the oracle's literal
    quadrature: one reference prism (unit right triangle, height 1, so
    |det J| = 1) assembled against each unit vector."""
    from . import Mesh
    m = Mesh(np.array([[0, 1, 2]], dtype=np.int32),
             np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]))
    prob = Problem(m, 1, counts, tri, line, ncomp, tri_deg, line_deg,
                   layer_height=1.0)
    k = prob.k
    cmap = prob.map[0]
    M = np.zeros((k, k))
    for j in range(k):
        e = np.zeros(prob.total)
        e[cmap[j]] = 1.0
        M[:, j] = prob.assemble(e)[cmap]
    return M


def cpu_info():
    """(physical cores, logical cores, model name) of this host."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    logical = os.cpu_count() or 1
    physical = logical
    try:
        import psutil
        physical = psutil.cpu_count(logical=False) or logical
    except Exception:
        pass
    return physical, logical, model


class FastMass:
    """``y = M x`` over every cell-layer of (base, layers, layout) on the
    host cores (coloured schedule, pre-integrated M_ref)."""

    def __init__(self, base, layers, counts, tri, line, ncomp, tri_deg,
                 line_deg, layer_height=None, threads=0):
        self.base = base
        self.layers = layers
        h = 1.0 / layers if layer_height is None else layer_height
        self.map, self.off, self.total = cell_map(base, layers, counts)
        self.xmap, self.xoff, self.xtotal = cell_map(base, layers, {(0, 0): 3})
        self.coords = extrude(base.coords, layers, h)
        self.k = self.map.shape[1]
        self.mref = np.ascontiguousarray(
            reference_matrix(counts, tri, line, ncomp, tri_deg, line_deg))
        L, self.flags = _build()
        self.threads = threads or L.cf_threads()
        self.schedule = self._schedule(base, counts)
        self.y = np.empty(self.total)

    def _schedule(self, base, counts):
        """Per (colour, thread) cell ranges: one pass of contiguous blocks
        for cell-only (DG) layouts; two passes (even, odd blocks) when
        same-parity blocks share no vertex / edge (RCM-ordered meshes);
        else the greedy colouring, split evenly."""
        T, n = self.threads, base.num_cells
        shared = [d for d in (0, 1) if counts.get((d, 0)) or counts.get((d, 1))]
        if not shared:
            self.order = np.arange(n, dtype=np.int32)
            self.tptr = np.array([n * t // T for t in range(T + 1)],
                                 dtype=np.int64)
            self.n_colors = 1
            return f"{T} contiguous cell blocks (no shared DoFs)"
        nb = 2 * T
        bounds = np.array([n * b // nb for b in range(nb + 1)])
        ok = n >= nb
        for d in shared:
            ents = np.asarray(base.cell_vertices if d == 0 else
                              base.cell_edges)
            if not ok:
                break
            lo = np.minimum.reduceat(ents.min(axis=1), bounds[:-1])
            hi = np.maximum.reduceat(ents.max(axis=1), bounds[:-1])
            ok = bool(np.all(hi[:-2] < lo[2:]))
        if ok:
            even = [np.arange(bounds[b], bounds[b + 1]) for b in range(0, nb, 2)]
            odd = [np.arange(bounds[b], bounds[b + 1]) for b in range(1, nb, 2)]
            self.order = np.concatenate(even + odd).astype(np.int32)
            sz = [len(a) for a in even + odd]
            self.tptr = np.zeros(nb + 1, dtype=np.int64)
            np.cumsum(sz, out=self.tptr[1:])
            self.n_colors = 2
            return (f"{nb} contiguous cell blocks, even blocks then odd "
                    f"blocks, one block per thread")
        col, nc = greedy_color(base)
        self.order = np.argsort(col, kind="stable").astype(np.int32)
        cptr = np.zeros(nc + 1, dtype=np.int64)
        np.cumsum(np.bincount(col, minlength=nc), out=cptr[1:])
        self.tptr = np.array([cptr[c] + (cptr[c + 1] - cptr[c]) * t // T
                              for c in range(nc) for t in range(T)] +
                             [cptr[nc]], dtype=np.int64)
        self.n_colors = nc
        return f"greedy colouring ({nc} colours), cells split evenly"

    def apply(self, x, y=None):
        L, _ = _build()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = self.y if y is None else y
        rc = L.cf_mass(self.base.num_cells, self.layers, self.k,
                       _p(self.map, _i32p), _p(self.off, _i32p),
                       _p(self.xmap, _i32p), _p(self.xoff, _i32p),
                       _p(self.coords, _f64p), _p(self.mref, _f64p),
                       _p(x, _f64p), _p(y, _f64p), self.total,
                       _p(self.order, _i32p), _p(self.tptr, _i64p),
                       self.n_colors, self.threads)
        if rc:
            raise ValueError("cpu_fast rejected its arguments")
        return y

    def time(self, x):
        t0 = time.perf_counter()
        self.apply(x)
        return time.perf_counter() - t0
