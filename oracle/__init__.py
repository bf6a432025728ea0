"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/_build/liboracle.so`` (built from
``prismesh_oracle.c`` by ``oracle/Makefile``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference
arm may import this package, and only as the checker; the product package
``paper_1604_05937_b200`` never imports it.

Parity status: PINNED.  The numbering / maps / offsets / coordinates are
checked against golden vectors produced by running the reference package
itself (``tests/golden/make_golden.py``); the assembly is checked against a
brute-force dense assembler over the reference's own materialised
per-(cell, layer) maps with an independent (collapsed-Gauss) quadrature,
and against the SPEC known answers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_lib = None

FAMILY = {"P0": 0, "P1": 1, "P2": 2}


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        L.or_slot_table.restype = ctypes.c_int
        L.or_slot_table.argtypes = [_i32p] * 5
        L.or_build_cell_map.restype = ctypes.c_int64
        L.or_build_cell_map.argtypes = [_i32p, _i32p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, _i32p,
                                        ctypes.c_int32, _i32p, _i32p]
        L.or_extrude.restype = None
        L.or_extrude.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.c_double, _f64p]
        L.or_tri_rule.restype = ctypes.c_int
        L.or_tri_rule.argtypes = [ctypes.c_int, _f64p, _f64p]
        L.or_line_rule.restype = ctypes.c_int
        L.or_line_rule.argtypes = [ctypes.c_int, _f64p, _f64p]
        L.or_slot_basis.restype = ctypes.c_int
        L.or_slot_basis.argtypes = [_i32p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _i32p, _i32p, _i32p]
        common = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _i32p,
                  _i32p, _i32p, _i32p, _f64p, ctypes.c_int, ctypes.c_int,
                  ctypes.c_int, _i32p, _i32p, _i32p, ctypes.c_int,
                  ctypes.c_int, _f64p, _f64p]
        L.or_assemble.restype = ctypes.c_int
        L.or_assemble.argtypes = common + [_i32p, ctypes.c_int64]
        L.or_assemble_colored.restype = ctypes.c_int
        L.or_assemble_colored.argtypes = common + [_i32p, _i64p,
                                                   ctypes.c_int32,
                                                   ctypes.c_int32]
        L.or_greedy_color.restype = ctypes.c_int32
        L.or_greedy_color.argtypes = [_i32p, ctypes.c_int64, _i64p, _i32p,
                                      _i32p]
        L.or_max_threads.restype = ctypes.c_int
        L.or_max_threads.argtypes = []
        L.or_unit_square.restype = None
        L.or_unit_square.argtypes = [ctypes.c_int32, _i32p, _f64p]
        L.or_derive_edges.restype = ctypes.c_int64
        L.or_derive_edges.argtypes = [_i32p, ctypes.c_int64, _i32p, _i32p]
        L.or_rcm_order.restype = None
        L.or_rcm_order.argtypes = [_i32p, ctypes.c_int64, ctypes.c_int64,
                                   _i64p]
        L.or_apply_ordering.restype = None
        L.or_apply_ordering.argtypes = [_i32p, ctypes.c_int64, _f64p,
                                        ctypes.c_int64, _i64p, _i32p, _f64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def delta6(counts):
    """Layout dict {(d1,d2): n} -> int32[6]."""
    return np.array([counts.get((a, b), 0) for a in (0, 1, 2)
                     for b in (0, 1)], dtype=np.int32)


def slot_table(counts):
    d = delta6(counts)
    out = [np.zeros(64, dtype=np.int32) for _ in range(4)]
    k = lib().or_slot_table(_p(d, _i32p), *[_p(o, _i32p) for o in out])
    return tuple(o[:k].copy() for o in out)


def cell_map(base, layers, counts):
    """(map int32 (N2,k), offsets int32 (k,), total int)."""
    d = delta6(counts)
    k = len(slot_table(counts)[0])
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    ce = np.ascontiguousarray(base.cell_edges, dtype=np.int32)
    n = cv.shape[0]
    m = np.empty((n, k), dtype=np.int32)
    off = np.empty(k, dtype=np.int32)
    total = lib().or_build_cell_map(_p(cv, _i32p), _p(ce, _i32p), n,
                                    base.num_vertices, base.num_edges,
                                    _p(d, _i32p), layers, _p(m, _i32p),
                                    _p(off, _i32p))
    return m, off, int(total)


def extrude(base_coords, layers, h):
    b = np.ascontiguousarray(base_coords, dtype=np.float64)
    out = np.empty(3 * b.shape[0] * (layers + 1))
    lib().or_extrude(_p(b, _f64p), b.shape[0], layers, float(h),
                     _p(out, _f64p))
    return out


def tri_rule(degree):
    xy = np.zeros(64)
    w = np.zeros(32)
    n = lib().or_tri_rule(degree, _p(xy, _f64p), _p(w, _f64p))
    if n < 0:
        raise ValueError(f"unsupported degree {degree}")
    return xy[:2 * n].reshape(n, 2).copy(), w[:n].copy()


def line_rule(degree):
    z = np.zeros(16)
    w = np.zeros(16)
    n = lib().or_line_rule(degree, _p(z, _f64p), _p(w, _f64p))
    return z[:n].copy(), w[:n].copy()


def slot_basis(counts, tri, line, ncomp):
    d = delta6(counts)
    h, v, c = (np.zeros(64, dtype=np.int32) for _ in range(3))
    k = lib().or_slot_basis(_p(d, _i32p), FAMILY[tri], FAMILY[line], ncomp,
                            _p(h, _i32p), _p(v, _i32p), _p(c, _i32p))
    if k < 0:
        raise ValueError(f"layout {counts} incompatible with {tri}x{line}")
    return h[:k].copy(), v[:k].copy(), c[:k].copy()


def vertex_cells(base):
    flat = np.asarray(base.cell_vertices, dtype=np.int64).ravel()
    order = np.argsort(flat, kind="stable")
    cells = np.repeat(np.arange(base.num_cells, dtype=np.int32), 3)[order]
    off = np.zeros(base.num_vertices + 1, dtype=np.int64)
    np.cumsum(np.bincount(flat, minlength=base.num_vertices), out=off[1:])
    return off, np.ascontiguousarray(cells, dtype=np.int32)


def greedy_color(base):
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    off, cells = vertex_cells(base)
    col = np.empty(cv.shape[0], dtype=np.int32)
    n = lib().or_greedy_color(_p(cv, _i32p), cv.shape[0], _p(off, _i64p),
                              _p(cells, _i32p), _p(col, _i32p))
    return col, int(n)


class Problem:
    """One (mesh, layers, layout, element, quadrature) assembly case."""

    def __init__(self, base, layers, counts, tri, line, ncomp, tri_deg,
                 line_deg, layer_height=None):
        self.base = base
        self.layers = layers
        self.h = 1.0 / layers if layer_height is None else layer_height
        self.counts = dict(counts)
        self.map, self.off, self.total = cell_map(base, layers, counts)
        self.k = self.map.shape[1]
        self.xmap, self.xoff, self.xtotal = cell_map(base, layers,
                                                     {(0, 0): 3})
        self.coords = extrude(base.coords, layers, self.h)
        self.sh, self.sv, self.sc = slot_basis(counts, tri, line, ncomp)
        self.fam = (FAMILY[tri], FAMILY[line], ncomp)
        self.deg = (tri_deg, line_deg)

    def _args(self, f, out):
        return (self.base.num_cells, self.layers, self.k,
                _p(self.map, _i32p), _p(self.off, _i32p),
                _p(self.xmap, _i32p), _p(self.xoff, _i32p),
                _p(self.coords, _f64p), *self.fam, _p(self.sh, _i32p),
                _p(self.sv, _i32p), _p(self.sc, _i32p), *self.deg,
                _p(f, _f64p), _p(out, _f64p))

    def assemble(self, f, coords=None, order=None):
        """Sequential Alg. 3 over cells (index order or ``order``)."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        if coords is not None:
            self.coords = np.ascontiguousarray(coords, dtype=np.float64)
        out = np.zeros(self.total)
        if order is None:
            rc = lib().or_assemble(*self._args(f, out), None, 0)
        else:
            o = np.ascontiguousarray(order, dtype=np.int32)
            rc = lib().or_assemble(*self._args(f, out), _p(o, _i32p),
                                   o.shape[0])
        if rc:
            raise ValueError("oracle assembly rejected its arguments")
        return out

    def assemble_colored(self, f, threads=0, coloring=None, n_cells=None):
        """Coloured-parallel Alg. 3; ``n_cells`` restricts the loop to the
        first cells (a bounded sample for timing)."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        col, n = coloring if coloring is not None else greedy_color(self.base)
        if n_cells is not None:
            col = col[:n_cells]
        order = np.argsort(col, kind="stable").astype(np.int32)
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(col, minlength=n), out=ptr[1:])
        out = np.zeros(self.total)
        rc = lib().or_assemble_colored(*self._args(f, out),
                                       _p(order, _i32p), _p(ptr, _i64p), n,
                                       threads)
        if rc:
            raise ValueError("oracle assembly rejected its arguments")
        return out


def max_threads():
    return lib().or_max_threads()


# ---------------------------------------------------------------------------
# base meshes without the product library (oracle_mesh.c)
# ---------------------------------------------------------------------------

class Mesh:
    """Base mesh arrays (the attributes Problem and the product's
    ExtrudedMesh read): cell_vertices, coords, edge_vertices, cell_edges."""

    def __init__(self, cell_vertices, coords):
        self.cell_vertices = np.ascontiguousarray(cell_vertices,
                                                  dtype=np.int32)
        self.coords = np.ascontiguousarray(coords, dtype=np.float64)
        n = self.cell_vertices.shape[0]
        ev = np.empty((max(1, 3 * n), 2), dtype=np.int32)
        ce = np.empty((n, 3), dtype=np.int32)
        ne = lib().or_derive_edges(_p(self.cell_vertices, _i32p), n,
                                   _p(ev, _i32p), _p(ce, _i32p))
        if ne < 0:
            raise ValueError("edge shared by more than two cells")
        self.edge_vertices = ev[:ne].copy()
        self.cell_edges = ce

    @property
    def num_vertices(self):
        return self.coords.shape[0]

    @property
    def num_edges(self):
        return self.edge_vertices.shape[0]

    @property
    def num_cells(self):
        return self.cell_vertices.shape[0]


def unit_square(n):
    """mesh.py:228-254 generate_unit_square_mesh."""
    k = n + 1
    cells = np.empty((2 * n * n, 3), dtype=np.int32)
    coords = np.empty((k * k, 2), dtype=np.float64)
    lib().or_unit_square(n, _p(cells, _i32p), _p(coords, _f64p))
    return Mesh(cells, coords)


def rcm_forward(mesh):
    """ordering.py:93-120 rcm_vertex_order: forward[old] = new."""
    fwd = np.empty(mesh.num_vertices, dtype=np.int64)
    ev = np.ascontiguousarray(mesh.edge_vertices, dtype=np.int32)
    lib().or_rcm_order(_p(ev, _i32p), ev.shape[0], mesh.num_vertices,
                       _p(fwd, _i64p))
    return fwd


def random_forward(count, seed):
    """ordering.py:123-131 random_order (numpy's PCG64 permutation)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shuffled = rng.permutation(count)
    forward = np.empty(count, dtype=np.int64)
    forward[shuffled] = np.arange(count)
    return forward


def apply_ordering(mesh, forward):
    """ordering.py:134-152 apply_ordering."""
    fwd = np.ascontiguousarray(forward, dtype=np.int64)
    cells = np.empty_like(mesh.cell_vertices)
    coords = np.empty_like(mesh.coords)
    lib().or_apply_ordering(_p(mesh.cell_vertices, _i32p), mesh.num_cells,
                            _p(mesh.coords, _f64p), mesh.num_vertices,
                            _p(fwd, _i64p), _p(cells, _i32p),
                            _p(coords, _f64p))
    return Mesh(cells, coords)


def base_mesh(n, ordering="rcm", jitter=0.0, seed=0):
    """The BASELINE config meshes, built like the product's
    configs.base_mesh: (mesh, rng) with rng = default_rng(seed) positioned
    after the jitter draws (interior vertices moved by U(-jitter h,
    jitter h) before the ordering)."""
    rng = np.random.default_rng(seed)
    nv = (n + 1) ** 2
    d = rng.uniform(-jitter / n, jitter / n, size=(nv, 2)) if jitter else None
    m = unit_square(n)
    if jitter:
        c = m.coords.copy()
        inner = (c[:, 0] > 0) & (c[:, 0] < 1) & (c[:, 1] > 0) & (c[:, 1] < 1)
        c[inner] += d[inner]
        m = Mesh(m.cell_vertices, c)
    if ordering == "rcm":
        m = apply_ordering(m, rcm_forward(m))
    elif ordering == "random":
        m = apply_ordering(m, random_forward(m.num_vertices, seed))
    elif ordering != "natural":
        raise ValueError(f"unknown ordering {ordering!r}")
    return m, rng
