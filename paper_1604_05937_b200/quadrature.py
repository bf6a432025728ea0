"""Prism quadrature, tabulated bases and reference-prism mass matrices.

Restates the SPEC ``kernels`` module's host side (SPEC.md:381-410,
437-441): a prism rule is the tensor product of a symmetric triangle rule
of the requested degree with Gauss-Legendre points on [0, 1]; weights sum
to the reference prism measure 1/2.  Basis functions are the standard
affine/quadratic Lagrange functions on the reference triangle
``(0,0),(1,0),(0,1)`` times Lagrange functions on the interval.

Slot <-> basis convention (SPEC.md:300, 314 leave it open; fixed here and
in DESIGN.md): a slot's horizontal function is its vertex (``a``), edge
(``3+e``, edge ``e`` opposite vertex ``e``) or, for cell DoFs, the
``dof // (n_vert_funcs*ncomp)``-th triangle function; its vertical function
is 0 for the bottom level copy, the last for the top copy and the interior
/ discontinuous functions for the connecting entity.  So DG1xDG1 slot
``j = 2a + b`` and CG1xCG1 slot ``2a + b`` coincide, P2xP2 slot ``3t + b``
and the 3-vector P1 slot ``6a + 3b + comp``.

The column loop applies the pre-integrated matrix
``M_ref[j, j'] = sum_q w_q B_j(q) B_j'(q)`` scaled by ``|det J|`` per
cell-layer, which equals the SPEC's literal quadrature kernel up to
rounding because the rules are exact for these products.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

# Symmetric triangle rules on the reference triangle (area 1/2), polished
# to full precision by tools/polish_triangle_rules.py.
_S4 = (0.11169079483900567, 0.4459484909159648,
       0.054975871827661, 0.09157621350977078)
_S6 = (0.05839313786319256, 0.24928674517090688,
       0.025422453185103333, 0.06308901449150202,
       0.041425537809185384, 0.05314504984481456, 0.31035245103378556)


def _orbit_a(w, a):
    return [(a, a), (1 - 2 * a, a), (a, 1 - 2 * a)], [w] * 3


def _orbit_ab(w, a, b):
    c = 1 - a - b
    return [(a, b), (b, a), (a, c), (c, a), (b, c), (c, b)], [w] * 6


def _rule(parts):
    pts, ws = [], []
    for p, w in parts:
        pts += p
        ws += w
    return np.array(pts, dtype=np.float64), np.array(ws, dtype=np.float64)


@lru_cache(maxsize=None)
def triangle_rule(degree: int):
    """(points (n,2), weights (n,)) exact for polynomials of ``degree``."""
    if degree < 0:
        raise ValueError(f"quadrature degree must be >= 0, got {degree}")
    if degree <= 1:
        return np.array([[1 / 3, 1 / 3]]), np.array([0.5])
    if degree == 2:
        return _rule([_orbit_a(1 / 6, 1 / 6)])
    if degree <= 4:
        return _rule([_orbit_a(_S4[0], _S4[1]), _orbit_a(_S4[2], _S4[3])])
    if degree == 5:
        r = np.sqrt(15.0)
        return _rule([([(1 / 3, 1 / 3)], [9 / 80]),
                      _orbit_a((155 - r) / 2400, (6 - r) / 21),
                      _orbit_a((155 + r) / 2400, (6 + r) / 21)])
    if degree == 6:
        return _rule([_orbit_a(_S6[0], _S6[1]), _orbit_a(_S6[2], _S6[3]),
                      _orbit_ab(_S6[4], _S6[5], _S6[6])])
    raise ValueError(f"unsupported triangle quadrature degree {degree} "
                     "(supported: 0..6)")


@lru_cache(maxsize=None)
def line_rule(degree: int):
    """Gauss-Legendre on [0,1] with ``degree//2 + 1`` points."""
    if degree < 0:
        raise ValueError(f"quadrature degree must be >= 0, got {degree}")
    n = degree // 2 + 1
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


@dataclass(frozen=True)
class QuadratureRule:
    """Tensor-product prism rule: points (n,3) = (xi, eta, zeta)."""

    points: np.ndarray
    weights: np.ndarray
    tri_degree: int
    line_degree: int

    @property
    def num_points(self) -> int:
        return self.weights.shape[0]


def prism_quadrature(tri_degree: int = 2, line_degree: int = 2):
    """Triangle rule x Gauss line rule; triangle index runs slowest."""
    tp, tw = triangle_rule(tri_degree)
    lp, lw = line_rule(line_degree)
    pts = np.empty((tp.shape[0] * lp.shape[0], 3))
    pts[:, :2] = np.repeat(tp, lp.shape[0], axis=0)
    pts[:, 2] = np.tile(lp, tp.shape[0])
    w = np.repeat(tw, lp.shape[0]) * np.tile(lw, tp.shape[0])
    return QuadratureRule(pts, w, tri_degree, line_degree)


# ---------------------------------------------------------------------------
# basis functions
# ---------------------------------------------------------------------------
TRI_SIZE = {"P0": 1, "P1": 3, "P2": 6}
LINE_SIZE = {"P0": 1, "P1": 2, "P2": 3}


def tri_basis(family: str, xi, eta):
    """Rows = basis functions, columns = points."""
    xi = np.asarray(xi, dtype=np.float64)
    eta = np.asarray(eta, dtype=np.float64)
    l0, l1, l2 = 1.0 - xi - eta, xi, eta
    if family == "P0":
        return np.ones((1,) + xi.shape)
    if family == "P1":
        return np.stack([l0, l1, l2])
    if family == "P2":
        return np.stack([l0 * (2 * l0 - 1), l1 * (2 * l1 - 1),
                         l2 * (2 * l2 - 1), 4 * l1 * l2, 4 * l2 * l0,
                         4 * l0 * l1])
    raise ValueError(f"unknown triangle family {family!r}")


def line_basis(family: str, z):
    z = np.asarray(z, dtype=np.float64)
    if family == "P0":
        return np.ones((1,) + z.shape)
    if family == "P1":
        return np.stack([1.0 - z, z])
    if family == "P2":
        return np.stack([(1 - z) * (1 - 2 * z), 4 * z * (1 - z),
                         z * (2 * z - 1)])
    raise ValueError(f"unknown line family {family!r}")


# ---------------------------------------------------------------------------
# elements: layout + families -> per-slot basis indices
# ---------------------------------------------------------------------------
_LABEL_FAMILY = {"CG1": "P1", "DG1": "P1", "DG0": "P0"}


@dataclass(frozen=True)
class PrismElement:
    """Tensor-product prism element bound to a layout's slot order."""

    tri: str
    line: str
    ncomp: int
    slot_h: tuple
    slot_v: tuple
    slot_comp: tuple

    @property
    def num_slots(self) -> int:
        return len(self.slot_h)


def _infer_families(layout):
    from .fspace import _BUILTIN, P2_LAYOUT, VP1_LAYOUT
    for (h, v), counts in _BUILTIN.items():
        if counts == layout.counts:
            return _LABEL_FAMILY[h], _LABEL_FAMILY[v], 1
    if layout.counts == P2_LAYOUT.counts:
        return "P2", "P2", 1
    if layout.counts == VP1_LAYOUT.counts:
        return "P1", "P1", 3
    raise ValueError(
        f"cannot infer the element of layout {layout.name!r}; pass "
        "tri=, line=, ncomp= explicitly")


def element_for_layout(layout, tri=None, line=None, ncomp=None):
    """Per-slot (horizontal, vertical, component) basis indices."""
    from .fspace import slot_table
    if tri is None or line is None or ncomp is None:
        t, l_, c = _infer_families(layout)
        tri, line, ncomp = tri or t, line or l_, ncomp or c
    nh, nv = TRI_SIZE[tri], LINE_SIZE[line]
    hs, vs, cs = [], [], []
    for s in slot_table(layout):
        d = s.base_dim
        v_cont = layout.dofs(d, 0) > 0          # vertically continuous
        if s.level_kind == 0:
            v_opts = [0]
        elif s.level_kind == 2:
            v_opts = [nv - 1]
        else:
            v_opts = list(range(1, nv - 1)) if v_cont else list(range(nv))
        if d == 0:
            h_opts = [s.local]
        elif d == 1:
            if tri != "P2":
                raise ValueError("edge DoFs need a P2 triangle family")
            h_opts = [3 + s.local]
        else:
            h_opts = list(range(nh))
        n_v, n_h = len(v_opts), len(h_opts)
        per = n_h * n_v * ncomp
        want = layout.dofs(d, 1 if s.level_kind == 1 else 0)
        if want != per:
            raise ValueError(
                f"layout {layout.name!r}: entity ({d},{int(s.level_kind == 1)})"
                f" holds {want} DoFs but {tri}x{line}x{ncomp} needs {per}")
        hi, rem = divmod(s.dof, n_v * ncomp)
        vi, comp = divmod(rem, ncomp)
        hs.append(h_opts[hi])
        vs.append(v_opts[vi])
        cs.append(comp)
    return PrismElement(tri, line, ncomp, tuple(hs), tuple(vs), tuple(cs))


def tabulate(element: PrismElement, rule: QuadratureRule):
    """B[j, q] = value of slot j's scalar basis at quadrature point q."""
    T = tri_basis(element.tri, rule.points[:, 0], rule.points[:, 1])
    L = line_basis(element.line, rule.points[:, 2])
    h = np.array(element.slot_h)
    v = np.array(element.slot_v)
    return T[h] * L[v]


def reference_mass_matrix(element: PrismElement, rule: QuadratureRule):
    """M_ref[j, j'] = delta(comp) * sum_q w_q B_j(q) B_j'(q)."""
    B = tabulate(element, rule)
    M = (B * rule.weights) @ B.T
    comp = np.array(element.slot_comp)
    M *= (comp[:, None] == comp[None, :])
    return np.ascontiguousarray(M)


def tensor_factors(rule: QuadratureRule):
    """Split a prism rule into its triangle and interval rules:
    ``((tri points (nt,2), tri weights), (line points (nl,), line weights))``
    when the points are the product grid (triangle index slowest, as
    ``prism_quadrature`` builds them) and the weights the outer product;
    ``None`` otherwise."""
    pts = np.asarray(rule.points, dtype=np.float64)
    w = np.asarray(rule.weights, dtype=np.float64)
    n = w.shape[0]
    if n == 0:
        return None
    same = np.all(pts[:, :2] == pts[0, :2], axis=1)
    nl = int(np.argmin(same)) if not same.all() else n
    if n % nl:
        return None
    nt = n // nl
    P = pts.reshape(nt, nl, 3)
    W = w.reshape(nt, nl)
    tri, line = P[:, 0, :2], P[0, :, 2]
    wt = W.sum(axis=1)
    if wt[0] == 0:
        return None
    wl = W[0] / wt[0]
    ok = (np.array_equal(P[:, :, :2], np.broadcast_to(tri[:, None, :],
                                                        (nt, nl, 2))) and
          np.array_equal(P[:, :, 2], np.broadcast_to(line[None, :], (nt, nl)))
          and np.allclose(W, np.outer(wt, wl), rtol=1e-14, atol=0))
    return ((tri, wt), (line, wl)) if ok else None


def kronecker_factors(element: PrismElement, rule: QuadratureRule):
    """(Mtri, Mline) with Mref[j,j'] = delta(comp) Mtri[h,h'] Mline[v,v']:
    the triangle / interval mass matrices under the rule's own two factors
    (``tensor_factors``); ``None`` for a rule that is not a tensor product
    (the dense generic kernel then applies Mref)."""
    f = tensor_factors(rule)
    if f is None:
        return None
    (tp, tw), (lp, lw) = f
    T = tri_basis(element.tri, tp[:, 0], tp[:, 1])
    L = line_basis(element.line, lp)
    return (np.ascontiguousarray((T * tw) @ T.T),
            np.ascontiguousarray((L * lw) @ L.T))


def sharing_class(layout) -> int:
    """0: no sharing (DG on (2,1)); 1: vertical only; 2: horizontal."""
    dims = {d for (d, _v) in layout.counts}
    if dims - {2}:
        return 2
    if layout.dofs(2, 0):
        return 1
    return 0
