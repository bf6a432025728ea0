"""Generate tests/golden/golden.npz by running the REFERENCE package.

Run in the build container (the reference is importable from
/root/reference/pkg/src; it does not exist on the GPU box, so its outputs
are frozen here as small fixtures):

    python tests/golden/make_golden.py

Contents (all produced by reference code unless noted):
* meshes: ``generate_unit_square_mesh`` (n=3,4,5), the two in-code fixture
  meshes of verification.py:129-135, ``rcm_vertex_order`` /
  ``random_order`` permutations and ``apply_ordering`` results;
* numbering: ``cell_map``, ``offsets``, ``total_dofs`` for the nine
  builtin layouts, P2xP2, 3-vector P1 and COORDS at several layer counts;
  ``materialized_cell_maps`` (verification.py:47-75) for small cases;
* ``extrude_coordinates`` output;
* assembly: b = int f v dx for seeded f, from a brute-force DENSE global
  assembler driven by the reference's materialised per-(cell, layer) maps
  with an independent collapsed-Gauss (Duffy) quadrature and |detJ| =
  2*area*h.  The basis<->slot convention is the one fixed in DESIGN.md.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from prismesh import extrusion, fspace, mesh, ordering, verification  # noqa

# the reference's own check_space calls a method its FunctionSpace lacks
# (verification.py:102); shim it in this process only.
fspace.FunctionSpace.dof_origin_index = (
    lambda s, d, i: s.dof_origin(mesh.EntityId(d, i)))

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

LAYOUTS = {f"{h}x{v}": fspace.builtin_layout(h, v)
           for h in ("CG1", "DG0", "DG1") for v in ("CG1", "DG0", "DG1")}
LAYOUTS["P2xP2"] = fspace.DofLayout("P2xP2", {(0, 0): 1, (0, 1): 1,
                                              (1, 0): 1, (1, 1): 1})
LAYOUTS["VP1"] = fspace.DofLayout("VP1", {(0, 0): 3})
LAYOUTS["coords"] = fspace.COORDS_LAYOUT

FAMILIES = {"CG1": "P1", "DG1": "P1", "DG0": "P0"}


def families(name):
    if name == "P2xP2":
        return "P2", "P2", 1
    if name in ("VP1", "coords"):
        return "P1", "P1", 3
    h, v = name.split("x")
    return FAMILIES[h], FAMILIES[v], 1


# ---------------------------------------------------------------- basis
def tri_fn(fam, h, x, y):
    l0, l1, l2 = 1 - x - y, x, y
    lam = (l0, l1, l2)
    if fam == "P0":
        return np.ones_like(x)
    if fam == "P1":
        return lam[h]
    if h < 3:
        return lam[h] * (2 * lam[h] - 1)
    e = h - 3
    return 4 * lam[(e + 1) % 3] * lam[(e + 2) % 3]


def line_fn(fam, v, z):
    if fam == "P0":
        return np.ones_like(z)
    if fam == "P1":
        return (1 - z, z)[v]
    return ((1 - z) * (1 - 2 * z), 4 * z * (1 - z), z * (2 * z - 1))[v]


def slot_basis(layout, tri, line, ncomp):
    """DESIGN.md convention, restated independently of the product."""
    nh = {"P0": 1, "P1": 3, "P2": 6}[tri]
    nv = {"P0": 1, "P1": 2, "P2": 3}[line]
    out = []
    for s in fspace.slot_table(layout):
        d = s.base_dim
        vcont = layout.dofs(d, 0) > 0
        n_v = 1 if s.level_kind != 1 else (nv - 2 if vcont else nv)
        hi, rem = divmod(s.dof, n_v * ncomp)
        vi, comp = divmod(rem, ncomp)
        h = s.local if d == 0 else (3 + s.local if d == 1 else hi)
        v = {0: 0, 2: nv - 1}.get(s.level_kind, (1 if vcont else 0) + vi)
        out.append((h, v, comp))
    return out


def duffy_rule(n=7):
    """Collapsed Gauss on the reference triangle: exact to degree 2n-2."""
    g, w = np.polynomial.legendre.leggauss(n)
    g, w = 0.5 * (g + 1), 0.5 * w
    U, V = np.meshgrid(g, g, indexing="ij")
    WU, WV = np.meshgrid(w, w, indexing="ij")
    x = U.ravel()
    y = (V * (1 - U)).ravel()
    wt = (WU * WV * (1 - U)).ravel()
    return x, y, wt


def local_mass(layout, name):
    tri, line, ncomp = families(name)
    sb = slot_basis(layout, tri, line, ncomp)
    x, y, wt = duffy_rule()
    gz, gw = np.polynomial.legendre.leggauss(6)
    gz, gw = 0.5 * (gz + 1), 0.5 * gw
    X = np.repeat(x, gz.size)
    Y = np.repeat(y, gz.size)
    Z = np.tile(gz, x.size)
    W = np.repeat(wt, gz.size) * np.tile(gw, x.size)
    B = np.array([tri_fn(tri, h, X, Y) * line_fn(line, v, Z)
                  for (h, v, _c) in sb])
    comp = np.array([c for (_h, _v, c) in sb])
    M = (B * W) @ B.T
    return M * (comp[:, None] == comp[None, :])


def dense_assembly(fs, f, name):
    """Brute force: materialised lists + dense global matrix."""
    base = fs.mesh.base
    maps = verification.materialized_cell_maps(fs)   # (N2, L, k) int64
    Mref = local_mass(fs.layout, name)
    A = np.zeros((fs.total_dofs, fs.total_dofs))
    h = fs.mesh.layer_height
    for c in range(base.num_cells):
        p = base.coords[base.cell_vertices[c]]
        area2 = abs((p[1, 0] - p[0, 0]) * (p[2, 1] - p[0, 1]) -
                    (p[2, 0] - p[0, 0]) * (p[1, 1] - p[0, 1]))
        for l in range(fs.mesh.layers):
            idx = maps[c, l]
            A[np.ix_(idx, idx)] += area2 * h * Mref
    return A @ f


def main():
    g = {}
    one = mesh.BaseMesh([[0, 1, 2]], [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    two = mesh.BaseMesh([[0, 1, 2], [1, 3, 2]],
                        [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    meshes = {"one": one, "two": two}
    for n in (3, 4, 5):
        meshes[f"sq{n}"] = mesh.generate_unit_square_mesh(n)
    sq4 = meshes["sq4"]
    rcm = ordering.rcm_vertex_order(sq4)
    rnd = ordering.random_order(sq4.num_vertices, 7)
    g["sq4_rcm_forward"] = rcm.forward
    g["sq4_rnd7_forward"] = rnd.forward
    meshes["sq4rcm"] = ordering.apply_ordering(sq4, rcm)
    meshes["sq4rnd"] = ordering.apply_ordering(sq4, rnd)
    sq3 = meshes["sq3"]
    meshes["sq3rcm"] = ordering.apply_ordering(
        sq3, ordering.rcm_vertex_order(sq3))
    # a larger mesh for RCM parity (bandwidth matters at scale)
    sq16 = mesh.generate_unit_square_mesh(16)
    g["sq16_rcm_forward"] = ordering.rcm_vertex_order(sq16).forward
    g["sq16_rnd3_forward"] = ordering.random_order(sq16.num_vertices,
                                                   3).forward

    for mname, m in meshes.items():
        g[f"mesh/{mname}/cell_vertices"] = m.cell_vertices
        g[f"mesh/{mname}/coords"] = m.coords
        g[f"mesh/{mname}/cell_edges"] = m.cell_edges
        g[f"mesh/{mname}/edge_vertices"] = m.edge_vertices
        vo, vc = m._vertex_cells
        g[f"mesh/{mname}/vertex_cells_off"] = vo
        g[f"mesh/{mname}/vertex_cells"] = vc

    for mname in ("one", "two", "sq5", "sq4rcm", "sq4rnd"):
        for layers in (1, 3, 4):
            em = extrusion.ExtrudedMesh(meshes[mname], layers)
            g[f"coords/{mname}/L{layers}"] = extrusion.extrude_coordinates(
                meshes[mname].coords, layers, em.layer_height)
            for lname, layout in LAYOUTS.items():
                fs = fspace.number_dofs(em, layout)
                key = f"fs/{mname}/L{layers}/{lname}"
                g[key + "/cell_map"] = fs.cell_map
                g[key + "/offsets"] = fs.offsets
                g[key + "/total"] = np.int64(fs.total_dofs)
                if mname in ("one", "two", "sq4rcm") and layers <= 3:
                    g[key + "/materialized"] = (
                        verification.materialized_cell_maps(fs))
                    fails = verification.check_space(em, layout)
                    assert not fails, (key, fails)

    rng = np.random.default_rng(20161604)
    for mname in ("one", "two", "sq3rcm"):
        for layers in (1, 3):
            em = extrusion.ExtrudedMesh(meshes[mname], layers)
            for lname, layout in LAYOUTS.items():
                if lname == "coords":
                    continue
                fs = fspace.number_dofs(em, layout)
                f = rng.random(fs.total_dofs)
                key = f"asm/{mname}/L{layers}/{lname}"
                g[key + "/f"] = f
                g[key + "/b"] = dense_assembly(fs, f, lname)
                g[key + "/b_one"] = dense_assembly(
                    fs, np.ones(fs.total_dofs), lname)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, "
          f"{os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
