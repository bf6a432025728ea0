"""Slow-path baselines for the numbering, the addressing and the loop.

Mirrors the reference's ``verification`` module (``verification.py:18-158``:
``number_dofs_literal``, ``materialized_cell_maps``, ``check_space``,
``run_oracle_suite``) and adds the B200 checks the ``verify`` CLI runs
when a GPU is present: the device-built maps (K0), the per-(cell, layer)
lists the device column loop itself addresses (``ListProbeKernel``) and
the device assembly against a dense host assembler over the materialised
lists.  Everything here is a checker; the product path never calls it.
"""
from __future__ import annotations

import numpy as np

from .extrusion import ExtrudedMesh
from .fspace import (COORDS_LAYOUT, DofLayout, FunctionSpace,
                     all_builtin_layouts, number_dofs)
from .mesh import BaseMesh, generate_unit_square_mesh


def number_dofs_literal(mesh: ExtrudedMesh, layout: DofLayout):
    """Alg. 1 as a literal counter (reference ``verification.py:18-44``).

    Entities are visited vertices → edges → cells in index order; inside
    a column the level copy of layer l, then the connecting entity of
    layer l, and the top level copy last.  Returns ``(assignment, total)``
    with ``assignment[((d1, d2), (i, l))]`` = tuple of global numbers.
    """
    out = {}
    n = 0
    lam = mesh.layers
    for d in (0, 1, 2):
        nl, nc = layout.dofs(d, 0), layout.dofs(d, 1)
        for i in range(mesh.base.entity_count(d)):
            for l in range(lam + 1):
                out[((d, 0), (i, l))] = tuple(range(n, n + nl))
                n += nl
                if l < lam:
                    out[((d, 1), (i, l))] = tuple(range(n, n + nc))
                    n += nc
    return out, n


def materialized_cell_maps(fs: FunctionSpace) -> np.ndarray:
    """Explicit (N2, λ, k) int64 DoF lists read from the literal numbering
    (reference ``verification.py:47-75``)."""
    mesh = fs.mesh
    base = mesh.base
    assignment, total = number_dofs_literal(mesh, fs.layout)
    if total != fs.total_dofs:
        raise AssertionError(
            f"literal numbering total {total} != {fs.total_dofs}")
    local = (np.asarray(base.cell_vertices), np.asarray(base.cell_edges),
             np.arange(base.num_cells)[:, None])
    out = np.empty((base.num_cells, mesh.layers, fs.num_slots), np.int64)
    for j, s in enumerate(fs.slots):
        ents = local[s.kind][:, s.local]
        for c in range(base.num_cells):
            i = int(ents[c])
            for l in range(mesh.layers):
                if s.level_kind == 1:
                    key = ((s.base_dim, 1), (i, l))
                else:
                    key = ((s.base_dim, 0), (i, l + (s.level_kind == 2)))
                out[c, l, j] = assignment[key][s.dof]
    return out


def check_space(mesh: ExtrudedMesh, layout: DofLayout, device=False):
    """Cross-check one space against the literal baseline (reference
    ``verification.py:78-126``): bijection onto 0..total-1, the closed-form
    total and column origins, vertical stride δ(d,0)+δ(d,1), and bottom map
    + l·offsets == every materialised list (the device K0 maps with
    ``device``, else their host closed form).  Returns failure strings."""
    fails = []
    fs = number_dofs(mesh, layout)
    assignment, total = number_dofs_literal(mesh, layout)
    if total != fs.total_dofs:
        fails.append(f"total mismatch: literal {total}, closed form "
                     f"{fs.total_dofs}")
    nums = np.sort(np.fromiter((n for t in assignment.values() for n in t),
                               dtype=np.int64))
    if not np.array_equal(nums, np.arange(total)):
        fails.append("assigned numbers are not exactly 0..total-1")
    lam = mesh.layers
    for d in (0, 1, 2):
        stride = layout.dofs(d, 0) + layout.dofs(d, 1)
        for i in range(mesh.base.entity_count(d)):
            first = assignment[((d, 0), (i, 0))] or \
                assignment.get(((d, 1), (i, 0)), ())
            if first and fs.dof_origin_index(d, i) != first[0]:
                fails.append(f"column origin mismatch at ({d},{i})")
            for d2, top in ((0, lam), (1, lam - 1)):
                for l in range(top):
                    lo = assignment[((d, d2), (i, l))]
                    hi = assignment[((d, d2), (i, l + 1))]
                    if any(b - a != stride for a, b in zip(lo, hi)):
                        fails.append(f"vertical stride at ({d},{d2}) "
                                     f"column {i} layer {l}")
                        break
    maps = materialized_cell_maps(fs)
    if device:
        bottom = np.asarray(fs.cell_map, dtype=np.int64)   # K0, device
        offs = np.asarray(fs.offsets, dtype=np.int64)
    else:
        bottom, offs = closed_form_maps(fs)
    for l in range(lam):
        if not np.array_equal(maps[:, l, :], bottom + l * offs):
            fails.append(f"offset addressing differs at layer {l}")
    return fails


def closed_form_maps(fs: FunctionSpace):
    """Host statement of the bottom map (origin + within, fspace.py
    ``build_cell_map``) and Alg. 2 offsets, int64, no int32 wrap: what
    ``check_space`` compares the literal lists with when there is no GPU
    (the production maps are built on the device by K0)."""
    base = fs.mesh.base
    local = (np.asarray(base.cell_vertices, np.int64),
             np.asarray(base.cell_edges, np.int64),
             np.arange(base.num_cells, dtype=np.int64)[:, None])
    layout = fs.layout
    cols = []
    offs = []
    for s in fs.slots:
        d = s.base_dim
        cols.append(fs.origin_starts[d] + fs.column_sizes[d] *
                    local[s.kind][:, s.local] + s.within(layout))
        offs.append(layout.dofs(d, 0) + layout.dofs(d, 1))
    return np.stack(cols, axis=1), np.asarray(offs, dtype=np.int64)


def dense_mass_action(fs: FunctionSpace, x, coords, mref) -> np.ndarray:
    """``y = Σ_{c,l} scatter(|det J| · Mref · x[list(c,l)])`` over the
    materialised lists of ``fs`` and of the coordinate space: the loop
    with no offset arithmetic, no schedule and no sum factorisation."""
    mesh = fs.mesh
    maps = materialized_cell_maps(fs)
    cmaps = materialized_cell_maps(number_dofs(mesh, COORDS_LAYOUT))
    coords = np.asarray(coords, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    # coordinate slot 6a + 3b + comp: vertex a, level b, component comp
    P = coords[cmaps].reshape(cmaps.shape[0], cmaps.shape[1], 3, 2, 3)
    xm = 0.5 * (P[..., 0, 0] + P[..., 1, 0])
    ym = 0.5 * (P[..., 0, 1] + P[..., 1, 1])
    a2 = ((xm[..., 1] - xm[..., 0]) * (ym[..., 2] - ym[..., 0]) -
          (xm[..., 2] - xm[..., 0]) * (ym[..., 1] - ym[..., 0]))
    dz = P[..., 1, 2] - P[..., 0, 2]
    h = (dz[..., 0] + dz[..., 1] + dz[..., 2]) / 3.0
    det = np.abs(a2 * h)
    local = np.einsum("ij,clj->cli", np.asarray(mref), x[maps]) * det[..., None]
    y = np.zeros(fs.total_dofs)
    np.add.at(y, maps.ravel(), local.ravel())
    return y


def _fixture_meshes():
    one = BaseMesh([[0, 1, 2]], [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    two = BaseMesh([[0, 1, 2], [1, 3, 2]],
                   [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    return (("single-triangle", one), ("two-triangle", two),
            ("unit-square-5", generate_unit_square_mesh(5)))


def check_device(mesh: ExtrudedMesh, layout: DofLayout, seed: int = 0):
    """The B200 path against the baselines: K0 maps, the loop's own
    per-(cell, layer) lists and the assembled field (≤ 1e-13 relative to
    max |y|).  Needs a GPU.  Returns failure strings."""
    import torch
    from . import kernels
    fails = []
    fs = number_dofs(mesh, layout)
    if not np.array_equal(fs.device_cell_map().cpu().numpy(),
                          np.asarray(fs.cell_map)):
        fails.append("device cell map differs")
    maps = materialized_cell_maps(fs)
    dev = torch.device("cuda")
    probe = torch.empty(maps.shape, dtype=torch.int64, device=dev)
    from .iterate import iterate_columns
    iterate_columns([fs], kernels.ListProbeKernel(fs), [probe])
    if not np.array_equal(probe.cpu().numpy(), maps):
        fails.append("device loop addresses differ from the literal lists")
    from .extrusion import extrude_coordinates
    m = fs.mesh
    coords = np.asarray(extrude_coordinates(m.base.coords, m.layers,
                                            m.layer_height).cpu())
    x = np.random.default_rng(seed).random(fs.total_dofs)
    op = kernels.MassOperator(fs)
    y = kernels.mass_action(fs, x, coords, operator=op)
    ref = dense_mass_action(fs, x, coords, op.mref)
    scale = max(1.0, float(np.abs(ref).max()))
    err = float(np.abs(np.asarray(y) - ref).max()) / scale
    if not err <= 1e-13:
        fails.append(f"device assembly differs from the dense assembler "
                     f"({err:.2e})")
    return fails


def run_oracle_suite(layers: int = 4, report=print, device=None) -> bool:
    """All nine layouts × the three fixture meshes (reference
    ``verification.py:138-158``); with ``device`` (default: when CUDA is
    available) also the B200 maps, loop lists and assembly."""
    if device is None:
        try:
            import torch
            device = torch.cuda.is_available()
        except ImportError:
            device = False
    layouts = all_builtin_layouts()
    meshes = _fixture_meshes()
    passed, total = 0, len(layouts) * len(meshes)
    for name, base in meshes:
        mesh = ExtrudedMesh(base, layers)
        for layout in layouts:
            fails = check_space(mesh, layout, device=device)
            if device:
                fails += check_device(mesh, layout)
            for f in fails:
                report(f"FAIL {layout.name} on {name}: {f}")
            passed += not fails
    where = "host + device" if device else "host"
    report(f"{passed}/{total} layout-mesh-layers oracle checks passed "
           f"({where})")
    return passed == total
