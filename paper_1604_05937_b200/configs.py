"""BASELINE.json workload presets (synthetic stand-ins for the paper's
Gmsh meshes, which are not available): split-square base meshes
(``generate_unit_square_mesh``), RCM- or seeded-random-ordered
(``ordering.py``), optional interior-vertex jitter, uniform extrusion on
z in [0,1], seeded field values drawn in DoF order.

Draw order per seed: ``rng = default_rng(seed)``; jitter
first (config 4 only), then the input field.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .extrusion import ExtrudedMesh
from .fspace import P2_LAYOUT, VP1_LAYOUT, builtin_layout, number_dofs
from .mesh import BaseMesh, generate_unit_square_mesh
from .ordering import apply_ordering, random_order, rcm_vertex_order
from .quadrature import prism_quadrature


@dataclass(frozen=True)
class Workload:
    name: str
    n: int                  # split-square subdivisions
    layers: int
    layout: str             # "CG1xCG1" | "DG1xDG1" | "P2xP2" | "VP1"
    quad: tuple = (2, 2)    # (triangle degree, line degree)
    ordering: str = "rcm"   # "rcm" | "random"
    jitter: float = 0.0     # fraction of h, interior vertices only
    values: str = "u01"     # "u01": U[0,1), "u11": U[-1,1)
    seed: int = 0
    note: str = field(default="", compare=False)


WORKLOADS = {
    "C1": Workload("C1", 64, 10, "CG1xCG1", (4, 4), note="P1 CG RHS, 64^2, 10 layers"),
    "C2": Workload("C2", 256, 50, "DG1xDG1", (2, 2), values="u11",
                   note="DG1 mass action, 256^2, 50 layers"),
    "C3": Workload("C3", 512, 100, "P2xP2", (6, 6), note="P2 CG RHS, 512^2, 100 layers"),
    "C5a": Workload("C5a", 2048, 64, "CG1xCG1", (4, 4), note="P1 CG RHS, 2048^2, 64 layers"),
    "C5b": Workload("C5b", 2048, 64, "VP1", (2, 2), note="3-vector P1 mass, 2048^2, 64 layers"),
}

SWEEP_LAYERS = (1, 2, 5, 10, 20, 50, 100, 256)


def sweep_workload(layout: str, layers: int, ordering: str) -> Workload:
    """BASELINE config 4: 256^2 base, jitter +-0.3h."""
    return Workload(f"C4-{layout}-{ordering}-L{layers}", 256, layers, layout,
                    (2, 2), ordering, 0.3,
                    "u11" if layout.startswith("DG") else "u01")


def layout_of(name: str):
    if name == "P2xP2":
        return P2_LAYOUT
    if name == "VP1":
        return VP1_LAYOUT
    h, v = name.split("x")
    return builtin_layout(h, v)


_BASE_CACHE = {}


def base_mesh(n: int, ordering: str = "rcm", jitter: float = 0.0,
              seed: int = 0):
    """(BaseMesh, rng) -- rng is positioned after the jitter draws."""
    rng = np.random.default_rng(seed)
    nv = (n + 1) ** 2
    d = rng.uniform(-jitter / n, jitter / n, size=(nv, 2)) if jitter else None
    key = (n, ordering, jitter, seed)
    if key in _BASE_CACHE:
        return _BASE_CACHE[key], rng
    m = generate_unit_square_mesh(n)
    if jitter:
        coords = m.coords.copy()
        interior = ((coords[:, 0] > 0) & (coords[:, 0] < 1) &
                    (coords[:, 1] > 0) & (coords[:, 1] < 1))
        coords[interior] += d[interior]
        m = BaseMesh(m.cell_vertices, coords)
    if ordering == "rcm":
        m = apply_ordering(m, rcm_vertex_order(m))
    elif ordering == "random":
        m = apply_ordering(m, random_order(m.num_vertices, seed))
    elif ordering != "natural":
        raise ValueError(f"unknown ordering {ordering!r}")
    _BASE_CACHE[key] = m
    return m, rng


def build(w: Workload):
    """(fs, quadrature, x numpy, rng) for a workload."""
    base, rng = base_mesh(w.n, w.ordering, w.jitter, w.seed)
    mesh = ExtrudedMesh(base, w.layers)
    fs = number_dofs(mesh, layout_of(w.layout))
    if w.values == "u01":
        x = rng.random(fs.total_dofs)
    else:
        x = rng.uniform(-1.0, 1.0, fs.total_dofs)
    return fs, prism_quadrature(*w.quad), x, rng


def workload(name: str) -> Workload:
    """``C1``..``C5b`` or a config-4 sweep point ``C4-<layout>-<ordering>-L<n>``
    (e.g. ``C4-CG1xCG1-rcm-L50``)."""
    if name in WORKLOADS:
        return WORKLOADS[name]
    parts = name.split("-")
    if len(parts) == 4 and parts[0] == "C4" and parts[3].startswith("L"):
        return sweep_workload(parts[1], int(parts[3][1:]), parts[2])
    raise ValueError(f"unknown workload {name!r}")
