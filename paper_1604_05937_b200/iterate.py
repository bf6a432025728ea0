"""Algorithm 3 -- the column par-loop -- on the GPU.

Drop-in for the SPEC's ``iterate`` module (PAPER.md
Alg. 3 :567-587):

* ``iterate_columns(fs_list, kernel, fields, schedule)``
* ``color_base_cells(mesh) -> Coloring``

For every base cell the device kernel loads the bottom-layer lists of each
argument space once, then walks up the column adding the per-slot offsets
(``dof_j = L_j + l*offset_j``).  Output is accumulated ``+=`` into the
output field.  Kernels are the device kernels of
``kernels.py``; arbitrary Python callables are not supported (there is no
CPU execution path).

Schedules (``schedule=``):

``"auto"``      DG (2,1) fields in overwrite mode: ``"stream"``; CG
                fields on vertex (P1, 3-vector P1, CG1xDGk) or vertex + edge
                (P2) columns: ``"stripred"``; otherwise ``"column"``.
``"patch"``     owner-computes over compact patches, shared-memory
                accumulation, no atomics, deterministic (schedule.py).
``"stripred"``  vertex-column layouts: global sequential strips, one
                vertex load and one fp64 REDG flush per cell.
``"strip"``     vertex-column layouts: patches staged in shared memory,
                cells walked as strips (one new vertex per cell), owner
                gather of per-residency partials; deterministic.
``"stream"``    DG (2,1) fields through TMA bulk copies (dg_stream.cu).
``"column"``    warp segment per column, lanes = layers; vertical sharing
                in registers, column-shared DoFs via fp64 REDG.
``"atomic"``    one thread per cell-layer, shared DoFs via fp64 REDG.
``"colored"``   ``"column"`` once per colour of ``color_base_cells`` with
                plain read-add-stores: bitwise deterministic
                (SPEC.md:358-364).
``"sequential"`` alias of ``"colored"`` (the deterministic schedule).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

SCHEDULES = ("auto", "atomic", "colored", "sequential", "column", "stream",
             "patch", "strip", "stripred", "striptma", "pstrip", "stripdg",
             "tile")


@dataclass(frozen=True)
class Coloring:
    """Per-base-cell colour id; cells sharing a vertex differ."""

    color_of: np.ndarray
    num_colors: int

    def cells_by_color(self):
        """(order, ptr): cells grouped by colour, each group ascending."""
        order = np.argsort(self.color_of, kind="stable").astype(np.int32)
        counts = np.bincount(self.color_of, minlength=self.num_colors)
        ptr = np.zeros(self.num_colors + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        return order, ptr


def color_base_cells(mesh) -> Coloring:
    """Greedy colouring of base cells over "shares a vertex" (host)."""
    base = getattr(mesh, "base", mesh)
    n_cells = base.num_cells
    if n_cells == 0:
        return Coloring(np.zeros(0, dtype=np.int32), 0)
    off, cells = _vertex_cells(base)
    color, n = _lib.greedy_color_cells(base.cell_vertices, off, cells)
    return Coloring(color, n)


def _vertex_cells(base):
    vc = getattr(base, "_vertex_cells", None)
    if vc is not None:
        return vc
    flat = np.asarray(base.cell_vertices, dtype=np.int64).ravel()
    order = np.argsort(flat, kind="stable")
    cells = np.repeat(np.arange(base.num_cells, dtype=np.int32), 3)[order]
    counts = np.bincount(flat, minlength=base.num_vertices)
    off = np.zeros(base.num_vertices + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, cells


def _check_spaces(fs_list, kernel):
    if not fs_list:
        raise ValueError("iterate_columns needs at least one space")
    mesh = fs_list[0].mesh
    for fs in fs_list[1:]:
        if fs.mesh is not mesh:
            raise ValueError("all argument spaces must share one ExtrudedMesh")
    arity = kernel.arity
    if len(arity) != len(fs_list):
        raise ValueError(f"kernel takes {len(arity)} spaces, got "
                         f"{len(fs_list)}")
    for fs, k in zip(fs_list, arity):
        if fs.num_slots != k:
            raise ValueError(
                f"kernel arity {k} != {fs.num_slots} slots of {fs.layout.name}")
        if not fs.fits_int32:
            raise ValueError(
                f"{fs!r}: {fs.total_dofs} DoFs overflow the int32 cell map")
    return mesh


def iterate_columns(fs_list, kernel, fields, schedule="auto", stream=None):
    """Apply ``kernel`` to every cell-layer of the extruded mesh.

    ``fs_list``: argument spaces in the kernel's order; ``fields``: device
    tensors (inputs..., output) -- the output receives ``+=``.
    """
    if schedule not in SCHEDULES:
        raise ValueError(f"unknown schedule {schedule!r}; one of {SCHEDULES}")
    _check_spaces(fs_list, kernel)
    kernel.launch(fs_list, fields, schedule, stream=stream)
