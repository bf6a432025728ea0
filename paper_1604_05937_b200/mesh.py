"""Base (2D, triangle) meshes for the extruded-mesh column loop.

Host-side setup only: the column loop consumes ``cell_vertices``,
``cell_edges`` and ``coords`` (and, for the patch schedule, the
vertex->cell incidence).  API and numbering rules follow the reference
``prismesh.mesh`` module:

* ``derive_edges``            -- reference ``mesh.py:33-84``
* ``BaseMesh``                -- reference ``mesh.py:92-181``
* ``adjacency``               -- reference ``mesh.py:184-225``
* ``generate_unit_square_mesh`` -- reference ``mesh.py:228-254``

Edges are numbered lexicographically by their sorted vertex pair and
``cell_edges[c, k]`` is the edge opposite local vertex ``k``.  The
implementation here sorts packed 64-bit ``(min << 32) | max`` keys instead
of doing row-wise ``unique(axis=0)``; the resulting numbering is identical
(the packed key order *is* the lexicographic pair order).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np


class MeshFormatError(ValueError):
    """A mesh file does not parse under its declared format."""


class MeshTopologyError(ValueError):
    """Connectivity input violates the triangle-mesh contract."""


@dataclass(frozen=True)
class EntityId:
    """A base-mesh entity: topological dimension and index."""

    dim: int
    index: int


def _pair_keys(lo, hi):
    return (lo.astype(np.int64) << 32) | hi.astype(np.int64)


# Meshes with at least this many cells derive their edges on the GPU when
# one is present (csrc/mesh_pipeline.cu; PM_DEVICE_MESH=0 disables).
DEVICE_MESH_MIN_CELLS = 1 << 16


def device_mesh_ok(n_cells: int) -> bool:
    """Use the device mesh pipeline for a mesh of ``n_cells`` cells?"""
    import os
    if n_cells < DEVICE_MESH_MIN_CELLS or \
            os.environ.get("PM_DEVICE_MESH", "1") == "0":
        return False
    try:
        import torch
        if not torch.cuda.is_available():
            return False
        from . import _lib
        _lib.host_lib()
    except Exception:
        return False
    return True


def derive_edges(cell_vertices, num_vertices=None, device=None):
    """Edge set and cell->edge incidence of a triangle mesh.

    Returns ``(edge_vertices int32 (E,2), cell_edges int32 (C,3))``; see
    reference ``mesh.py:33-84`` for the contract (same errors, same
    numbering).  ``device`` (default: large meshes when a GPU is present)
    runs the sort-based device pipeline (``pm_derive_edges``), bit-exact
    with the host path below; on a topology error the host path runs and
    raises the reference's message.
    """
    cells = np.asarray(cell_vertices)
    if device is None:
        device = cells.ndim == 2 and device_mesh_ok(cells.shape[0])
    if device and cells.ndim == 2 and cells.shape[1] == 3:
        from . import _lib
        ev, ce, status = _lib.derive_edges_device(cells, num_vertices)
        if not status:
            return ev, ce
    if cells.ndim != 2 or cells.shape[1] != 3:
        raise MeshTopologyError(
            f"cell_vertices must have shape (n_cells, 3), got {cells.shape}")
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    n_cells = cells.shape[0]
    if n_cells and cells.min() < 0:
        raise MeshTopologyError("negative vertex index in cell_vertices")
    top = int(cells.max()) + 1 if n_cells else 0
    if num_vertices is not None:
        if n_cells and top > num_vertices:
            raise MeshTopologyError(
                f"vertex index {top - 1} out of range for "
                f"{num_vertices} vertices")

    a, b, c = cells[:, 0], cells[:, 1], cells[:, 2]
    bad = (a == b) | (b == c) | (a == c)
    if bad.any():
        raise MeshTopologyError(
            f"cell {int(np.flatnonzero(bad)[0])} has repeated vertices")

    tri = np.sort(cells, axis=1)
    # Unique cell vertex sets: pack the sorted triple (indices < 2**21 fit
    # in one int64 word; otherwise fall back to a row sort).
    if top < (1 << 21):
        ckey = (tri[:, 0] << 42) | (tri[:, 1] << 21) | tri[:, 2]
        dup = np.unique(ckey).shape[0] != n_cells
    else:
        dup = np.unique(tri, axis=0).shape[0] != n_cells
    if dup:
        raise MeshTopologyError("duplicate cell (same vertex set)")

    # Side k is opposite local vertex k: (v1,v2), (v2,v0), (v0,v1).
    s_lo = np.concatenate([np.minimum(b, c), np.minimum(c, a), np.minimum(a, b)])
    s_hi = np.concatenate([np.maximum(b, c), np.maximum(c, a), np.maximum(a, b)])
    keys = _pair_keys(s_lo, s_hi)
    uniq, inverse, counts = np.unique(keys, return_inverse=True,
                                      return_counts=True)
    if counts.size and counts.max() > 2:
        e = int(np.argmax(counts))
        pair = (int(uniq[e] >> 32), int(uniq[e] & 0xFFFFFFFF))
        raise MeshTopologyError(f"edge {pair} shared by more than two cells")
    edge_vertices = np.empty((uniq.shape[0], 2), dtype=np.int32)
    edge_vertices[:, 0] = uniq >> 32
    edge_vertices[:, 1] = uniq & 0xFFFFFFFF
    cell_edges = np.ascontiguousarray(
        inverse.reshape(3, n_cells).T, dtype=np.int32)
    return edge_vertices, cell_edges


def _frozen(a):
    a.flags.writeable = False
    return a


def _csr(rows, values, n_rows):
    """CSR of (row -> values) with values ascending inside a row."""
    order = np.lexsort((values, rows))
    counts = np.bincount(rows, minlength=n_rows)
    offsets = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, np.ascontiguousarray(values[order], dtype=np.int32)


class BaseMesh:
    """Immutable unstructured triangle mesh (reference ``mesh.py:92-181``)."""

    def __init__(self, cell_vertices, coords):
        coords = np.asarray(coords, dtype=np.float64)
        if coords.ndim != 2 or coords.shape[1] != 2:
            raise MeshTopologyError(
                f"coords must have shape (n_vertices, 2), got {coords.shape}")
        coords = np.ascontiguousarray(coords)
        cells = np.ascontiguousarray(cell_vertices, dtype=np.int32)
        edge_vertices, cell_edges = derive_edges(cells, coords.shape[0])
        self.coords = _frozen(coords)
        self.cell_vertices = _frozen(cells)
        self.edge_vertices = _frozen(edge_vertices)
        self.cell_edges = _frozen(cell_edges)

    @property
    def num_vertices(self) -> int:
        return self.coords.shape[0]

    @property
    def num_edges(self) -> int:
        return self.edge_vertices.shape[0]

    @property
    def num_cells(self) -> int:
        return self.cell_vertices.shape[0]

    def entity_count(self, dim: int) -> int:
        return (self.num_vertices, self.num_edges, self.num_cells)[dim]

    def __repr__(self):
        return (f"BaseMesh(vertices={self.num_vertices}, "
                f"edges={self.num_edges}, cells={self.num_cells})")

    # -- incidence (CSR, rows ascending) ---------------------------------
    @cached_property
    def _edge_cells(self):
        cells = np.repeat(np.arange(self.num_cells, dtype=np.int64), 3)
        return _csr(self.cell_edges.ravel().astype(np.int64), cells,
                    self.num_edges)

    @cached_property
    def _vertex_cells(self):
        cells = np.repeat(np.arange(self.num_cells, dtype=np.int64), 3)
        return _csr(self.cell_vertices.ravel().astype(np.int64), cells,
                    self.num_vertices)

    @cached_property
    def _vertex_edges(self):
        edges = np.repeat(np.arange(self.num_edges, dtype=np.int64), 2)
        return _csr(self.edge_vertices.ravel().astype(np.int64), edges,
                    self.num_vertices)

    def vertex_neighbours(self):
        """CSR vertex-vertex adjacency through edges, rows ascending."""
        return self._vertex_vertices

    @cached_property
    def _vertex_vertices(self):
        ev = self.edge_vertices.astype(np.int64)
        src = np.concatenate([ev[:, 0], ev[:, 1]])
        dst = np.concatenate([ev[:, 1], ev[:, 0]])
        return _csr(src, dst, self.num_vertices)


def adjacency(mesh: BaseMesh, d1: int, d2: int, v: EntityId):
    """Entities of dimension ``d2`` adjacent to ``v`` (dimension ``d1``).

    Same coverage as reference ``mesh.py:184-225``; (1,1) is not derived.
    """
    if v.dim != d1:
        raise ValueError(f"entity {v} does not have dimension {d1}")
    if not 0 <= v.index < mesh.entity_count(d1):
        raise ValueError(f"entity index {v.index} out of range for dim {d1}")
    i = v.index
    direct = {(2, 0): mesh.cell_vertices, (2, 1): mesh.cell_edges,
              (1, 0): mesh.edge_vertices}
    csr = {(1, 2): "_edge_cells", (0, 2): "_vertex_cells",
           (0, 1): "_vertex_edges", (0, 0): "_vertex_vertices"}
    if (d1, d2) in direct:
        ids = direct[(d1, d2)][i]
    elif (d1, d2) in csr:
        off, val = getattr(mesh, csr[(d1, d2)])
        ids = val[off[i]:off[i + 1]]
    elif (d1, d2) == (2, 2):
        off, val = mesh._edge_cells
        ids = [c for e in mesh.cell_edges[i]
               for c in val[off[e]:off[e + 1]] if c != i]
    else:
        raise NotImplementedError(
            f"adjacency ({d1},{d2}) not derived in this build")
    return tuple(EntityId(d2, int(j)) for j in ids)


def generate_unit_square_mesh(n: int) -> BaseMesh:
    """Split-square triangulation of the unit square (``2 n^2`` cells).

    Vertex ``i*(n+1)+j`` sits at ``(i/n, j/n)``; the ``n^2`` cells
    ``[v00, v10, v11]`` come first, then ``[v00, v11, v01]``
    (reference ``mesh.py:228-254``).
    """
    if n < 1:
        raise ValueError(f"subdivision count must be >= 1, got {n}")
    m = n + 1
    t = np.arange(m) / n
    coords = np.empty((m * m, 2))
    coords[:, 0] = np.repeat(t, m)
    coords[:, 1] = np.tile(t, m)
    i = np.repeat(np.arange(n, dtype=np.int64), n)
    j = np.tile(np.arange(n, dtype=np.int64), n)
    v00 = i * m + j
    v10 = v00 + m
    v01 = v00 + 1
    v11 = v10 + 1
    cells = np.concatenate([np.stack([v00, v10, v11], axis=1),
                            np.stack([v00, v11, v01], axis=1)])
    mesh = BaseMesh(cells, coords)
    assert mesh.num_vertices - mesh.num_edges + mesh.num_cells == 1
    return mesh
