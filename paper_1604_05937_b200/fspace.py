"""Function spaces on extruded meshes: layouts, numbering, maps, offsets.

Drop-in for reference ``prismesh.fspace``:

* ``DofLayout`` / ``builtin_layout`` / ``all_builtin_layouts`` /
  ``COORDS_LAYOUT``                        -- ``fspace.py:23-84``
* ``Slot`` / ``slot_table``                -- ``fspace.py:87-131``
* ``FunctionSpace`` / ``number_dofs``      -- ``fspace.py:134-189``
  (Algorithm 1, ``PAPER.md:432-459``, in closed form)
* ``build_cell_map``                       -- ``fspace.py:192-215``
* ``compute_offsets``                      -- ``fspace.py:218-229``
  (Algorithm 2, ``PAPER.md:530-544``)
* ``dofs_at_layer``                        -- ``fspace.py:232-237``
  (the n-th layer formula, ``PAPER.md:546-553``)

Numbering: base entities in order (vertices, edges, cells); column
``(d, i)`` owns ``layers*(delta(d,0)+delta(d,1)) + delta(d,0)`` consecutive
numbers starting at ``start_d + column_d * i``.

The bottom-layer map and the offsets are generated ON THE DEVICE by the K0
kernel (``pm_build_cell_map``); ``cell_map``/``offsets`` return host copies
for API compatibility, ``device_cell_map()``/``device_offsets()`` return the
resident CUDA tensors the column loop uses.  The int32 map wraps past
2**31-1 exactly like the reference (``fspace.py:203,214``); the column loop
refuses such spaces.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .extrusion import ExtrudedEntityType, ExtrudedMesh
from .mesh import EntityId

_BUILTIN = {
    ("CG1", "CG1"): {(0, 0): 1},
    ("CG1", "DG0"): {(0, 1): 1},
    ("CG1", "DG1"): {(0, 1): 2},
    ("DG0", "CG1"): {(2, 0): 1},
    ("DG0", "DG0"): {(2, 1): 1},
    ("DG0", "DG1"): {(2, 1): 2},
    ("DG1", "CG1"): {(2, 0): 3},
    ("DG1", "DG0"): {(2, 1): 3},
    ("DG1", "DG1"): {(2, 1): 6},
}

ELEMENT_LABELS = ("CG1", "DG0", "DG1")

INT32_MAX = 2**31 - 1


@dataclass(frozen=True)
class DofLayout:
    """DoF count per extruded entity type ``(d1, d2)``."""

    name: str
    counts: dict

    def __post_init__(self):
        kept = {}
        for key, n in self.counts.items():
            t = key if isinstance(key, tuple) else (key.horiz_dim,
                                                    key.vert_dim)
            ExtrudedEntityType(*t)
            if n < 0:
                raise ValueError(f"negative DoF count for entity type {t}")
            if n:
                kept[tuple(t)] = int(n)
        if not kept:
            raise ValueError("layout assigns no DoFs at all")
        object.__setattr__(self, "counts", kept)

    def dofs(self, d1: int, d2: int) -> int:
        return self.counts.get((d1, d2), 0)

    def column_dofs(self, d: int, layers: int) -> int:
        """DoFs owned by one column over a dimension-``d`` base entity."""
        return layers * (self.dofs(d, 0) + self.dofs(d, 1)) + self.dofs(d, 0)

    def delta6(self):
        """``delta`` as the flat int32[6] the C ABI takes (index 2*d1+d2)."""
        return np.array([self.dofs(d1, d2) for d1 in (0, 1, 2)
                         for d2 in (0, 1)], dtype=np.int32)


def builtin_layout(horiz: str, vert: str) -> DofLayout:
    """One of the nine CG1/DG0/DG1 tensor-product layouts."""
    if (horiz, vert) not in _BUILTIN:
        raise ValueError(
            f"unknown discretisation {horiz!r} x {vert!r}; "
            f"labels are {ELEMENT_LABELS}")
    return DofLayout(name=f"{horiz}x{vert}", counts=dict(_BUILTIN[(horiz,
                                                                   vert)]))


def all_builtin_layouts():
    return tuple(builtin_layout(h, v) for h in ELEMENT_LABELS
                 for v in ELEMENT_LABELS)


#: The extruded coordinate field: a 3-vector at every vertex.
COORDS_LAYOUT = DofLayout(name="coords", counts={(0, 0): 3})

#: P2 x P2 (the BASELINE config-3 space): one DoF on every vertex, vertical
#: edge, horizontal edge and vertical quad facet.
P2_LAYOUT = DofLayout(name="P2xP2",
                      counts={(0, 0): 1, (0, 1): 1, (1, 0): 1, (1, 1): 1})

#: 3-component vector P1 x P1 (BASELINE config 5b).
VP1_LAYOUT = DofLayout(name="VP1xP1", counts={(0, 0): 3})


@dataclass(frozen=True)
class Slot:
    """One entry of a cell stencil's bottom-layer DoF list.

    ``kind``: local entity family (0 vertices, 1 edges, 2 the cell);
    ``local``: index in the family; ``base_dim``: base dimension;
    ``level_kind``: 0 level copy at the stencil layer, 1 connecting
    entity, 2 level copy one layer up; ``dof``: index within the entity.
    """

    kind: int
    local: int
    base_dim: int
    level_kind: int
    dof: int

    @property
    def entity_type(self) -> ExtrudedEntityType:
        return ExtrudedEntityType(self.base_dim,
                                  1 if self.level_kind == 1 else 0)

    def within(self, layout: DofLayout) -> int:
        """Offset of this slot's DoF inside its column's layer block."""
        lo, conn = layout.dofs(self.base_dim, 0), layout.dofs(self.base_dim, 1)
        return self.dof + (0, lo, lo + conn)[self.level_kind]


def slot_table(layout: DofLayout):
    """Fixed stencil slot order: vertices 0-2, edges 0-2, cell; within an
    entity bottom copy, connecting entity, top copy; within a copy, DoF."""
    out = []
    for kind, n_local in ((0, 3), (1, 3), (2, 1)):
        d = kind
        lo, conn = layout.dofs(d, 0), layout.dofs(d, 1)
        if lo == 0 and conn == 0:
            continue
        for local in range(n_local):
            for level_kind, count in ((0, lo), (1, conn), (2, lo)):
                out.extend(Slot(kind, local, d, level_kind, j)
                           for j in range(count))
    return tuple(out)


class FunctionSpace:
    """A layout bound to an extruded mesh: numbering, maps and offsets."""

    def __init__(self, mesh: ExtrudedMesh, layout: DofLayout):
        self.mesh = mesh
        self.layout = layout
        base = mesh.base
        self._column = tuple(layout.column_dofs(d, mesh.layers)
                             for d in (0, 1, 2))
        starts, acc = [], 0
        for d in (0, 1, 2):
            starts.append(acc)
            acc += self._column[d] * base.entity_count(d)
        self._starts = tuple(starts)
        self.total_dofs = acc
        self._device_cache = {}

    # -- numbering --------------------------------------------------------
    def dof_origin(self, entity: EntityId) -> int:
        """First global DoF of the entity's column (closed form)."""
        d, i = entity.dim, entity.index
        if not 0 <= i < self.mesh.base.entity_count(d):
            raise IndexError(f"entity {entity} out of range")
        return self._starts[d] + self._column[d] * i

    def dof_origin_index(self, d: int, i: int) -> int:
        return self.dof_origin(EntityId(d, i))

    @property
    def origin_starts(self):
        return self._starts

    @property
    def column_sizes(self):
        return self._column

    # -- stencil ------------------------------------------------------------
    @cached_property
    def slots(self):
        return slot_table(self.layout)

    @property
    def num_slots(self) -> int:
        return len(self.slots)

    @cached_property
    def slot_types(self):
        return tuple(s.entity_type for s in self.slots)

    @property
    def fits_int32(self) -> bool:
        return self.total_dofs <= INT32_MAX

    def device_cell_map(self):
        """(N2, k) int32 CUDA tensor built by the K0 kernel (cached)."""
        if "map" not in self._device_cache:
            from . import _lib
            cmap, offs = _lib.build_cell_map_device(self)
            self._device_cache["map"] = cmap
            self._device_cache["offsets"] = offs
        return self._device_cache["map"]

    def device_offsets(self):
        """(k,) int32 CUDA tensor of per-slot vertical offsets (K0)."""
        self.device_cell_map()
        return self._device_cache["offsets"]

    @property
    def cell_map(self):
        """Host copy of the device-built bottom-layer map (int32 (N2,k))."""
        if "host_map" not in self._device_cache:
            self._device_cache["host_map"] = (
                self.device_cell_map().cpu().numpy())
        return self._device_cache["host_map"]

    @property
    def offsets(self):
        if "host_offsets" not in self._device_cache:
            self._device_cache["host_offsets"] = (
                self.device_offsets().cpu().numpy())
        return self._device_cache["host_offsets"]

    def __repr__(self):
        return (f"FunctionSpace({self.layout.name}, "
                f"layers={self.mesh.layers}, total_dofs={self.total_dofs})")


def number_dofs(mesh: ExtrudedMesh, layout: DofLayout) -> FunctionSpace:
    """Global column-innermost numbering of ``layout`` over ``mesh``."""
    return FunctionSpace(mesh, layout)


def build_cell_map(fs: FunctionSpace):
    """Bottom-layer explicit DoF list per base cell (int32 ``(N2, k)``)."""
    return fs.cell_map


def compute_offsets(fs: FunctionSpace):
    """Per-slot vertical offset ``delta(d,0)+delta(d,1)`` (int32 ``(k,)``)."""
    return fs.offsets


def dofs_at_layer(fs: FunctionSpace, cell: int, n: int):
    """DoF list of the stencil's ``n``-th application up ``cell``'s column."""
    if not 0 <= n < fs.mesh.layers:
        raise ValueError(
            f"layer index {n} out of range for {fs.mesh.layers} layers")
    return fs.cell_map[cell].astype(np.int64) + n * fs.offsets.astype(np.int64)
