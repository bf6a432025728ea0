"""prismesh-b200: the extruded-mesh column loop of Bercea et al. (2016),
arXiv:1604.05937, rebuilt for NVIDIA B200 (sm_100a).

Host-side mirror of the reference ``prismesh`` API (mesh, ordering,
extrusion, fspace) plus the SPEC's par-loop entry points (iterate,
kernels), backed by hand-written CUDA kernels in ``csrc/`` behind the C ABI
``include/prismesh_cuda.h``.
"""
from .extrusion import (ENTITY_TYPES, ExtrudedEntityType, ExtrudedMesh,
                        entity_count, extrude_coordinates)
from .fspace import (COORDS_LAYOUT, P2_LAYOUT, VP1_LAYOUT, DofLayout,
                     FunctionSpace, Slot, all_builtin_layouts,
                     build_cell_map, builtin_layout, compute_offsets,
                     dofs_at_layer, number_dofs, slot_table)
from .mesh import (BaseMesh, EntityId, MeshFormatError, MeshTopologyError,
                   adjacency, derive_edges, generate_unit_square_mesh)
from .ordering import (Permutation, apply_ordering, random_order, rcm_order,
                       rcm_vertex_order)
from .quadrature import (PrismElement, QuadratureRule, element_for_layout,
                         prism_quadrature, reference_mass_matrix)

__version__ = "0.1.0"
