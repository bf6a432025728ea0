"""Device base-mesh pipeline (csrc/mesh_pipeline.cu)
against the host restatement: bit-exact edges, cell_edges, re-sorted cells,
and the same topology errors."""
import numpy as np
import pytest

from paper_1604_05937_b200 import mesh as M
from paper_1604_05937_b200.mesh import (BaseMesh, MeshTopologyError,
                                        derive_edges,
                                        generate_unit_square_mesh)
from paper_1604_05937_b200.ordering import (apply_ordering, random_order,
                                            rcm_vertex_order)

pytestmark = pytest.mark.gpu


def _random_mesh(n, seed):
    m = generate_unit_square_mesh(n)
    p = random_order(m.num_vertices, seed)
    return apply_ordering(m, p)


@pytest.mark.parametrize("n,seed", [(1, 0), (3, 1), (17, 2), (64, 3)])
def test_derive_edges_bit_exact(n, seed):
    m = _random_mesh(n, seed)
    cells = np.asarray(m.cell_vertices)
    # shuffle rows and rotate vertices so the input is not pre-sorted
    rng = np.random.default_rng(seed)
    cells = cells[rng.permutation(cells.shape[0])]
    cells = np.roll(cells, seed % 3, axis=1)
    ev_h, ce_h = derive_edges(cells, m.num_vertices, device=False)
    ev_d, ce_d = derive_edges(cells, m.num_vertices, device=True)
    assert ev_d.dtype == ev_h.dtype == np.int32
    assert np.array_equal(ev_d, ev_h)
    assert np.array_equal(ce_d, ce_h)


def test_derive_edges_large_default_is_device():
    m = generate_unit_square_mesh(256)            # 131072 cells -> device
    assert M.device_mesh_ok(m.num_cells)
    ev_h, ce_h = derive_edges(np.asarray(m.cell_vertices), m.num_vertices,
                              device=False)
    assert np.array_equal(m.edge_vertices, ev_h)
    assert np.array_equal(m.cell_edges, ce_h)


@pytest.mark.parametrize("cells,nv,msg", [
    ([[0, 1, 2], [1, 1, 2]], 3, "repeated vertices"),
    ([[0, 1, 2], [2, 1, 0]], 3, "duplicate cell"),
    ([[0, 1, 2], [0, 1, 3], [0, 1, 4]], 5, "shared by more than two"),
    ([[0, 1, 5]], 3, "out of range"),
    ([[0, -1, 2]], 3, "negative"),
])
def test_device_errors_match_host(cells, nv, msg):
    with pytest.raises(MeshTopologyError, match=msg):
        derive_edges(np.asarray(cells), nv, device=True)
    with pytest.raises(MeshTopologyError, match=msg):
        derive_edges(np.asarray(cells), nv, device=False)


@pytest.mark.parametrize("ordering", ["rcm", "random"])
def test_apply_ordering_device_matches_host(ordering, monkeypatch):
    m = generate_unit_square_mesh(200)            # 80000 cells -> device
    p = rcm_vertex_order(m) if ordering == "rcm" else \
        random_order(m.num_vertices, 7)
    dev = apply_ordering(m, p)
    monkeypatch.setenv("PM_DEVICE_MESH", "0")
    host = apply_ordering(m, p)
    for a in ("cell_vertices", "coords", "edge_vertices", "cell_edges"):
        assert np.array_equal(getattr(dev, a), getattr(host, a)), a
