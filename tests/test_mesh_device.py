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


@pytest.mark.parametrize("n,seed", [(200, 0), (257, 3)])
def test_vertex_graph_sorted_matches_host(n, seed):
    from paper_1604_05937_b200 import _lib
    m = _random_mesh(n, seed)
    off_d, nb_d = _lib.vertex_graph_sorted_device(m.edge_vertices,
                                                  m.num_vertices)
    off, nb = m.vertex_neighbours()
    off = np.asarray(off, dtype=np.int64)
    deg = np.diff(off)
    rows = np.repeat(np.arange(m.num_vertices), deg)
    nb = np.asarray(nb, dtype=np.int64)
    ref = nb[np.lexsort((nb, deg[nb], rows))]
    assert np.array_equal(off_d, off)
    assert np.array_equal(nb_d, ref)


@pytest.mark.parametrize("n,seed", [(200, None), (190, 5), (300, 11)])
def test_rcm_device_graph_matches_host(n, seed, monkeypatch):
    m = generate_unit_square_mesh(n) if seed is None else _random_mesh(n, seed)
    assert M.device_mesh_ok(m.num_cells)
    dev = rcm_vertex_order(m).forward
    monkeypatch.setenv("PM_DEVICE_MESH", "0")
    host = rcm_vertex_order(m).forward
    assert np.array_equal(dev, host)


def test_rcm_device_graph_disconnected(monkeypatch):
    """Two squares side by side, no shared vertex: components in order of
    their smallest vertex, each from its min-degree vertex."""
    a = generate_unit_square_mesh(200)
    cells = np.asarray(a.cell_vertices)
    coords = np.asarray(a.coords)
    nv = coords.shape[0]
    both = BaseMesh(np.vstack([cells, cells + nv]),
                    np.vstack([coords, coords + [2.0, 0.0]]))
    dev = rcm_vertex_order(both).forward
    monkeypatch.setenv("PM_DEVICE_MESH", "0")
    host = rcm_vertex_order(both).forward
    assert np.array_equal(dev, host)


def _csr(n, pairs):
    """Symmetric CSR (offsets, neighbours) of an undirected edge list."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    a = np.concatenate([pairs[:, 0], pairs[:, 1]])
    b = np.concatenate([pairs[:, 1], pairs[:, 0]])
    o = np.lexsort((b, a))
    a, b = a[o], b[o]
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, a + 1, 1)
    return np.cumsum(off), b


@pytest.mark.parametrize("seed", range(6))
def test_rcm_device_walk_bit_exact(seed):
    """pm_rcm_order_device == the host walk (== ordering.py:45-90) on
    random graphs with several components, isolated vertices, hubs and
    degree ties."""
    from paper_1604_05937_b200.ordering import rcm_order
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 4 * n))
    pairs = rng.integers(0, n, size=(m, 2))
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    if seed % 2 and n > 10:       # a hub: one vertex adjacent to many
        hub = np.stack([np.zeros(n // 2, np.int64),
                        rng.integers(1, n, n // 2)], 1)
        pairs = np.concatenate([pairs, hub])
    pairs = np.unique(np.sort(pairs, axis=1), axis=0)
    off, nb = _csr(n, pairs)
    host = rcm_order(off, nb).forward
    dev = rcm_order(off, nb, device=True).forward
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("n,seed", [(4, None), (16, None), (64, 5),
                                    (300, 7)])
def test_rcm_vertex_order_device_matches_host(n, seed):
    """The mesh path (device graph + device walk) equals the host path."""
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.ordering import rcm_order
    m = generate_unit_square_mesh(n)
    if seed is not None:
        m = apply_ordering(m, random_order(m.num_vertices, seed))
    off, nbr = m.vertex_neighbours()
    host = rcm_order(off, nbr).forward
    dev = _lib.rcm_forward_device(m.edge_vertices, m.num_vertices)
    assert np.array_equal(host, dev)


def test_rcm_device_golden(golden):
    """Device walk against the reference's own RCM permutations."""
    from paper_1604_05937_b200 import _lib
    for name in ("sq4", "sq16"):
        key = f"{name}_rcm_forward"
        assert key in golden
        m = generate_unit_square_mesh(int(name[2:]))
        dev = _lib.rcm_forward_device(m.edge_vertices, m.num_vertices)
        assert np.array_equal(dev, golden[key])
