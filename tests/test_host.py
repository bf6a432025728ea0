"""Host-side parts of the product (setup, numbering metadata, formulas)
against the reference's golden outputs and the oracle.  CPU only."""
import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees
from paper_1604_05937_b200 import (BaseMesh, DofLayout, ExtrudedMesh,
                                   MeshTopologyError, apply_ordering,
                                   builtin_layout, derive_edges,
                                   generate_unit_square_mesh, number_dofs,
                                   random_order, rcm_vertex_order, slot_table)
from paper_1604_05937_b200 import perfbench
from paper_1604_05937_b200.kernels import count_flops
from paper_1604_05937_b200.quadrature import (element_for_layout,
                                              line_rule, prism_quadrature,
                                              reference_mass_matrix,
                                              sharing_class, triangle_rule)


def _same_mesh(m, golden, name):
    p = f"mesh/{name}/"
    np.testing.assert_array_equal(m.cell_vertices, golden[p + "cell_vertices"])
    np.testing.assert_array_equal(m.coords, golden[p + "coords"])
    np.testing.assert_array_equal(m.cell_edges, golden[p + "cell_edges"])
    np.testing.assert_array_equal(m.edge_vertices, golden[p + "edge_vertices"])
    off, cells = m._vertex_cells
    np.testing.assert_array_equal(off, golden[p + "vertex_cells_off"])
    np.testing.assert_array_equal(cells, golden[p + "vertex_cells"])


@pytest.mark.parametrize("n", (3, 4, 5))
def test_unit_square_mesh_matches_reference(golden, n):
    _same_mesh(generate_unit_square_mesh(n), golden, f"sq{n}")


def test_fixture_meshes_match_reference(golden):
    one = BaseMesh([[0, 1, 2]], [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    two = BaseMesh([[0, 1, 2], [1, 3, 2]],
                   [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    _same_mesh(one, golden, "one")
    _same_mesh(two, golden, "two")


def test_orderings_match_reference(golden):
    sq4 = generate_unit_square_mesh(4)
    rcm = rcm_vertex_order(sq4)
    np.testing.assert_array_equal(rcm.forward, golden["sq4_rcm_forward"])
    rnd = random_order(sq4.num_vertices, 7)
    np.testing.assert_array_equal(rnd.forward, golden["sq4_rnd7_forward"])
    _same_mesh(apply_ordering(sq4, rcm), golden, "sq4rcm")
    _same_mesh(apply_ordering(sq4, rnd), golden, "sq4rnd")
    sq16 = generate_unit_square_mesh(16)
    np.testing.assert_array_equal(rcm_vertex_order(sq16).forward,
                                  golden["sq16_rcm_forward"])
    np.testing.assert_array_equal(random_order(sq16.num_vertices, 3).forward,
                                  golden["sq16_rnd3_forward"])


def test_rcm_disconnected_components():
    # two disjoint triangles: components in order of smallest vertex
    m = BaseMesh([[0, 1, 2], [3, 4, 5]], np.random.default_rng(0).random((6, 2)))
    fwd = rcm_vertex_order(m).forward
    assert sorted(fwd.tolist()) == list(range(6))


def test_mesh_errors():
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1]])
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1, -1]])
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1, 1]])
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1, 2], [2, 1, 0]])
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1, 2], [0, 1, 3], [0, 1, 4]])
    with pytest.raises(MeshTopologyError):
        derive_edges([[0, 1, 5]], num_vertices=3)
    with pytest.raises(ValueError):
        generate_unit_square_mesh(0)
    with pytest.raises(ValueError):
        ExtrudedMesh(generate_unit_square_mesh(1), 0)
    with pytest.raises(ValueError):
        builtin_layout("CG2", "CG1")
    with pytest.raises(ValueError):
        DofLayout("empty", {(0, 0): 0})
    with pytest.raises(ValueError):
        DofLayout("bad", {(3, 0): 1})


@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_slot_table_matches_oracle(lname):
    counts = LAYOUT_COUNTS[lname]
    kind, local, level, dof = oracle.slot_table(counts)
    slots = slot_table(DofLayout(lname, counts))
    assert [s.kind for s in slots] == kind.tolist()
    assert [s.local for s in slots] == local.tolist()
    assert [s.level_kind for s in slots] == level.tolist()
    assert [s.dof for s in slots] == dof.tolist()


@pytest.mark.parametrize("mname", ("one", "two", "sq5", "sq4rcm"))
@pytest.mark.parametrize("layers", (1, 3, 4))
@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_numbering_closed_form(golden, gmesh, mname, layers, lname):
    fs = number_dofs(ExtrudedMesh(gmesh(mname), layers),
                     DofLayout(lname, LAYOUT_COUNTS[lname]))
    assert fs.total_dofs == int(golden[f"fs/{mname}/L{layers}/{lname}/total"])
    # dof_origin(entity) == first DoF of the column in the literal numbering
    mat = golden.get(f"fs/{mname}/L{layers}/{lname}/materialized")
    if mat is not None:
        from paper_1604_05937_b200 import EntityId
        base = gmesh(mname)
        slots = fs.slots
        for j, s in enumerate(slots):
            if s.level_kind == 0 and s.dof == 0:
                ents = (base.cell_vertices, base.cell_edges,
                        np.arange(base.num_cells)[:, None])[s.kind][:, s.local]
                for c in range(min(base.num_cells, 8)):
                    assert fs.dof_origin(EntityId(s.base_dim, int(ents[c]))) \
                        == mat[c, 0, j]


@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords"}))
def test_element_slot_basis_matches_oracle(lname):
    counts = LAYOUT_COUNTS[lname]
    tri, line, nc = families(lname)
    el = element_for_layout(DofLayout(lname, counts))
    h, v, c = oracle.slot_basis(counts, tri, line, nc)
    assert (el.tri, el.line, el.ncomp) == (tri, line, nc)
    assert list(el.slot_h) == h.tolist()
    assert list(el.slot_v) == v.tolist()
    assert list(el.slot_comp) == c.tolist()


@pytest.mark.parametrize("deg", range(0, 7))
def test_quadrature_matches_oracle(deg):
    p, w = triangle_rule(deg)
    op, ow = oracle.tri_rule(deg)
    np.testing.assert_array_equal(p, op)
    np.testing.assert_array_equal(w, ow)
    z, zw = line_rule(deg)
    oz, ozw = oracle.line_rule(deg)
    np.testing.assert_allclose(z, oz, rtol=0, atol=5e-16)
    np.testing.assert_allclose(zw, ozw, rtol=0, atol=5e-16)


def test_prism_quadrature_spec_examples():
    q = prism_quadrature()
    assert q.num_points == 6 and abs(q.weights.sum() - 0.5) < 1e-15
    q0 = prism_quadrature(0, 0)
    assert q0.num_points == 1 and q0.weights[0] == 0.5
    assert abs(np.sum(q.weights * q.points[:, 0]) - 1 / 6) < 1e-15


@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords"}))
def test_reference_mass_matrix_properties(lname):
    el = element_for_layout(DofLayout(lname, LAYOUT_COUNTS[lname]))
    tri, line, _ = families(lname)
    M = reference_mass_matrix(el, prism_quadrature(*quad_degrees(lname)))
    np.testing.assert_allclose(M, M.T, atol=1e-16)
    assert np.all(np.linalg.eigvalsh(M) > 0)
    # sum of all entries = reference volume * ncomp
    assert abs(M.sum() - 0.5 * el.ncomp) < 1e-14
    # a higher-degree rule gives the same matrix (exactness)
    M2 = reference_mass_matrix(el, prism_quadrature(6, 8))
    np.testing.assert_allclose(M, M2, rtol=0, atol=1e-15)


def test_sharing_classes():
    assert sharing_class(builtin_layout("DG1", "DG1")) == 0
    assert sharing_class(builtin_layout("DG0", "DG0")) == 0
    assert sharing_class(builtin_layout("DG1", "CG1")) == 1
    assert sharing_class(builtin_layout("CG1", "DG0")) == 2
    assert sharing_class(builtin_layout("CG1", "CG1")) == 2


def test_count_flops_spec_examples():
    p = count_flops(builtin_layout("DG0", "DG0"), prism_quadrature(0, 0))
    assert (p.adds, p.muls) == (1, 3)
    a = count_flops(builtin_layout("CG1", "CG1"), prism_quadrature())
    b = count_flops(builtin_layout("DG1", "DG1"), prism_quadrature())
    assert a == b
    q6 = prism_quadrature(2, 2)
    q12 = prism_quadrature(4, 2)
    assert count_flops(builtin_layout("CG1", "CG1"), q12).muls == \
        2 * count_flops(builtin_layout("CG1", "CG1"), q6).muls


def test_perfbench_formulas():
    one = BaseMesh([[0, 1, 2]], [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    fs = number_dofs(ExtrudedMesh(one, 1), builtin_layout("CG1", "CG1"))
    assert perfbench.valuable_volume(fs) == 240
    assert perfbench.balance_factor(5, 5) == 2.0
    assert perfbench.balance_factor(3, 0) == 1.0
    assert abs(perfbench.balance_factor(7, 10) - 1.7) < 1e-2
    assert perfbench.vector_factor(0, 10) == 1.0
    assert perfbench.vector_factor(10, 10) == 4.0
    assert abs(perfbench.vector_factor(0.1933, 1.0) - 1.58) < 1e-2
    assert perfbench.peak_throughput(2.0, 2, 4) == 16.0
    with pytest.raises(ValueError):
        perfbench.balance_factor(0, 0, 0)
    with pytest.raises(ValueError):
        perfbench.vector_factor(2, 1)


@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords"}))
def test_kronecker_factors_reproduce_mref(lname):
    from paper_1604_05937_b200.quadrature import kronecker_factors
    el = element_for_layout(DofLayout(lname, LAYOUT_COUNTS[lname]))
    q = prism_quadrature(*quad_degrees(lname))
    M = reference_mass_matrix(el, q)
    Mt, Ml = kronecker_factors(el, q)
    h, v, c = (np.array(a) for a in (el.slot_h, el.slot_v, el.slot_comp))
    K = Mt[h][:, h] * Ml[v][:, v] * (c[:, None] == c[None, :])
    np.testing.assert_allclose(K, M, rtol=0, atol=1e-16)


@pytest.mark.parametrize("n,ordering,jitter", [(32, "rcm", 0.0),
                                                (64, "rcm", 0.0),
                                                (48, "random", 0.3),
                                                (40, "natural", 0.3)])
def test_product_mesh_equals_oracle_mesh(n, ordering, jitter):
    """configs.base_mesh (product: mesh.py / ordering.py mirrors, host C++
    RCM) against the oracle's independent C restatement: bit-exact."""
    import oracle
    from paper_1604_05937_b200 import configs
    mp, rp = configs.base_mesh(n, ordering, jitter, seed=5)
    mo, ro = oracle.base_mesh(n, ordering, jitter, seed=5)
    for k in ("cell_vertices", "coords", "cell_edges", "edge_vertices"):
        assert np.array_equal(np.asarray(getattr(mp, k)), getattr(mo, k)), k
    assert rp.random() == ro.random()   # same draw position afterwards
