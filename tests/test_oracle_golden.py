"""The CPU oracle against the reference's own outputs (golden.npz) and the
SPEC known answers.  Pins the oracle before it is used to check the GPU."""
from math import factorial

import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees

MESHES = ("one", "two", "sq5", "sq4rcm", "sq4rnd")


@pytest.mark.parametrize("mname", MESHES)
@pytest.mark.parametrize("layers", (1, 3, 4))
@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_oracle_maps_match_reference(golden, gmesh, mname, layers, lname):
    m, off, total = oracle.cell_map(gmesh(mname), layers,
                                    LAYOUT_COUNTS[lname])
    key = f"fs/{mname}/L{layers}/{lname}"
    np.testing.assert_array_equal(m, golden[key + "/cell_map"])
    np.testing.assert_array_equal(off, golden[key + "/offsets"])
    assert total == int(golden[key + "/total"])


@pytest.mark.parametrize("mname", ("one", "two", "sq4rcm"))
@pytest.mark.parametrize("layers", (1, 3))
@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_offset_addressing_equals_materialised(golden, gmesh, mname, layers,
                                               lname):
    """PAPER.md:546-553 / SPEC acceptance 2: map + l*offset == literal."""
    m, off, _ = oracle.cell_map(gmesh(mname), layers, LAYOUT_COUNTS[lname])
    mat = golden[f"fs/{mname}/L{layers}/{lname}/materialized"]
    for l in range(layers):
        np.testing.assert_array_equal(
            m.astype(np.int64) + l * off.astype(np.int64), mat[:, l, :])


@pytest.mark.parametrize("mname", MESHES)
@pytest.mark.parametrize("layers", (1, 3, 4))
def test_oracle_extrude_matches_reference(golden, gmesh, mname, layers):
    got = oracle.extrude(gmesh(mname).coords, layers, 1.0 / layers)
    np.testing.assert_array_equal(got, golden[f"coords/{mname}/L{layers}"])


def test_spec_known_answers(gmesh):
    one = gmesh("one")
    m, off, total = oracle.cell_map(one, 2, {(0, 0): 1})
    assert tuple(m[0]) == (0, 1, 3, 4, 6, 7) and total == 9
    assert tuple(m[0] + off) == (1, 2, 4, 5, 7, 8)
    m, _, _ = oracle.cell_map(one, 1, {(2, 1): 6})
    assert tuple(m[0]) == tuple(range(6))
    for name, want in (("CG1xCG1", 1), ("CG1xDG1", 2), ("DG1xDG1", 6)):
        _, off, _ = oracle.cell_map(one, 3, LAYOUT_COUNTS[name])
        assert set(off.tolist()) == {want}
    ks = [len(oracle.slot_table(LAYOUT_COUNTS[f"{h}x{v}"])[0])
          for h in ("CG1", "DG0", "DG1") for v in ("CG1", "DG0", "DG1")]
    assert ks == [6, 3, 6, 2, 1, 2, 6, 3, 6]


def _exact_monomial(i, j):
    return factorial(i) * factorial(j) / factorial(i + j + 2)


@pytest.mark.parametrize("deg", range(0, 7))
def test_triangle_rules_exact(deg):
    xy, w = oracle.tri_rule(deg)
    assert abs(w.sum() - 0.5) < 1e-15
    for i in range(deg + 1):
        for j in range(deg + 1 - i):
            got = np.sum(w * xy[:, 0] ** i * xy[:, 1] ** j)
            assert abs(got - _exact_monomial(i, j)) < 1e-15, (deg, i, j)


@pytest.mark.parametrize("deg", range(0, 9))
def test_line_rules_exact(deg):
    z, w = oracle.line_rule(deg)
    assert len(z) == deg // 2 + 1
    for p in range(deg + 1):
        assert abs(np.sum(w * z ** p) - 1.0 / (p + 1)) < 1e-15


@pytest.mark.parametrize("mname", ("one", "two", "sq3rcm"))
@pytest.mark.parametrize("layers", (1, 3))
@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords"}))
def test_oracle_assembly_matches_dense_bruteforce(golden, gmesh, mname,
                                                  layers, lname):
    """within 1e-13 absolute per entry of the dense assembler
    over the reference's materialised maps."""
    tri, line, nc = families(lname)
    prob = oracle.Problem(gmesh(mname), layers, LAYOUT_COUNTS[lname], tri,
                          line, nc, *quad_degrees(lname))
    key = f"asm/{mname}/L{layers}/{lname}"
    b = prob.assemble(golden[key + "/f"])
    np.testing.assert_allclose(b, golden[key + "/b"], rtol=0, atol=1e-13)
    b1 = prob.assemble(np.ones(prob.total))
    np.testing.assert_allclose(b1, golden[key + "/b_one"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("layers", (1, 4))
@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords",
                                                              "VP1"}))
def test_conservation(gmesh, layers, lname):
    """f = 1 on the unit cube -> sum b = 1."""
    tri, line, nc = families(lname)
    prob = oracle.Problem(gmesh("sq5"), layers, LAYOUT_COUNTS[lname], tri,
                          line, nc, *quad_degrees(lname))
    b = prob.assemble(np.ones(prob.total))
    assert abs(b.sum() - 1.0) < 1e-12


def test_dg0_single_prism(gmesh):
    """DG0xDG0, one prism of volume V, f = c -> c*V."""
    prob = oracle.Problem(gmesh("one"), 1, {(2, 1): 1}, "P0", "P0", 1, 0, 0,
                          layer_height=2.5)
    b = prob.assemble(np.array([3.0]))
    assert abs(b[0] - 3.0 * 0.5 * 2.5) < 1e-14


def test_colored_is_bitwise_thread_independent(gmesh):
    """coloured-parallel determinism."""
    for lname in ("CG1xCG1", "P2xP2", "DG1xCG1", "CG1xDG1"):
        tri, line, nc = families(lname)
        prob = oracle.Problem(gmesh("sq5"), 4, LAYOUT_COUNTS[lname], tri,
                              line, nc, *quad_degrees(lname))
        f = np.random.default_rng(1).random(prob.total)
        one = prob.assemble_colored(f, threads=1)
        four = prob.assemble_colored(f, threads=4)
        assert np.array_equal(one, four)
        seq = prob.assemble(f)
        np.testing.assert_allclose(one, seq, rtol=0, atol=1e-15)


def test_greedy_coloring_is_proper(gmesh):
    for name in ("one", "two", "sq4rcm", "sq5"):
        m = gmesh(name)
        col, n = oracle.greedy_color(m)
        cv = m.cell_vertices
        for v in range(m.num_vertices):
            cells = np.flatnonzero((cv == v).any(axis=1))
            assert len(set(col[cells].tolist())) == len(cells)
    assert oracle.greedy_color(gmesh("one"))[1] == 1
    assert oracle.greedy_color(gmesh("two"))[1] == 2


# --- the oracle's own base-mesh pipeline (oracle_mesh.c) against the
# reference's meshes and permutations (mesh.py:33-84, 228-254;
# ordering.py:45-152) --------------------------------------------------------

def _same_mesh(m, golden, name):
    p = f"mesh/{name}/"
    for k in ("cell_vertices", "coords", "cell_edges", "edge_vertices"):
        assert np.array_equal(getattr(m, k), golden[p + k]), (name, k)


@pytest.mark.parametrize("n", [3, 4, 5])
def test_oracle_unit_square_matches_reference(golden, n):
    _same_mesh(oracle.unit_square(n), golden, f"sq{n}")


@pytest.mark.parametrize("n", [4, 16])
def test_oracle_rcm_matches_reference(golden, n):
    fwd = oracle.rcm_forward(oracle.unit_square(n))
    assert np.array_equal(fwd, golden[f"sq{n}_rcm_forward"])


def test_oracle_random_order_matches_reference(golden):
    assert np.array_equal(oracle.random_forward(25, 7),
                          golden["sq4_rnd7_forward"])
    assert np.array_equal(oracle.random_forward(289, 3),
                          golden["sq16_rnd3_forward"])


@pytest.mark.parametrize("name,ordering", [("sq4rcm", "rcm"),
                                           ("sq3rcm", "rcm")])
def test_oracle_apply_ordering_matches_reference(golden, name, ordering):
    n = int(name[2])
    m = oracle.apply_ordering(oracle.unit_square(n),
                              oracle.rcm_forward(oracle.unit_square(n)))
    _same_mesh(m, golden, name)


def test_oracle_random_reordered_mesh_matches_reference(golden):
    sq4 = oracle.unit_square(4)
    _same_mesh(oracle.apply_ordering(sq4, golden["sq4_rnd7_forward"]),
               golden, "sq4rnd")
