"""Custom quadrature rules: the Kronecker factors come from the rule's own
tensor factors (or do not exist), and every schedule applies them
correctly — including the general (non ta·I + tb·J) triangle stage of the
strip kernel."""
import numpy as np
import pytest

from paper_1604_05937_b200.extrusion import ExtrudedMesh
from paper_1604_05937_b200.fspace import builtin_layout, number_dofs
from paper_1604_05937_b200.kernels import kron_reproduces
from paper_1604_05937_b200.mesh import generate_unit_square_mesh
from paper_1604_05937_b200.quadrature import (QuadratureRule,
                                              element_for_layout,
                                              kronecker_factors,
                                              reference_mass_matrix,
                                              tensor_factors)


def _asym_tensor_rule():
    # a (deliberately unsymmetric) 3-point triangle rule x 2-point Gauss
    tp = np.array([[0.2, 0.1], [0.6, 0.2], [0.1, 0.7]])
    tw = np.array([0.2, 0.15, 0.15])
    g = 0.5 / np.sqrt(3.0)
    lp, lw = np.array([0.5 - g, 0.5 + g]), np.array([0.5, 0.5])
    pts = np.array([[a, b, z] for (a, b), _ in zip(tp, tw) for z in lp])
    w = np.array([wa * wb for wa in tw for wb in lw])
    return QuadratureRule(pts, w, 2, 3)


def _non_tensor_rule():
    rng = np.random.default_rng(3)
    pts = np.column_stack([rng.uniform(0, 0.5, 6), rng.uniform(0, 0.5, 6),
                           rng.uniform(0, 1, 6)])
    return QuadratureRule(pts, np.full(6, 0.5 / 6), 1, 1)


def test_asymmetric_tensor_rule_factors():
    el = element_for_layout(builtin_layout("CG1", "CG1"))
    rule = _asym_tensor_rule()
    assert tensor_factors(rule) is not None
    kron = kronecker_factors(el, rule)
    assert kron_reproduces(el, kron, reference_mass_matrix(el, rule))
    t = kron[0]
    # not of the form ta I + tb J: the strip kernel's general path
    assert not np.allclose(np.diag(t), t[0, 0])


def test_default_rules_are_permutation_invariant():
    from paper_1604_05937_b200.fspace import P2_LAYOUT, VP1_LAYOUT
    from paper_1604_05937_b200.kernels import (default_quadrature,
                                               tri_permutation_invariant)
    for lay in (builtin_layout("CG1", "CG1"), builtin_layout("CG1", "DG1"),
                P2_LAYOUT, VP1_LAYOUT):
        el = element_for_layout(lay)
        assert tri_permutation_invariant(
            kronecker_factors(el, default_quadrature(el))[0]), lay.name
    el = element_for_layout(builtin_layout("CG1", "CG1"))
    assert not tri_permutation_invariant(
        kronecker_factors(el, _asym_tensor_rule())[0])


def test_non_tensor_rule_has_no_factors():
    el = element_for_layout(builtin_layout("CG1", "CG1"))
    rule = _non_tensor_rule()
    assert tensor_factors(rule) is None
    assert kronecker_factors(el, rule) is None
    assert not kron_reproduces(el, None, reference_mass_matrix(el, rule))


@pytest.mark.gpu
@pytest.mark.parametrize("rule", ["asym", "non_tensor"])
@pytest.mark.parametrize("layout", ["CG1xCG1", "CG1xDG1", "DG1xDG1"])
@pytest.mark.parametrize("schedule", ["auto", "stripred", "column"])
def test_custom_rule_matches_dense_assembler(rule, layout, schedule):
    import torch
    from paper_1604_05937_b200 import verification
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    h, v = layout.split("x")
    lay = builtin_layout(h, v)
    if schedule == "stripred" and h != "CG1":
        pytest.skip("strips are for vertex-column layouts")
    if schedule == "column" and h == "DG1":
        schedule = "stream"
    base = generate_unit_square_mesh(6)
    mesh = ExtrudedMesh(base, 5)
    fs = number_dofs(mesh, lay)
    q = _asym_tensor_rule() if rule == "asym" else _non_tensor_rule()
    op = MassOperator(fs, q, schedule=schedule)
    assert op.kron_ok == (rule == "asym")
    # an unsymmetric triangle rule is not invariant under vertex
    # permutations: the strip kernels (window-slot placement) refuse it; a
    # non-tensor rule has no factors (every schedule: dense generic kernel)
    assert not op.strip_invariant
    coords = extrude_coordinates(base.coords, 5, mesh.layer_height)
    x = np.random.default_rng(1).uniform(-1, 1, fs.total_dofs)
    if schedule == "stripred" and rule == "asym":
        with pytest.raises(ValueError, match="permutation invariant"):
            op.apply(torch.from_numpy(x).cuda(), coords)
        return
    y = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    ref = verification.dense_mass_action(fs, x, coords.cpu().numpy(), op.mref)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
