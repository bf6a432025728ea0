"""Edge cases of the column loop on the device: an empty cell set, the DG
stream's full units + ragged tail for every DG layout, one layer, a
strip longer than the staged id block, int32 overflow refusal, and the
host-side validation of bad inputs ("rejected before
iteration")."""
import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _space(base, layers, lname):
    from paper_1604_05937_b200 import DofLayout, ExtrudedMesh, number_dofs
    return number_dofs(ExtrudedMesh(base, layers),
                       DofLayout(lname, LAYOUT_COUNTS[lname]))


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _oracle(base, layers, lname, f):
    tri, line, nc = families(lname)
    prob = oracle.Problem(base, layers, LAYOUT_COUNTS[lname], tri, line, nc,
                          *quad_degrees(lname))
    return prob.assemble(f)


@pytest.mark.parametrize("lname", ["CG1xCG1", "P2xP2", "VP1", "DG1xDG1",
                                   "DG1xCG1"])
def test_empty_cell_set(lname):
    """Vertices but no cells: every column receives nothing -> zeros."""
    from paper_1604_05937_b200.kernels import mass_action
    from paper_1604_05937_b200.mesh import BaseMesh
    base = BaseMesh(np.zeros((0, 3), dtype=np.int32),
                    [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    fs = _space(base, 3, lname)
    f = np.random.default_rng(0).random(fs.total_dofs)
    y = mass_action(fs, f)
    assert y.shape == (fs.total_dofs,)
    assert not np.any(y)


@pytest.mark.parametrize("lname", ["DG0xDG0", "DG0xDG1", "DG1xDG0",
                                   "DG1xDG1"])
@pytest.mark.parametrize("n,layers", [(17, 3), (23, 11), (40, 7)])
def test_dg_stream_units_and_ragged_tail(lname, n, layers):
    """2n² cells x layers cell-layers: whole 256-cell-layer TMA units, several
    per CTA, plus a tail handled by the generic kernel."""
    from paper_1604_05937_b200.kernels import mass_action
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    base = generate_unit_square_mesh(n)
    n_cl = base.num_cells * layers
    assert n_cl >= 256 and n_cl % 256
    fs = _space(base, layers, lname)
    f = np.random.default_rng(n).uniform(-1, 1, fs.total_dofs)
    from paper_1604_05937_b200.quadrature import prism_quadrature
    got = mass_action(fs, f, quadrature=prism_quadrature(*quad_degrees(lname)),
                      schedule="stream")
    assert _rel(got, _oracle(base, layers, lname, f)) <= 1e-12


@pytest.mark.parametrize("lname", ["CG1xCG1", "P2xP2", "CG1xDG1"])
def test_long_strips_restage_ids(lname, monkeypatch):
    """Strips longer than the 64 staged vertex ids per segment."""
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    from paper_1604_05937_b200.quadrature import prism_quadrature
    monkeypatch.setattr(kernels, "strip_max_len", lambda n, l: 200)
    base = generate_unit_square_mesh(64)   # diagonal strips of ~129 steps
    fs = _space(base, 5, lname)
    op = kernels.MassOperator(
        fs, prism_quadrature(*quad_degrees(lname)), schedule="stripred")
    (ptr, _steps, *_), _w = op._global_strips()
    lens = np.diff(ptr.cpu().numpy())
    assert lens.max() > 64
    f = np.random.default_rng(3).uniform(-1, 1, fs.total_dofs)
    got = kernels.mass_action(fs, f, operator=op)
    assert _rel(got, _oracle(base, 5, lname, f)) <= 1e-10


def test_int32_overflow_refused():
    """A space whose DoF numbers overflow int32 is refused by the loop (the
    reference would wrap them silently, fspace.py:203/214)."""
    from paper_1604_05937_b200 import DofLayout, ExtrudedMesh, number_dofs
    from paper_1604_05937_b200.kernels import MassOperator
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    fs = number_dofs(ExtrudedMesh(generate_unit_square_mesh(4), 3),
                     DofLayout("huge", {(0, 0): 1 << 26}))
    assert not fs.fits_int32
    with pytest.raises(ValueError, match="int32"):
        MassOperator(fs)


def test_bad_inputs_rejected_before_iteration():
    from paper_1604_05937_b200.kernels import MassOperator
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    base = generate_unit_square_mesh(4)
    fs = _space(base, 3, "CG1xCG1")
    op = MassOperator(fs)
    coords = extrude_coordinates(base.coords, 3, 1 / 3)
    x = torch.zeros(fs.total_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        op.apply(x[:-1], coords)                       # wrong length
    with pytest.raises(ValueError):
        op.apply(x, coords[:-3])                       # wrong mesh
    with pytest.raises(ValueError):
        op.apply(x, coords, schedule="no-such-schedule")
    with pytest.raises(ValueError):
        op.apply(x, coords, schedule="stream")         # CG is not a DG field


@pytest.mark.parametrize("lname", ["DG1xDG1", "DG0xDG1", "CG1xCG1", "P2xP2"])
@pytest.mark.parametrize("overlap", [False, True])
def test_graph_of_repeated_applies(lname, overlap):
    """MassOperator.graph(repeat=K, overlap): K captured applies (DG: with
    programmatic dependent launch between them) leave exactly the result of
    one apply (bitwise for the deterministic DG stream)."""
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    base = generate_unit_square_mesh(48)
    fs = _space(base, 10, lname)
    coords = extrude_coordinates(base.coords, 10, 0.1)
    op = MassOperator(fs)
    x = torch.from_numpy(
        np.random.default_rng(5).uniform(-1, 1, fs.total_dofs)).cuda()
    ref = op.apply(x, coords).clone()
    y = torch.full_like(x, np.nan)
    g = op.graph(x, coords, y, repeat=7, overlap=overlap)
    y.fill_(np.nan)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    if lname.startswith("DG"):
        assert torch.equal(y, ref)
    else:
        assert _rel(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-12



@pytest.mark.parametrize("lname", ["DG0xCG1", "DG1xCG1"])
@pytest.mark.parametrize("n,layers,ordering", [(6, 16, "rcm"), (12, 20, "rcm"),
                                               (16, 33, "random"),
                                               (40, 17, "rcm")])
def test_cell_stream_vs_oracle(lname, n, layers, ordering):
    """Vertical-only cell columns through the TMA cell-stream kernel (units
    overlapping by one cell-layer; column tops and unit boundaries)."""
    from paper_1604_05937_b200.configs import base_mesh
    from paper_1604_05937_b200.kernels import mass_action
    from paper_1604_05937_b200.quadrature import prism_quadrature
    base, _ = base_mesh(n, ordering)
    fs = _space(base, layers, lname)
    assert base.num_cells * layers > 256     # several units
    f = np.random.default_rng(layers).uniform(-1, 1, fs.total_dofs)
    got = mass_action(fs, f, quadrature=prism_quadrature(*quad_degrees(lname)))
    assert _rel(got, _oracle(base, layers, lname, f)) <= 1e-12


@pytest.mark.gpu
def test_dg_stream_honours_a_caller_map():
    """pm_column_mass (AUTO) with a DG layout and a caller-supplied map that
    is not the dense Alg. 1 numbering (cells' blocks in reverse order): the
    stream kernel, which never reads the field map, must not take it."""
    import torch
    from paper_1604_05937_b200 import (ExtrudedMesh, builtin_layout,
                                       extrude_coordinates,
                                       generate_unit_square_mesh,
                                       number_dofs)
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.kernels import MassOperator
    m = ExtrudedMesh(generate_unit_square_mesh(16), 8)
    fs = number_dofs(m, builtin_layout("DG1", "DG1"))
    op = MassOperator(fs)
    n2, k, L = m.base.num_cells, fs.num_slots, m.layers
    coords = extrude_coordinates(m.base.coords, L, m.layer_height)
    x = torch.from_numpy(np.random.default_rng(5).uniform(
        -1, 1, fs.total_dofs)).cuda()
    y_ref = op.apply(x, coords).cpu().numpy().reshape(n2, L * k)
    rev = torch.arange(n2 - 1, -1, -1, device="cuda", dtype=torch.int32)
    cmap2 = (rev[:, None] * (k * L) +
             torch.arange(k, device="cuda", dtype=torch.int32)).contiguous()
    x2 = x.reshape(n2, L * k).flip(0).contiguous().reshape(-1)
    y2 = torch.full_like(x2, float("nan"))
    _lib.column_mass(fs.layout, k, n2, L, cmap2, op.offs, op.xmap, op.xoffs,
                     coords, op.mref, x2, y2, fs.total_dofs, kron=op.kron)
    got = y2.cpu().numpy().reshape(n2, L * k)[::-1]
    assert np.abs(got - y_ref).max() <= 1e-12 * np.abs(y_ref).max()
    # and the dense map itself still takes the stream kernel's result
    y3 = torch.empty_like(x)
    _lib.column_mass(fs.layout, k, n2, L, op.cmap, op.offs, op.xmap,
                     op.xoffs, coords, op.mref, x, y3, fs.total_dofs,
                     kron=op.kron)
    assert np.array_equal(y3.cpu().numpy().reshape(n2, L * k), y_ref)
