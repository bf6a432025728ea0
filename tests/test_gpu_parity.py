"""CUDA path vs the oracle / reference golden vectors (needs a B200).

Bars (BASELINE.json north_star): bit-exact for maps and numbering; 1e-12
relative for DG (deterministic); 1e-10 relative for CG (re-ordered
increments).  "Relative" = max-norm error / max-norm of the oracle.
"""
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


def _tol(lname):
    from paper_1604_05937_b200.quadrature import sharing_class
    from paper_1604_05937_b200 import DofLayout
    return 1e-12 if sharing_class(DofLayout(lname, LAYOUT_COUNTS[lname])) \
        == 0 else 1e-10


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


# ------------------------------------------------------------- K0 maps
@pytest.mark.parametrize("mname", ("one", "two", "sq5", "sq4rcm", "sq4rnd"))
@pytest.mark.parametrize("layers", (1, 3, 4))
@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_device_maps_bit_exact(golden, gmesh, mname, layers, lname):
    fs = _space(gmesh(mname), layers, lname)
    key = f"fs/{mname}/L{layers}/{lname}"
    np.testing.assert_array_equal(fs.cell_map, golden[key + "/cell_map"])
    np.testing.assert_array_equal(fs.offsets, golden[key + "/offsets"])
    assert fs.total_dofs == int(golden[key + "/total"])


def test_device_maps_large_vs_oracle():
    from paper_1604_05937_b200 import configs
    for w in (configs.WORKLOADS["C2"], configs.WORKLOADS["C3"]):
        fs, _, _, _ = configs.build(w)
        m, off, total = oracle.cell_map(fs.mesh.base, fs.mesh.layers,
                                        fs.layout.counts)
        assert np.array_equal(fs.cell_map, m)
        assert np.array_equal(fs.offsets, off) and total == fs.total_dofs


def test_device_map_wraps_like_reference():
    """fspace.py:203/214 store int64 origins into int32 (wraps)."""
    from paper_1604_05937_b200 import (BaseMesh, DofLayout, ExtrudedMesh,
                                       number_dofs)
    one = BaseMesh([[0, 1, 2]], [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    lay = DofLayout("big", {(0, 0): 1, (2, 1): 1})
    fs = number_dofs(ExtrudedMesh(one, 800_000_000), lay)
    m, _, total = oracle.cell_map(one, 800_000_000, lay.counts)
    assert total == fs.total_dofs > 2**31
    np.testing.assert_array_equal(fs.cell_map, m)
    assert not fs.fits_int32


@pytest.mark.parametrize("mname", ("one", "two", "sq5", "sq4rcm"))
@pytest.mark.parametrize("layers", (1, 3, 4))
def test_device_extrude_bit_exact(golden, gmesh, mname, layers):
    from paper_1604_05937_b200 import extrude_coordinates
    got = extrude_coordinates(gmesh(mname).coords, layers, 1.0 / layers,
                              device="cpu")
    np.testing.assert_array_equal(got, golden[f"coords/{mname}/L{layers}"])


# ------------------------------------------------------------- par-loop
@pytest.mark.parametrize("mname", ("one", "two", "sq4rcm"))
@pytest.mark.parametrize("layers", (1, 3))
@pytest.mark.parametrize("lname", sorted(LAYOUT_COUNTS))
def test_loop_addresses_equal_materialised(golden, gmesh, mname, layers,
                                           lname):
    """The device loop's per-(cell,layer) lists == verification.py:47-75."""
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.kernels import ListProbeKernel
    fs = _space(gmesh(mname), layers, lname)
    out = torch.empty((fs.mesh.base.num_cells, layers, fs.num_slots),
                      dtype=torch.int64, device="cuda")
    iterate_columns([fs], ListProbeKernel(fs), [out])
    np.testing.assert_array_equal(
        out.cpu().numpy(), golden[f"fs/{mname}/L{layers}/{lname}/materialized"])


def test_counting_kernel(gmesh):
    """DG0xDG0 counting kernel -> all ones, sum N2*layers."""
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.kernels import CountingKernel
    fs = _space(gmesh("sq5"), 4, "DG0xDG0")
    out = torch.zeros(fs.total_dofs, dtype=torch.float64, device="cuda")
    iterate_columns([fs], CountingKernel(fs), [out])
    o = out.cpu().numpy()
    assert np.all(o == 1.0) and o.sum() == fs.mesh.base.num_cells * 4


def test_arity_and_mesh_mismatch_rejected(gmesh):
    from paper_1604_05937_b200 import COORDS_LAYOUT, ExtrudedMesh, number_dofs
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.kernels import MassKernel
    fs = _space(gmesh("sq5"), 3, "CG1xCG1")
    other = _space(gmesh("sq5"), 3, "P2xP2")
    xfs = number_dofs(fs.mesh, COORDS_LAYOUT)
    k = MassKernel(fs)
    with pytest.raises(ValueError):
        iterate_columns([other, xfs], k, [None, None, None])
    xfs2 = number_dofs(ExtrudedMesh(gmesh("sq5"), 3), COORDS_LAYOUT)
    with pytest.raises(ValueError):
        iterate_columns([fs, xfs2], k, [None, None, None])


SCHEDULES = ("auto", "atomic", "colored", "column", "patch", "strip",
             "stripred", "striptma", "pstrip", "stripdg")


def _experimental():
    from paper_1604_05937_b200 import _lib
    return _lib.experimental()


def _schedule_applies(lname, schedule):
    if schedule == "pstrip" and not _experimental():
        return False    # built without PM_EXPERIMENTAL
    if schedule == "patch":
        return lname in ("CG1xCG1", "CG1xDG0", "CG1xDG1", "P2xP2", "VP1")
    if schedule == "strip":
        return lname in ("CG1xCG1", "CG1xDG0", "CG1xDG1", "VP1")
    if schedule in ("stripred", "pstrip"):
        return lname in ("CG1xCG1", "CG1xDG0", "CG1xDG1", "VP1", "P2xP2")
    if schedule == "striptma":
        return lname in ("CG1xCG1", "VP1")
    if schedule == "stripdg":
        return lname in ("DG0xDG0", "DG0xDG1", "DG1xDG0", "DG1xDG1",
                         "DG0xCG1", "DG1xCG1")
    return True


@pytest.mark.parametrize("mname", ("one", "two", "sq5", "sq4rnd"))
@pytest.mark.parametrize("layers", (1, 3, 5))
@pytest.mark.parametrize("lname", sorted(set(LAYOUT_COUNTS) - {"coords"}))
@pytest.mark.parametrize("schedule", SCHEDULES)
def test_mass_action_matches_oracle(gmesh, mname, layers, lname, schedule):
    from paper_1604_05937_b200.kernels import mass_action
    if not _schedule_applies(lname, schedule):
        pytest.skip("schedule not defined for this layout")
    from paper_1604_05937_b200.quadrature import prism_quadrature
    base = gmesh(mname)
    fs = _space(base, layers, lname)
    tri, line, nc = families(lname)
    qd = quad_degrees(lname)
    prob = oracle.Problem(base, layers, LAYOUT_COUNTS[lname], tri, line, nc,
                          *qd)
    f = np.random.default_rng(layers).uniform(-1, 1, fs.total_dofs)
    ref = prob.assemble(f)
    got = mass_action(fs, f, quadrature=prism_quadrature(*qd),
                      schedule=schedule)
    assert _rel(got, ref) <= _tol(lname), (lname, schedule)


@pytest.mark.parametrize("lname", ("CG1xCG1", "P2xP2", "DG1xCG1", "VP1"))
def test_iterate_columns_accumulates(gmesh, lname):
    """iterate_columns adds into the output."""
    from paper_1604_05937_b200 import COORDS_LAYOUT, number_dofs
    from paper_1604_05937_b200 import extrude_coordinates
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.kernels import MassKernel
    base = gmesh("sq5")
    fs = _space(base, 3, lname)
    xfs = number_dofs(fs.mesh, COORDS_LAYOUT)
    coords = extrude_coordinates(base.coords, 3, 1 / 3)
    f = torch.rand(fs.total_dofs, dtype=torch.float64, device="cuda")
    out = torch.zeros_like(f)
    k = MassKernel(fs)
    iterate_columns([fs, xfs], k, [f, coords, out])
    once = out.clone()
    iterate_columns([fs, xfs], k, [f, coords, out], schedule="colored")
    assert _rel(out.cpu().numpy(), 2 * once.cpu().numpy()) < 1e-12


@pytest.mark.parametrize("lname", ("CG1xCG1", "P2xP2", "VP1", "CG1xDG1"))
@pytest.mark.parametrize("schedule", ("colored", "patch", "strip"))
def test_deterministic_schedules(gmesh, lname, schedule):
    from paper_1604_05937_b200.kernels import mass_action
    if not _schedule_applies(lname, schedule):
        pytest.skip("schedule not defined for this layout")
    fs = _space(gmesh("sq5"), 4, lname)
    f = torch.rand(fs.total_dofs, dtype=torch.float64, device="cuda")
    a = mass_action(fs, f, schedule=schedule)
    b = mass_action(fs, f, schedule=schedule)
    assert torch.equal(a, b)


@pytest.mark.parametrize("lname", ("CG1xCG1", "P2xP2", "VP1"))
@pytest.mark.parametrize("W", (8, 16, 32))
@pytest.mark.parametrize("layers", (1, 7, 33))
def test_patch_chunk_widths(lname, W, layers):
    """Every chunk width and ragged chunk tails against the oracle."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    from paper_1604_05937_b200.schedule import plan_for
    w = configs.Workload("pw", 12, layers, lname, quad_degrees(lname),
                         jitter=0.2)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad, schedule="patch")
    from paper_1604_05937_b200.kernels import _color
    col = _color(m)
    plan, W2, _, _ = plan_for(m.base, fs.layout, layers, col.color_of,
                              col.num_colors, W=W, smem_budget=24 * 1024)
    op._patch = (plan, plan.device(op._dev), W2)
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    y = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    ref = _oracle_for(w, fs).assemble(x)
    assert _rel(y, ref) <= 1e-10


def test_residual_field_api_and_conservation(gmesh):
    from paper_1604_05937_b200.kernels import Field, assemble_residual
    for lname in sorted(set(LAYOUT_COUNTS) - {"coords", "VP1"}):
        fs = _space(gmesh("sq5"), 4, lname)
        b = assemble_residual(fs, Field(fs, np.ones(fs.total_dofs)))
        assert isinstance(b, Field)
        assert abs(b.values.sum() - 1.0) < 1e-12, lname


# ------------------------------------------------------- BASELINE configs
def _config_case(name, schedule="auto"):
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.WORKLOADS[name]
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    op = MassOperator(fs, quad, schedule=schedule)
    y = op.apply(torch.from_numpy(x).cuda(), coords)
    return w, fs, x, y.cpu().numpy()


def _oracle_for(w, fs):
    from paper_1604_05937_b200.quadrature import element_for_layout
    el = element_for_layout(fs.layout)
    return oracle.Problem(fs.mesh.base, fs.mesh.layers, fs.layout.counts,
                          el.tri, el.line, el.ncomp, *w.quad)


@pytest.mark.parametrize("name", ("C1", "C2"))
def test_config_full_size_vs_oracle(name):
    w, fs, x, y = _config_case(name)
    ref = _oracle_for(w, fs).assemble_colored(x)
    assert _rel(y, ref) <= (1e-12 if w.layout.startswith("DG") else 1e-10)


def test_config3_reduced_vs_oracle():
    """C3's space and degree-6 quadrature on a 64^2 base, 12 layers."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.Workload("C3-small", 64, 12, "P2xP2", (6, 6))
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    for sched in ("auto", "colored"):
        y = MassOperator(fs, quad, schedule=sched).apply(
            torch.from_numpy(x).cuda(), coords).cpu().numpy()
        assert _rel(y, _oracle_for(w, fs).assemble_colored(x)) <= 1e-10


@pytest.mark.parametrize("layout", ("CG1xCG1", "DG1xDG1"))
@pytest.mark.parametrize("ordering", ("rcm", "random"))
@pytest.mark.parametrize("layers", (1, 2, 5))
def test_config4_sweep_points_vs_oracle(layout, ordering, layers):
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.sweep_workload(layout, layers, ordering)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    y = MassOperator(fs, quad).apply(torch.from_numpy(x).cuda(),
                                     coords).cpu().numpy()
    ref = _oracle_for(w, fs).assemble_colored(x)
    assert _rel(y, ref) <= (1e-12 if layout.startswith("DG") else 1e-10)


def test_config3_full_size_properties():
    """C3 at full size: schedules agree, conservation, symmetry."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.WORKLOADS["C3"]
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    xa = torch.from_numpy(x).cuda()
    ya = MassOperator(fs, quad, schedule="atomic").apply(xa, coords)
    yc = MassOperator(fs, quad, schedule="colored").apply(xa, coords)
    yp = MassOperator(fs, quad, schedule="patch").apply(xa, coords)
    assert _rel(ya.cpu().numpy(), yc.cpu().numpy()) <= 1e-10
    assert _rel(yp.cpu().numpy(), yc.cpu().numpy()) <= 1e-10
    one = torch.ones_like(xa)
    s = MassOperator(fs, quad).apply(one, coords).sum().item()
    assert abs(s - 1.0) < 1e-10
    z = torch.rand_like(xa)
    op = MassOperator(fs, quad)
    lhs = torch.dot(z, op.apply(xa, coords)).item()
    rhs = torch.dot(xa, op.apply(z, coords)).item()
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "P2xP2"))
@pytest.mark.parametrize("world", (1, 2, 4))
def test_sharded_windows_on_one_gpu(lname, world):
    """Each rank's windowed column loop (no exchange), then the halo adds
    emulated on the host: equals the full mass action (config-5 path)."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.shard import ShardedMassOperator, ghost_origins
    w = configs.Workload("c5-small", 24, 6, lname, quad_degrees(lname))
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    ref = _oracle_for(w, fs).assemble(x)
    xd = torch.from_numpy(x).cuda()
    ops = [ShardedMassOperator(fs, r, world, quad) for r in range(world)]
    wins = []
    for op in ops:
        lo, hi = op.window
        clo, chi = op.shard.coord_window
        wins.append(op.apply(xd[lo:hi].clone(), coords[clo:chi].clone(),
                             exchange=False).cpu().numpy())
    for op in ops:
        s = op.shard
        for q, ids in s.send.items():
            for _d, o, c in ghost_origins(fs, ids):
                for org in o:
                    a = org - s.window[0]
                    b = org - ops[q].window[0]
                    wins[q][b:b + c] += wins[s.rank][a:a + c]
    got = np.zeros_like(ref)
    for op in ops:
        for _d, o, c in ghost_origins(fs, op.shard.owned):
            for org in o:
                a = org - op.window[0]
                got[org:org + c] = wins[op.rank][a:a + c]
    assert _rel(got, ref) <= 1e-10


def test_halo_kernels_match_host():
    from paper_1604_05937_b200 import _lib
    y = torch.rand(1000, dtype=torch.float64, device="cuda")
    cols = torch.tensor([100, 300, 650], dtype=torch.int64, device="cuda")
    buf = torch.empty(3 * 7, dtype=torch.float64, device="cuda")
    _lib.halo_pack(y, cols, 7, buf, base=50)   # window starts at DoF 50
    yh = y.cpu().numpy()
    want = np.concatenate([yh[c - 50:c - 50 + 7] for c in (100, 300, 650)])
    np.testing.assert_array_equal(buf.cpu().numpy(), want)
    y2 = y.clone()
    _lib.halo_unpack_add(y2, cols, 7, buf, base=50)
    d = (y2 - y).cpu().numpy()
    for c in (100, 300, 650):
        np.testing.assert_array_equal(d[c - 50:c - 50 + 7], yh[c - 50:c - 50 + 7])


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "CG1xDG1", "CG1xDG0"))
@pytest.mark.parametrize("W", (8, 16, 32))
@pytest.mark.parametrize("layers", (1, 7, 33, 64))
def test_strip_chunk_widths(lname, W, layers):
    """Strip schedule: every chunk width, ragged tails, small patches."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator, _color
    from paper_1604_05937_b200.schedule import build_strip_plan
    w = configs.Workload("sw", 14, layers, lname, quad_degrees(lname),
                         ordering="random", jitter=0.2)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad, schedule="strip")
    col = _color(m)
    plan = build_strip_plan(m.base, fs.layout, layers, col.color_of,
                            col.num_colors, W=W, smem_budget=48 * 1024,
                            max_strip=11)
    op._strip = (plan, plan.device(op._dev))
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    y = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    ref = _oracle_for(w, fs).assemble(x)
    assert _rel(y, ref) <= 1e-10


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "CG1xDG1", "CG1xDG0",
                                   "P2xP2"))
@pytest.mark.parametrize("layers", (1, 5, 16, 33, 64))
def test_stripred_layers(lname, layers):
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.Workload("srl", 14, layers, lname, quad_degrees(lname),
                         ordering="random", jitter=0.2)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad, schedule="stripred")
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    xd = torch.from_numpy(x).cuda()
    y = op.apply(xd, coords).cpu().numpy()
    ref = _oracle_for(w, fs).assemble(x)
    assert _rel(y, ref) <= 1e-10
    y2 = op.apply(xd, coords, torch.from_numpy(y).cuda(), accumulate=True)
    assert _rel(y2.cpu().numpy(), 2 * ref) <= 1e-10


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "CG1xDG1", "CG1xDG0",
                                   "P2xP2"))
@pytest.mark.parametrize("layers", (1, 5, 16, 33, 64, 100))
@pytest.mark.parametrize("patch", (1, 8, 64, 100000))
def test_patch_strips_layers(lname, layers, patch, monkeypatch):
    """Store-first patch strips: every DoF written (y starts as NaN), equal
    to the oracle, for one-cell patches (everything shared), small and
    whole-mesh patches and every chunk-boundary case; accumulate adds."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    if not _experimental():
        pytest.skip("patch strips: library built without PM_EXPERIMENTAL")
    monkeypatch.setenv("PM_PATCH_CELLS", str(patch))
    w = configs.Workload("psl", 12, layers, lname, quad_degrees(lname),
                         ordering="random", jitter=0.2)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad, schedule="pstrip")
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    xd = torch.from_numpy(x).cuda()
    y = torch.full_like(xd, float("nan"))
    op.apply(xd, coords, y)
    ref = _oracle_for(w, fs).assemble(x)
    yh = y.cpu().numpy()
    assert np.isfinite(yh).all()
    assert _rel(yh, ref) <= 1e-10
    y2 = op.apply(xd, coords, y, accumulate=True)
    assert _rel(y2.cpu().numpy(), 2 * ref) <= 1e-10


@pytest.mark.parametrize("lname,layers,n", (("DG1xDG1", 50, 32),
                                            ("DG1xDG1", 7, 24),
                                            ("DG0xDG1", 33, 20),
                                            ("CG1xCG1", 10, 16)))
def test_host_pipelined_mass_action(lname, layers, n):
    """mass_action with pinned host buffers (chunked H2D / compute / D2H
    for DG fields) equals the device path and the oracle."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator, mass_action
    w = configs.Workload("hp", n, layers, lname, quad_degrees(lname))
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad)
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    got = mass_action(fs, xh, coords, operator=op, out=yh).numpy()
    dev = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    if lname.startswith("DG"):
        # the host path streams DG fields by cell ranges (the stream
        # kernel): bitwise equal to it; the device default may walk strips
        # (stripdg) with another operation order
        dev_s = op.apply(torch.from_numpy(x).cuda(), coords,
                         schedule="stream").cpu().numpy()
        assert np.array_equal(got, dev_s)
    assert _rel(got, dev) <= _tol(lname)
    assert _rel(got, _oracle_for(w, fs).assemble(x)) <= _tol(lname)


@pytest.mark.parametrize("lname", ("DG0xDG0", "DG0xDG1", "DG1xDG0",
                                   "DG1xDG1", "DG0xCG1", "DG1xCG1"))
@pytest.mark.parametrize("ordering", ("rcm", "random"))
@pytest.mark.parametrize("layers", (1, 7, 16, 33, 64, 100))
def test_dg_strips(lname, ordering, layers):
    """DG layouts along strips (schedule "stripdg"): every chunk width
    (W by layers), ragged tails, jittered random meshes, NaN-filled output
    (every DoF stored), accumulate mode."""
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.Workload("sdg", 18, layers, lname, quad_degrees(lname),
                         ordering=ordering, jitter=0.2)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad, schedule="stripdg")
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    ref = _oracle_for(w, fs).assemble(x)
    xd = torch.from_numpy(x).cuda()
    y = torch.full_like(xd, float("nan"))
    op.apply(xd, coords, y)
    yh = y.cpu().numpy()
    assert np.isfinite(yh).all()
    tol = 1e-12 if lname.endswith("DG0") or lname.endswith("DG1") else 1e-10
    assert _rel(yh, ref) <= tol
    y2 = op.apply(xd, coords, y, accumulate=True)
    assert _rel(y2.cpu().numpy(), 2 * ref) <= tol


@pytest.mark.parametrize("lname", ("DG0xDG0", "DG1xDG0", "DG0xCG1",
                                   "DG1xCG1"))
@pytest.mark.parametrize("ordering", ("rcm", "random"))
def test_dg_strips_medium(lname, ordering):
    """The cell-only strip kernels where they are the default, on a mesh
    with long strips, many items and several layer chunks (128^2, 70
    layers: W = 32, three chunks, the last one ragged), against the
    oracle's column loop (oracle/fast.py)."""
    from oracle import fast
    from paper_1604_05937_b200 import configs, extrude_coordinates
    from paper_1604_05937_b200.configs import layout_of
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.Workload("sdgm", 128, 70, lname, quad_degrees(lname),
                         ordering=ordering)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    op = MassOperator(fs, quad)
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    xd = torch.from_numpy(x).cuda()
    y = torch.full_like(xd, float("nan"))
    op.apply(xd, coords, y)
    assert op.last_schedule == "stripdg"
    tri, line, nc = families(lname)
    arm = fast.FastMass(m.base, m.layers, layout_of(lname).counts, tri, line,
                        nc, *quad_degrees(lname))
    ref = arm.apply(x)
    tol = 1e-12 if lname.endswith(("DG0", "DG1")) else 1e-10
    assert _rel(y.cpu().numpy(), ref) <= tol
