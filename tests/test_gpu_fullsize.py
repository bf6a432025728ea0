"""Oracle parity at every BASELINE config's stated size (needs a B200).

The checker at full size is the oracle's column loop with the element
matrix integrated by the oracle's own literal quadrature (oracle/fast.py,
pinned against the literal-quadrature loop in tests/test_cpu_baseline.py),
on meshes built by the oracle alone (oracle/oracle_mesh.c, pinned against
the reference's meshes in tests/test_oracle_golden.py).  The literal loop
itself is also run on a sample of the cells and compared on every DoF whose
cells all lie in the sample.  Bars (BASELINE.json north_star): 1e-10
relative for CG, 1e-12 for DG (max-norm error / max-norm of the oracle).
SPEC.md:354 (every cell-layer exactly once), :433-435 (oracle equivalence).
"""
import numpy as np
import pytest

import oracle
from oracle import fast

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

FAMILY = {"CG1xCG1": ("P1", "P1", 1), "DG1xDG1": ("P1", "P1", 1),
          "P2xP2": ("P2", "P2", 1), "VP1": ("P1", "P1", 3)}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _tol(layout):
    return 1e-12 if layout.startswith("DG") else 1e-10


_MESH = {}


def _oracle_mesh(w):
    key = (w.n, w.ordering, w.jitter, w.seed)
    if key not in _MESH:
        _MESH.clear()
        _MESH[key] = oracle.base_mesh(w.n, w.ordering, w.jitter, w.seed)[0]
    return _MESH[key]


def _build(w):
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    return fs, quad, x, coords


def _check_mesh(fs, w):
    """The product's mesh (device pipeline) equals the oracle's, bit-exact."""
    mo = _oracle_mesh(w)
    b = fs.mesh.base
    for k in ("cell_vertices", "coords", "cell_edges"):
        assert np.array_equal(np.asarray(getattr(b, k)), getattr(mo, k)), k


def _oracle_y(w, x):
    tri, line, nc = FAMILY[w.layout]
    from paper_1604_05937_b200.configs import layout_of
    arm = fast.FastMass(_oracle_mesh(w), w.layers, layout_of(w.layout).counts,
                        tri, line, nc, *w.quad)
    return arm.apply(x).copy(), arm


def _literal_interior(w, x, y, n_cells):
    """The literal-quadrature oracle over the first n_cells cells agrees
    with y on every vertex-column DoF whose cells are all among them."""
    tri, line, nc = FAMILY[w.layout]
    from paper_1604_05937_b200.configs import layout_of
    base = _oracle_mesh(w)
    prob = oracle.Problem(base, w.layers, layout_of(w.layout).counts, tri,
                          line, nc, *w.quad)
    part = prob.assemble_colored(x, n_cells=n_cells)
    cv = base.cell_vertices
    last = np.zeros(base.num_vertices, dtype=np.int64)
    np.maximum.at(last, cv.ravel(), np.repeat(np.arange(base.num_cells), 3))
    inner = np.nonzero(last < n_cells)[0]
    assert inner.size > 100
    col = (w.layers + 1) * {"CG1xCG1": 1, "VP1": 3}.get(w.layout, 0)
    if col == 0:
        return
    idx = (inner[:, None] * col + np.arange(col)).ravel()
    assert _rel(y[idx], part[idx]) <= _tol(w.layout)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_configs_at_full_size(name):
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.WORKLOADS[name]
    fs, quad, x, coords = _build(w)
    _check_mesh(fs, w)
    op = MassOperator(fs, quad)
    y = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    ref, _arm = _oracle_y(w, x)
    assert _rel(y, ref) <= _tol(w.layout), op.last_schedule
    if name == "C1":
        _literal_interior(w, x, y, w.n * w.n * 2)


@pytest.mark.parametrize("layout", ["CG1xCG1", "DG1xDG1"])
@pytest.mark.parametrize("ordering", ["rcm", "random"])
@pytest.mark.parametrize("layers", [10, 20, 50, 100, 256])
def test_config4_sweep_at_full_size(layout, ordering, layers):
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.kernels import MassOperator
    w = configs.sweep_workload(layout, layers, ordering)
    fs, quad, x, coords = _build(w)
    if layers == 10:
        _check_mesh(fs, w)
    op = MassOperator(fs, quad)
    y = op.apply(torch.from_numpy(x).cuda(), coords).cpu().numpy()
    ref, _arm = _oracle_y(w, x)
    assert _rel(y, ref) <= _tol(layout), op.last_schedule


_C5 = {}


def _c5(name):
    """(workload, fs, quad, x, coords, oracle y) of C5a / C5b, cached."""
    if name not in _C5:
        from paper_1604_05937_b200 import configs
        _C5.clear()
        w = configs.WORKLOADS[name]
        fs, quad, x, coords = _build(w)
        _check_mesh(fs, w)
        ref, _arm = _oracle_y(w, x)
        _C5[name] = (w, fs, quad, x, coords, ref)
    return _C5[name]


@pytest.mark.parametrize("name", ["C5a", "C5b"])
@pytest.mark.parametrize("schedule", ["auto", "tile"])
def test_config5_one_gpu_at_full_size(name, schedule):
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.kernels import MassOperator
    if schedule == "tile" and not _lib.experimental():
        pytest.skip("tile schedule: library built without PM_EXPERIMENTAL")
    w, fs, quad, x, coords, ref = _c5(name)
    op = MassOperator(fs, quad)
    xd = torch.from_numpy(x).cuda()
    y = torch.full_like(xd, float("nan"))   # every DoF must be written
    op.apply(xd, coords, y, schedule=schedule)
    yh = y.cpu().numpy()
    assert _rel(yh, ref) <= 1e-10, op.last_schedule
    if schedule == "auto" and name == "C5a":
        _literal_interior(w, x, yh, 200000)
    del y, xd


@pytest.mark.parametrize("name", ["C5a", "C5b"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("halo", ["fused", "exchange"])
def test_config5_sharded_at_full_size(name, world, halo):
    """Every rank's column loop over its RCM cell block on one GPU, the
    ghost columns summed either by the fused kernel (peer REDs into the
    rank below's window, here a buffer on the same device) or by the
    exchange kernels (pm_halo_pack on the sender, pm_halo_unpack_add on
    the owner, the send/recv emulated by the device copy); the owned
    columns of all ranks together equal the oracle."""
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.shard import (ShardedMassOperator,
                                             fused_halo_plan, partition)
    w, fs, quad, x, coords, ref = _c5(name)
    m = fs.mesh
    plan = fused_halo_plan(fs, partition(fs, world))
    assert plan is not None
    ops = [ShardedMassOperator(fs, r, world, quad) for r in range(world)]
    wins = [torch.zeros(op.window[1] - op.window[0], dtype=torch.float64,
                        device="cuda") for op in ops]
    for r, op in enumerate(ops):
        lo, hi = op.window
        clo, chi = op.shard.coord_window
        xw = torch.from_numpy(x[lo:hi]).cuda()
        cw = coords[clo:chi]
        if halo == "fused":
            peer = (wins[r - 1].data_ptr() - 8 * ops[r - 1].window[0]) \
                if r else 0
            strips, W = op.strips
            _lib.column_mass_strip_red_peer(
                fs.layout, op.op.k, m.layers, cw, op.op.mref, xw, wins[r],
                hi - lo, strips, op.op.kron, W, peer, plan[r] if r else 0,
                accumulate=True, x_base=lo, y_base=lo, coords_base=clo,
                n_vertices=m.base.num_vertices)
        else:
            op.apply(xw, cw, wins[r], exchange=False)
        del xw
    if halo == "exchange":
        for op in ops:
            for q, lst in op.halo.send.items():
                for (_d, o, c) in lst:
                    buf = op.halo._cuda_pack(wins[op.rank], o, c)
                    ops[q].halo._cuda_unpack(wins[q], o, c, buf)
    torch.cuda.synchronize()
    got = np.empty_like(ref)
    col = fs.column_sizes[0]
    covered = 0
    for op, win in zip(ops, wins):
        own = op.shard.owned[0]
        # owned vertices of an RCM block: one contiguous range
        assert own.size and own[-1] - own[0] + 1 == own.size
        a, b = int(own[0]) * col, (int(own[-1]) + 1) * col
        lo = op.window[0]
        got[a:b] = win[a - lo:b - lo].cpu().numpy()
        covered += b - a
    assert covered == ref.size
    assert _rel(got, ref) <= 1e-10
