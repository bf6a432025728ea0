"""The run-strip schedule ("striptma", csrc/strip_tma.cu): strips along the
vertex-id bands of a level-ordered mesh (pm_build_run_strips) and the strip
kernel fed by bulk copies of whole vertex columns.

CPU: the planner covers every cell once with valid sequential strips, and on
RCM split-square meshes nearly every step continues its side's id run.
GPU: oracle parity (1e-10, CG) for P1 and 3-vector P1 at 1-4 layer chunks,
partial chunks, RCM and random vertex orders (random = the one-copy-per-
column fallback), strips longer than the ring, and the last vertex of the
mesh (the copy that would reach past the arrays' end)."""
import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees


def _rcm_mesh(n, ordering="rcm", seed=0):
    import os
    os.environ.setdefault("PM_DEVICE_MESH", "0")
    from paper_1604_05937_b200 import configs
    base, _ = configs.base_mesh(n, ordering, 0.0, seed)
    return base


def _check_strips(base, sp, st):
    """Every cell once; consecutive steps of a strip form mesh cells."""
    cells = {tuple(sorted(c)): i
             for i, c in enumerate(np.asarray(base.cell_vertices).tolist())}
    seen = np.zeros(len(cells), dtype=np.int64)
    for s in range(len(sp) - 1):
        v = st[sp[s]:sp[s + 1]]
        assert len(v) >= 3
        for k in range(len(v) - 2):
            seen[cells[tuple(sorted(v[k:k + 3].tolist()))]] += 1
    assert np.all(seen == 1)


@pytest.mark.parametrize("n,ordering", [(6, "rcm"), (24, "rcm"),
                                        (12, "random")])
def test_run_strips_cover_every_cell_once(n, ordering):
    from paper_1604_05937_b200 import _lib
    base = _rcm_mesh(n, ordering)
    sp, st = _lib.build_global_strips(base, max_len=40, runs=True,
                                      order="creation")
    _check_strips(base, sp, st)
    sp2, st2 = _lib.build_global_strips(base, max_len=40, runs=True)
    _check_strips(base, sp2, st2)      # Morton-ordered strips: same cover


def test_run_strips_follow_the_id_bands():
    """On an RCM split-square mesh both sides of a run strip are runs of
    consecutive vertex ids (contiguous column slabs under Alg. 1)."""
    from paper_1604_05937_b200 import _lib
    base = _rcm_mesh(48)
    sp, st = _lib.build_global_strips(base, max_len=512, runs=True)
    inner = len(st) - 2 * (len(sp) - 1)
    frac = float((st[2:] == st[:-2] + 1).sum()) / inner
    assert frac > 0.95
    # the plain strips of the same mesh cross the bands
    sp0, st0 = _lib.build_global_strips(base, max_len=512)
    assert float((st0[2:] == st0[:-2] + 1).sum()) / len(st0) < 0.1


gpu = pytest.mark.gpu


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
    return prob.assemble_colored(f) if hasattr(prob, "assemble_colored") \
        else prob.assemble(f)


def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


@gpu
@pytest.mark.parametrize("lname", ["CG1xCG1", "VP1"])
@pytest.mark.parametrize("layers", [1, 7, 32, 33, 64, 70, 100, 128, 192, 256])
def test_striptma_matches_oracle_rcm(lname, layers):
    if layers > 128 and lname != "CG1xCG1":
        pytest.skip("3-vector columns: at most 128 layers")
    _need_cuda()
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.quadrature import prism_quadrature
    base = _rcm_mesh(40)
    fs = _space(base, layers, lname)
    op = kernels.MassOperator(fs, prism_quadrature(*quad_degrees(lname)),
                              schedule="striptma")
    f = np.random.default_rng(layers).uniform(-1, 1, fs.total_dofs)
    got = kernels.mass_action(fs, f, operator=op, schedule="striptma")
    assert op.last_schedule == "striptma"
    assert _rel(got, _oracle(base, layers, lname, f)) <= 1e-10


@gpu
@pytest.mark.parametrize("lname", ["CG1xCG1", "VP1"])
@pytest.mark.parametrize("env", [{"PM_TMA_NQ": "1"}, {"PM_TMA_GROUPS": "1"},
                                 {"PM_TMA_NQ": "1", "PM_TMA_GROUPS": "2"}])
def test_striptma_ring_shapes(lname, env, monkeypatch):
    """One chunk per warp (scalar columns default to two), one / two groups
    per CTA."""
    _need_cuda()
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.quadrature import prism_quadrature
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    base = _rcm_mesh(40)
    fs = _space(base, 64, lname)
    f = np.random.default_rng(5).uniform(-1, 1, fs.total_dofs)
    got = kernels.mass_action(
        fs, f, quadrature=prism_quadrature(*quad_degrees(lname)),
        schedule="striptma")
    assert _rel(got, _oracle(base, 64, lname, f)) <= 1e-10


@gpu
@pytest.mark.parametrize("lname", ["CG1xCG1", "VP1"])
def test_striptma_random_order_falls_back_to_single_columns(lname):
    """A random vertex order has no id runs: every column by its own copy."""
    _need_cuda()
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.quadrature import prism_quadrature
    base = _rcm_mesh(24, "random", seed=3)
    fs = _space(base, 40, lname)
    op = kernels.MassOperator(fs, prism_quadrature(*quad_degrees(lname)),
                              schedule="striptma")
    assert op._run_strips()[1] < 0.2
    f = np.random.default_rng(9).uniform(-1, 1, fs.total_dofs)
    got = kernels.mass_action(fs, f, operator=op, schedule="striptma")
    assert _rel(got, _oracle(base, 40, lname, f)) <= 1e-10


@gpu
def test_striptma_accumulates_and_repeats():
    """accumulate=True adds to y; repeated applies give the same result
    (mbarrier phases and stage counters carry over between strips)."""
    _need_cuda()
    import torch
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.quadrature import prism_quadrature
    base = _rcm_mesh(64)
    fs = _space(base, 64, "CG1xCG1")
    op = kernels.MassOperator(fs, prism_quadrature(*quad_degrees("CG1xCG1")),
                              schedule="striptma")
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    f = np.random.default_rng(1).uniform(-1, 1, fs.total_dofs)
    x = torch.from_numpy(f).cuda()
    y1 = op.apply(x, coords).clone()
    y2 = op.apply(x, coords).clone()
    ref = _oracle(base, 64, "CG1xCG1", f)
    assert _rel(y1.cpu().numpy(), ref) <= 1e-10
    assert _rel(y2.cpu().numpy(), ref) <= 1e-10
    y3 = y1.clone()
    op.apply(x, coords, y3, accumulate=True)
    assert _rel(y3.cpu().numpy(), 2 * ref) <= 1e-10


@gpu
@pytest.mark.parametrize("lname", ["CG1xCG1", "VP1"])
@pytest.mark.parametrize("n,max_len,groups,layers", [
    (64, 512, None, 64),    # strips of many granules, one per group
    (96, 37, "1", 64),      # several strips per group (stage counters and
                            # mbarrier phases carry over), ragged lengths
    (96, 50, "2", 100),     # two / four warps per group
    (64, 41, "1", 20),      # one chunk
])
def test_striptma_long_and_many_strips(lname, n, max_len, groups, layers,
                                       monkeypatch):
    _need_cuda()
    from paper_1604_05937_b200 import kernels
    from paper_1604_05937_b200.quadrature import prism_quadrature
    monkeypatch.setattr(kernels, "run_strip_max_len", lambda nc, l: max_len)
    if groups:
        monkeypatch.setenv("PM_TMA_GROUPS", groups)
    base = _rcm_mesh(n)
    fs = _space(base, layers, lname)
    op = kernels.MassOperator(fs, prism_quadrature(*quad_degrees(lname)),
                              schedule="striptma")
    (sp, _st), frac = op._run_strips()
    lens = np.diff(sp.cpu().numpy())
    assert lens.max() > 12 and frac > 0.8
    if groups:
        assert len(lens) > 148 * int(groups)
    f = np.random.default_rng(n).uniform(-1, 1, fs.total_dofs)
    got = kernels.mass_action(fs, f, operator=op, schedule="striptma")
    assert _rel(got, _oracle(base, layers, lname, f)) <= 1e-10
