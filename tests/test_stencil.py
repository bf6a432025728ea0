"""User stencil kernels through iterate_columns (SPEC.md:322-341,
csrc/stencil.cu): CUDA C local kernels compiled by NVRTC into the column
loop.  CPU: compile checks and argument validation.  GPU: a user-written
mass kernel against the oracle, a nonlinear kernel against a brute-force
assembler over the materialised per-(cell, layer) DoF lists
(verification.py:47-75, the SPEC's equivalence property), the counting
kernel, and the colored schedule's bitwise determinism."""
import numpy as np
import pytest

from paper_1604_05937_b200 import (COORDS_LAYOUT, ExtrudedMesh,
                                   builtin_layout, extrude_coordinates,
                                   generate_unit_square_mesh, number_dofs)
from paper_1604_05937_b200.stencil import CudaStencilKernel

NONLINEAR = """
__device__ void pm_kernel(double *out, const double *const *in,
                          long long cell, int layer) {
  // out_j = x_j^2 + 0.25 * sum_i x_i + (cell % 7) + 0.5 * layer
  double s = 0.0;
  for (int i = 0; i < 6; ++i) s += in[0][i];
  for (int j = 0; j < 6; ++j)
    out[j] = in[0][j] * in[0][j] + 0.25 * s + (double)(cell % 7) +
             0.5 * layer;
}
"""

COUNT = """
__device__ void pm_kernel(double *out, const double *const *in,
                          long long cell, int layer) {
  out[0] = 1.0;
}
"""


def mass_source(mref):
    """The P1 prism mass kernel written by a user: |det J| from the 18
    coordinate slots (slot 6a + 3b + comp: vertex a, bottom/top b), times
    the reference mass matrix."""
    k = mref.shape[0]
    vals = ", ".join("%.17g" % v for v in np.asarray(mref).ravel())
    return f"""
__device__ const double M[{k * k}] = {{{vals}}};
__device__ void pm_kernel(double *out, const double *const *in,
                          long long cell, int layer) {{
  const double *x = in[0], *c = in[1];
  double xm[3], ym[3], h = 0.0;
  for (int a = 0; a < 3; ++a) {{
    xm[a] = 0.5 * (c[6 * a] + c[6 * a + 3]);
    ym[a] = 0.5 * (c[6 * a + 1] + c[6 * a + 4]);
    h += c[6 * a + 5] - c[6 * a + 2];
  }}
  const double a2 = (xm[1] - xm[0]) * (ym[2] - ym[0]) -
                    (xm[2] - xm[0]) * (ym[1] - ym[0]);
  const double det = fabs(a2 * (h / 3.0));
  for (int j = 0; j < {k}; ++j) {{
    double s = 0.0;
    for (int i = 0; i < {k}; ++i) s += M[j * {k} + i] * x[i];
    out[j] = det * s;
  }}
}}
"""


def test_compile_check_no_device():
    k = CudaStencilKernel(NONLINEAR, (6, 6))
    assert k.check() > 0


def test_compile_errors_are_reported():
    bad = CudaStencilKernel(
        "__device__ void pm_kernel(double *out, const double *const *in,"
        " long long cell, int layer) { out[0] = not_declared; }", (6, 6))
    with pytest.raises(ValueError, match="not_declared"):
        bad.check()


@pytest.mark.parametrize("arity", [(), (0, 6), (6, 65), (6,) * 10])
def test_bad_arity(arity):
    with pytest.raises(ValueError):
        CudaStencilKernel(NONLINEAR, arity).check()


def _mesh(n=6, layers=5):
    return ExtrudedMesh(generate_unit_square_mesh(n), layers)


@pytest.mark.gpu
def test_user_mass_kernel_matches_oracle():
    import torch
    import oracle
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.kernels import MassOperator
    m = _mesh(8, 6)
    fs = number_dofs(m, builtin_layout("CG1", "CG1"))
    cfs = number_dofs(m, COORDS_LAYOUT)
    op = MassOperator(fs)
    rng = np.random.default_rng(3)
    x = rng.random(fs.total_dofs)
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    k = CudaStencilKernel(mass_source(op.mref), (6, 18, 6))
    q = op.quadrature
    ref = oracle.Problem(m.base, m.layers, fs.layout.counts, "P1", "P1", 1,
                         q.tri_degree, q.line_degree).assemble(x)
    xd = torch.from_numpy(x).cuda()
    for sched in ("atomic", "colored"):
        out = torch.zeros_like(xd)
        iterate_columns([fs, cfs, fs], k, [xd, coords, out], schedule=sched)
        y = out.cpu().numpy()
        built = op.apply(xd, coords).cpu().numpy()
        assert np.abs(y - built).max() <= 1e-12 * np.abs(built).max()
        assert np.abs(y - ref).max() <= 1e-10 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", [("CG1", "CG1"), ("DG1", "CG1"),
                                    ("CG1", "DG1"), ("DG0", "DG1")])
def test_nonlinear_kernel_equals_materialised_lists(layout):
    import torch
    from paper_1604_05937_b200.iterate import iterate_columns
    from paper_1604_05937_b200.verification import materialized_cell_maps
    m = _mesh(5, 4)
    fs = number_dofs(m, builtin_layout(*layout))
    k6 = fs.num_slots
    src = NONLINEAR.replace("6", str(k6)) if k6 != 6 else NONLINEAR
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, fs.total_dofs)
    lists = materialized_cell_maps(fs)             # (N2, layers, k)
    ref = np.zeros(fs.total_dofs)
    for c in range(lists.shape[0]):
        for l in range(lists.shape[1]):
            d = lists[c, l]
            v = x[d]
            np.add.at(ref, d, v * v + 0.25 * v.sum() + (c % 7) + 0.5 * l)
    kern = CudaStencilKernel(src, (k6, k6))
    xd = torch.from_numpy(x).cuda()
    outs = {}
    for sched in ("atomic", "colored", "sequential"):
        out = torch.zeros_like(xd)
        iterate_columns([fs, fs], kern, [xd, out], schedule=sched)
        outs[sched] = out.cpu().numpy()
        assert np.abs(outs[sched] - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(outs["colored"], outs["sequential"])


@pytest.mark.gpu
def test_counting_kernel_visits_every_cell_layer_once():
    import torch
    from paper_1604_05937_b200.iterate import iterate_columns
    m = _mesh(7, 3)
    fs = number_dofs(m, builtin_layout("DG0", "DG0"))
    out = torch.zeros(fs.total_dofs, dtype=torch.float64, device="cuda")
    iterate_columns([fs], CudaStencilKernel(COUNT, (1,)), [out])
    o = out.cpu().numpy()
    assert np.all(o == 1.0) and o.sum() == m.base.num_cells * m.layers


@pytest.mark.gpu
def test_user_kernel_rejects_other_schedules():
    import torch
    from paper_1604_05937_b200.iterate import iterate_columns
    m = _mesh(3, 2)
    fs = number_dofs(m, builtin_layout("DG0", "DG0"))
    out = torch.zeros(fs.total_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="schedule"):
        iterate_columns([fs], CudaStencilKernel(COUNT, (1,)), [out],
                        schedule="stripred")
