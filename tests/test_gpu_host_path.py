"""The host-buffer path (kernels.mass_action with pinned host tensors):
copies pipelined with the compute, chunked by cell ranges / entity bands
for vertex and edge column layouts, by cell ranges for DG -- against the
oracle (needs a B200)."""
import numpy as np
import pytest

import oracle
from conftest import quad_degrees

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("lname", ["CG1xCG1", "VP1", "P2xP2", "CG1xDG1",
                                   "DG1xDG1"])
@pytest.mark.parametrize("ordering", ["rcm", "random"])
def test_host_buffers_pipelined(lname, ordering, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    monkeypatch.setenv("PM_HOST_CHUNK_MB", "0.01")   # many chunks
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.kernels import MassOperator, mass_action
    from paper_1604_05937_b200.quadrature import element_for_layout
    w = configs.Workload("host", 40, 11, lname, quad_degrees(lname), ordering)
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    el = element_for_layout(fs.layout)
    ref = oracle.Problem(m.base, m.layers, fs.layout.counts, el.tri, el.line,
                         el.ncomp, *quad_degrees(lname)).assemble(x)
    op = MassOperator(fs, quad)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.full((x.shape[0],), float("nan"),
                    dtype=torch.float64).pin_memory()
    for _ in range(2):
        mass_action(fs, xh, operator=op, out=yh)
        y = yh.numpy()
        tol = 1e-12 if lname.startswith("DG") else 1e-10
        assert np.abs(y - ref).max() <= tol * np.abs(ref).max()
    if ordering == "rcm" and lname not in ("DG1xDG1",):
        assert op._bands() is not None and len(op._bands()[1]) > 4
