"""The bench's CPU baseline arm (oracle/fast.py, cpu_fast.c) against the
literal-quadrature oracle: same element matrix, same results (CPU only)."""
import numpy as np
import pytest

import oracle
from oracle import fast

CASES = [  # (layout counts, tri, line, ncomp, quad degrees)
    ({(0, 0): 1}, "P1", "P1", 1, (4, 4)),              # CG1 x CG1 (C1, C5a)
    ({(2, 1): 6}, "P1", "P1", 1, (2, 2)),              # DG1 x DG1 (C2)
    ({(0, 0): 1, (0, 1): 1, (1, 0): 1, (1, 1): 1}, "P2", "P2", 1, (6, 6)),
    ({(0, 0): 3}, "P1", "P1", 3, (2, 2)),              # 3-vector P1 (C5b)
    ({(0, 1): 1}, "P1", "P0", 1, (2, 2)),              # CG1 x DG0
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("ordering", ["rcm", "random"])
def test_fast_arm_matches_literal_oracle(case, ordering):
    counts, tri, line, nc, quad = CASES[case]
    base, rng = oracle.base_mesh(12, ordering, 0.3 if ordering == "random"
                                 else 0.0, seed=3)
    layers = 7
    prob = oracle.Problem(base, layers, counts, tri, line, nc, *quad)
    x = rng.random(prob.total)
    ref = prob.assemble(x)
    arm = fast.FastMass(base, layers, counts, tri, line, nc, *quad,
                        threads=3)
    y = arm.apply(x).copy()
    assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max()
    # a second call overwrites (zeroes first)
    assert np.array_equal(arm.apply(x), y)


def test_reference_matrix_is_symmetric_and_integrates_one():
    M = fast.reference_matrix({(0, 0): 1}, "P1", "P1", 1, 2, 2)
    assert np.allclose(M, M.T, atol=1e-15)
    # reference prism volume 1/2: sum of all entries = integral of 1
    assert abs(M.sum() - 0.5) < 1e-14


def test_cpu_info():
    phys, logical, model = fast.cpu_info()
    assert 1 <= phys <= logical and isinstance(model, str)
