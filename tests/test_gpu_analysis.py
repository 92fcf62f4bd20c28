"""F3: the iteration matrix built from GPU cycles equals the
oracle's column by column, bit for bit, is linear, and has the spectral radii the
paper reports in order of magnitude."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_01685_b200 import analysis, pmg
from paper_1901_01685_b200 import problems as P

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("smoother", ["ilut", "gs"])
def test_iteration_matrix_equals_oracle(smoother):
    pb = P.build(P.benchmark_spec(1, 2, 4))
    H = pmg.build_hierarchy(pb, smoother=smoother)
    M = analysis.iteration_matrix(H, workers=4)
    Ho = O.Hierarchy(pb, smoother=O.ILUT if smoother == "ilut" else O.GS)
    n = pb.n
    f = np.zeros(n)
    for i in range(0, n, max(1, n // 24)):  # a spread of columns against the oracle's cycle
        e = np.zeros(n)
        e[i] = 1.0
        np.testing.assert_array_equal(_bits(M[:, i]), _bits(Ho.cycle(e, f)), err_msg=f"column {i}")
    u0 = np.random.default_rng(0).uniform(-1, 1, n)  # linearity
    u1 = pmg.cycle(H, 0, u0, f)
    assert np.linalg.norm(u1 - M @ u0) <= 1e-10 * max(np.linalg.norm(u1), 1.0)
    rho = analysis.spectral_radius(M).rho
    assert 0.0 < rho < (0.2 if smoother == "ilut" else 1.0), rho


def test_spectral_radius_benchmark2_ilut_small():
    """Benchmark 2, p=4, h=2^-5, ILUT -> rho ~ 0.020 (order of magnitude)."""
    pb = P.build(P.benchmark_spec(2, 4, 5))
    if pb.n > 2500:
        pytest.skip("dense storage bound")
    H = pmg.build_hierarchy(pb, smoother="ilut")
    rho = analysis.spectral_radius(analysis.iteration_matrix(H, workers=8)).rho
    assert rho < 0.2, rho
