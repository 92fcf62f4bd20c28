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


@pytest.mark.parametrize("smoother,degrees", [("ilut", (3, 2, 1)), ("gs", (3, 2, 1)), ("ilut", (2, 1))])
def test_smooth_and_coarse_correction_equal_oracle(smoother, degrees):
    """pmg_smooth / pmg_coarse_correction (the halves of the cycle) are bitwise
    equal to the oracle's at every p-level, including the p = 1 level (h-level 0 ILUT smoother)."""
    p = degrees[0]
    spec = P.benchmark_spec(1, p, 4, consecutive=len(degrees) > 2)
    pb = P.build(spec)
    H = pmg.build_hierarchy(pb, smoother=smoother)
    Ho = O.Hierarchy(pb, smoother=O.ILUT if smoother == "ilut" else O.GS)
    rng = np.random.default_rng(1)
    for level, lev in enumerate(pb.plevels):
        n = lev.A.nrows
        u = rng.uniform(-1, 1, n)
        f = rng.uniform(-1, 1, n)
        np.testing.assert_array_equal(_bits(pmg.smooth(H, level, u, f)), _bits(Ho.smooth(u, f, level)))
        if level + 1 < len(pb.plevels):
            np.testing.assert_array_equal(_bits(pmg.coarse_correction(H, level, u, f)),
                                          _bits(Ho.coarse_correction(u, f, level)))
    with pytest.raises(ValueError):  # PMG_ERR_ARG: the last p-level has no coarser level
        pmg.coarse_correction(H, len(pb.plevels) - 1, np.zeros(pb.plevels[-1].A.nrows), np.zeros(pb.plevels[-1].A.nrows))


def test_reduction_factors_benchmark1_p4():
    """SPEC.md:437 on the GPU path: Benchmark 1, p=4, h=2^-5 -- the max GS smoother factor over the
    upper half of the spectrum is >= 10x ILUT's; every factor equals the one computed from the
    oracle's smoothing step / coarse-grid correction (the same arithmetic, bit for bit)."""
    pb = P.build(P.benchmark_spec(1, 4, 5))
    n = pb.n
    E = analysis.generalized_eigs(pb.plevels[0].A, P.matrix("M", geometry="annulus", p=4, nel=32))
    out = {}
    for sm in ("ilut", "gs"):
        H = pmg.build_hierarchy(pb, smoother=sm)
        out[sm] = analysis.reduction_factors(H, E, "smoother", workers=4).factors
        if sm == "ilut":
            cg = analysis.reduction_factors(H, E, "cgc", workers=4)
            Ho = O.Hierarchy(pb, smoother=O.ILUT)
            f = np.zeros(n)
            sel = np.arange(0, n, 37)
            ref = analysis._reduction(lambda v: Ho.coarse_correction(v, f), E.eigenvectors, sel, 1)
            np.testing.assert_array_equal(cg.factors[sel], ref)
            assert cg.factors[:10].max() < 0.5
    assert out["gs"][n // 2:].max() >= 10 * out["ilut"][n // 2:].max()
    with pytest.raises(ValueError):
        analysis.reduction_factors(H, E, "both")
