"""Spectral analysis helpers on the CPU (SPEC.md:450-466 trivial examples)."""
import numpy as np
import pytest

from paper_1901_01685_b200 import analysis
from paper_1901_01685_b200._native import Csr


def test_spectral_radius_trivial():
    assert analysis.spectral_radius(np.zeros((4, 4))).rho == 0.0
    R = np.array([[0.0, -0.5], [0.5, 0.0]])  # rotation-like: eigenvalues +-0.5i
    s = analysis.spectral_radius(R)
    assert s.rho == pytest.approx(0.5) and np.iscomplexobj(s.eigenvalues)
    with pytest.raises(ValueError):
        analysis.spectral_radius(np.zeros((2, 3)))


def test_condition_number_trivial():
    assert analysis.condition_number(np.eye(5)) == pytest.approx(1.0)
    assert analysis.condition_number(np.diag([1.0, 10.0])) == pytest.approx(10.0)
    A = Csr(2, 2, np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.array([1.0, 10.0]))
    assert analysis.condition_number(A) == pytest.approx(10.0)


# ---- F3: generalized eigenpairs and reduction factors ----
from paper_1901_01685_b200 import problems as P  # noqa: E402


def test_generalized_eigs_trivial():
    A = np.diag([3.0, 1.0, 2.0])
    E = analysis.generalized_eigs(A, A)  # A = M -> all lambda = 1
    np.testing.assert_allclose(E.eigenvalues, 1.0, rtol=1e-14)
    E = analysis.generalized_eigs(np.diag([1.0, 2.0]), np.eye(2))
    np.testing.assert_allclose(E.eigenvalues, [1.0, 2.0])
    np.testing.assert_allclose(np.abs(E.eigenvectors), np.eye(2), atol=1e-15)
    with pytest.raises(ArithmeticError):  # M not SPD -> analysis error
        analysis.generalized_eigs(np.eye(2), np.diag([1.0, -1.0]))
    with pytest.raises(ValueError):
        analysis.generalized_eigs(np.eye(2), np.eye(3))


def test_generalized_eigs_benchmark1_residuals():
    """Benchmark 1 Laplacian, p=2, h=2^-5: ||A v - lambda M v|| < 1e-8 for all pairs
    (relative to ||A|| ||v||, the invariant of SPEC.md:413); eigenvalues ascending and positive."""
    pb = P.build(P.benchmark_spec(1, 2, 5))
    E = analysis.generalized_eigs(pb.plevels[0].A, P.matrix("M", geometry="annulus", p=2, nel=32))
    assert E.residuals().max() < 1e-8
    assert np.all(np.diff(E.eigenvalues) >= 0) and E.eigenvalues[0] > 0
    np.testing.assert_allclose(np.linalg.norm(E.eigenvectors, axis=0), 1.0, rtol=1e-13)


def test_generalized_eigs_nonsymmetric():
    """The CDR operator of Benchmark 2 is non-symmetric: general eigensolve, pairs still satisfy
    A v = lambda M v."""
    pb = P.build(P.benchmark_spec(2, 2, 3))
    M = P.matrix("M", geometry="square", p=2, nel=8)
    E = analysis.generalized_eigs(pb.plevels[0].A, M)
    assert E.residuals().max() < 1e-8
    assert np.all(np.diff(E.eigenvalues.real) >= 0)


def _oracle_factors(pb, smoother, which, **kw):
    from oracle import oracle as O  # checker: the GPU path is tests/test_gpu_analysis.py
    E = analysis.generalized_eigs(pb.plevels[0].A, P.matrix("M", geometry="annulus", p=pb.spec["degrees"][0],
                                                             nel=2 ** pb.spec["h_exp"]))
    Ho = O.Hierarchy(pb, smoother=smoother, **kw)
    f = np.zeros(pb.n)
    step = Ho.smooth if which == "smoother" else Ho.coarse_correction
    return E, analysis._reduction(lambda v: step(v, f), E.eigenvectors, range(pb.n), 1)


def test_reduction_factors_exact_smoother_is_zero():
    """ILUT with tau = 0 and full fill (an exact LU) -> smoother factors ~ 0."""
    from oracle import oracle as O
    pb = P.build(P.benchmark_spec(1, 2, 4))
    _, rs = _oracle_factors(pb, O.ILUT, "smoother", tau=0.0, fillfactor=8.0)
    assert rs.max() < 1e-10, rs.max()


def test_reduction_factors_gs_vs_ilut_benchmark1():
    """Benchmark 1, p=4, h=2^-5: the max smoother factor of Gauss-Seidel over the upper
    half of the spectrum exceeds the ILUT counterpart by >= 10x; the coarse-grid correction reduces
    the lowest modes strongly (PAPER Fig. 3)."""
    from oracle import oracle as O
    pb = P.build(P.benchmark_spec(1, 4, 5))
    n = pb.n
    _, rs_gs = _oracle_factors(pb, O.GS, "smoother")
    _, rs_il = _oracle_factors(pb, O.ILUT, "smoother")
    assert rs_gs[n // 2:].max() >= 10 * rs_il[n // 2:].max(), (rs_gs[n // 2:].max(), rs_il[n // 2:].max())
    _, rc = _oracle_factors(pb, O.ILUT, "cgc")
    assert np.all(rc >= 0) and rc[:10].max() < 0.5 and np.median(rc[n // 2:]) > 0.9
