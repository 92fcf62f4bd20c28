"""Host discretization (input generation): SPEC.md `splines` and `discretization` examples
and invariants, and the BASELINE config sizes."""
import math

import numpy as np
import pytest

from paper_1901_01685_b200 import problems as P


# ---------------------------------------------------------------- splines
def test_find_span_examples():
    # kv = {0,0,0.5,1,1}, p=1: xi=0.25 -> first span; xi=1 -> right-closed last span
    first, N = P.eval_basis(1, 2, 0.25)
    assert first == 0
    np.testing.assert_allclose(N, [0.5, 0.5], rtol=0, atol=1e-15)  # hat values
    first, N = P.eval_basis(1, 2, 1.0)
    assert first == 1 and N[-1] == 1.0
    with pytest.raises(ValueError):
        P.eval_basis(1, 2, 1.5)  # domain error


def test_derivative_examples():
    first, N, dN = P.eval_basis(1, 2, 0.25, deriv=True)
    np.testing.assert_allclose(dN, [-2.0, 2.0], atol=1e-14)
    _, N0 = P.eval_basis(0, 4, 0.3)
    assert N0.tolist() == [1.0]  # p = 0: piecewise constant


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("spans", [4, 8, 16, 32, 64])
def test_partition_of_unity_and_derivative_sum(p, spans):
    rng = np.random.default_rng(p * 100 + spans)
    for x in rng.uniform(0, 1, 200):
        _, N, dN = P.eval_basis(p, spans, float(x), deriv=True)
        assert N.size == p + 1 and (N >= -1e-15).all()
        assert abs(N.sum() - 1.0) < 1e-13
        assert abs(dN.sum()) < 1e-12 * spans


def test_derivative_matches_finite_difference():
    p, spans, eps = 2, 4, 1e-6
    for x in (0.1, 0.33, 0.6, 0.9):
        f0, N, dN = P.eval_basis(p, spans, x, deriv=True)
        fa, Na = P.eval_basis(p, spans, x + eps)
        fb, Nb = P.eval_basis(p, spans, x - eps)
        assert fa == fb == f0
        np.testing.assert_allclose(dN, (Na - Nb) / (2 * eps), rtol=1e-6, atol=1e-6)


# ---------------------------------------------------------------- geometry
def test_identity_map():
    X, J = P.geometry_map("square", 0, 0.3, 0.7)
    np.testing.assert_allclose(X, [0.3, 0.7], atol=1e-15)
    np.testing.assert_allclose(J, np.eye(2), atol=1e-15)


def test_quarter_annulus_is_exact():
    for eta in np.linspace(0, 1, 11):
        for xi, r in ((0.0, 1.0), (1.0, 2.0)):
            X, J = P.geometry_map("annulus", 0, xi, float(eta))
            assert abs(np.hypot(*X) - r) < 1e-12
            assert np.linalg.det(J) > 0
    X, _ = P.geometry_map("annulus", 0, 0.0, 0.0)
    np.testing.assert_allclose(X, [1, 0], atol=1e-15)
    X, _ = P.geometry_map("annulus", 0, 0.0, 1.0)
    np.testing.assert_allclose(X, [0, 1], atol=1e-15)


def test_lshape_patch_corners():
    corners = {0: ((-1, 0), (0, 1)), 1: ((-1, -1), (0, 0)), 2: ((0, -1), (1, 0))}
    for patch, (lo, hi) in corners.items():
        X0, _ = P.geometry_map("lshape", patch, 0, 0)
        X1, _ = P.geometry_map("lshape", patch, 1, 1)
        np.testing.assert_allclose(X0, lo, atol=1e-15)
        np.testing.assert_allclose(X1, hi, atol=1e-15)


# ---------------------------------------------------------------- assembly
def test_single_element_mass_and_lumping():
    M = P.matrix("M", "square", p=1, nel=1).to_dense()
    ref = np.array([[4, 2, 2, 1], [2, 4, 1, 2], [2, 1, 4, 2], [1, 2, 2, 4]]) / 36.0
    np.testing.assert_allclose(M, ref, rtol=0, atol=1e-15)
    _, ml = P.matrix("ML", "square", p=1, nel=1)
    np.testing.assert_allclose(ml, 0.25, atol=1e-15)


@pytest.mark.parametrize("geometry,area", [("square", 1.0), ("annulus", 3 * math.pi / 4), ("lshape", 3.0)])
def test_mass_sums_to_area(geometry, area):
    # SPEC.md:148.  Exact for the affine maps; on the NURBS annulus the (p+1)-point rule does
    # not integrate the rational Jacobian exactly (error ~ h^(2p+2)), hence the finer mesh there.
    M = P.matrix("M", geometry, p=2, nel=16 if geometry == "annulus" else 8)
    assert (M.val >= 0).all()
    assert abs(M.val.sum() - area) < 1e-10


def test_mass_is_spd_on_annulus():
    M = P.matrix("M", "annulus", p=2, nel=16).to_dense()
    np.linalg.cholesky(M)


def test_poisson_operator_symmetric():
    for geometry in ("square", "annulus", "lshape"):
        A, _ = P.matrix("A", geometry, p=3, nel=4)
        D = A.to_dense()
        assert np.abs(D - D.T).max() / np.abs(D).max() < 1e-10


def test_reaction_rows_sum_to_integrals():
    # pure reaction (D = 0, v = 0, R = 1) without boundary terms is the mass matrix
    A, _ = P.matrix("A", "square", p=2, nel=4, D=(0, 0, 0, 0), R=1.0, nitsche_scale=1e-300)
    M = P.matrix("M", "square", p=2, nel=4)
    np.testing.assert_allclose(A.to_dense(), M.to_dense(), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("pf,pc", [(2, 1), (3, 2), (5, 1)])
def test_transfer_preserves_constants(pf, pc):
    Pm = P.matrix("P", "annulus", p=pf, p2=pc, nel=8)
    _, mlf = P.matrix("ML", "annulus", p=pf, nel=8)
    Pd = Pm.to_scipy()
    np.testing.assert_allclose(Pd @ np.ones(Pm.ncols) / mlf, 1.0, atol=1e-10)


def test_config_sizes_match_survey_appendix_a():
    pb = P.build(1)
    assert [l.A.nrows for l in pb.plevels] == [1156, 1089]
    assert [l.A.nnz for l in pb.plevels] == [26896, 9409]
    assert pb.plevels[0].P.nnz == 16900
    assert [h.A.nrows for h in pb.hlevels] == [1089, 289, 81, 25]
    for deg, n, nnz, pnnz in ((2, 16900, 414736, 264196), (3, 17161, 819025, 413449), (4, 17424, 1364224, 595984)):
        pb = P.build(2, deg)
        assert (pb.n, pb.plevels[0].A.nnz, pb.plevels[0].P.nnz) == (n, nnz, pnnz)
        assert len(pb.hlevels) == 6
    pb = P.build(3)
    assert [l.A.nrows for l in pb.plevels] == [67081, 66564, 66049]
    assert [l.A.nnz for l in pb.plevels] == [3243601, 1648656, 591361]
    assert [l.P.nnz for l in pb.plevels[:-1]] == [2377764, 1052676]
    assert len(pb.hlevels) == 7


def test_config4_multipatch_glue():
    pb = P.build(4)
    assert pb.n == 3 * 67600 - 2 * 260  # 202,280
    assert pb.plevels[1].A.nrows == 3 * 257 * 257 - 2 * 257
    assert pb.hlevels[-1].A.nrows == 3 * 25 - 2 * 5  # dense coarsest level


def test_seeded_initial_guess():
    s = P.config_spec(3)
    pb1 = P.build(3)
    u = pb1.u0
    assert u.min() >= -1 and u.max() < 1
    assert abs(u.mean()) < 0.01
    # splitmix64 stream from seed 0, first value by hand
    z = (0 + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    z ^= z >> 31
    assert u[0] == (z >> 11) * 2.0**-53 * 2.0 - 1.0
    assert s.seed == 0


def test_b1_source_is_minus_laplacian_of_exact_solution():
    # u = -(r^2-1)(r^2-4) x y^2; check f = -lap u by finite differences
    u = lambda x, y: -((x * x + y * y) - 1) * ((x * x + y * y) - 4) * x * y * y
    f = lambda x, y: 2 * x * ((x * x + y * y) ** 2 - 5 * (x * x + y * y) + 4) + x * y * y * (40 * (x * x + y * y) - 80)
    h = 1e-4
    for x, y in ((1.2, 0.5), (0.3, 1.5), (1.0, 1.0)):
        lap = (u(x + h, y) + u(x - h, y) + u(x, y + h) + u(x, y - h) - 4 * u(x, y)) / h**2
        assert abs(-lap - f(x, y)) < 1e-4 * max(1, abs(f(x, y)))
