"""GPU parity on the large BASELINE configs against the committed oracle outputs
(tests/golden/golden.json: generating them takes the single-core oracle ~8 min at config 5),
plus error paths and edge cases.  Bitwise: same cycle counts, residual histories as hex floats,
SHA-256 of the solution and of the ILUT factors."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_01685_b200 import pmg
from paper_1901_01685_b200 import problems as P
from paper_1901_01685_b200._native import Csr

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def check_against_golden(pb, key, smoother):
    rec = golden()[key]
    H = pmg.build_hierarchy(pb, smoother=smoother)
    u, rep = pmg.solve(H, pb.f, guess=pb.u0)
    assert rep.cycles == rec["cycles"]
    assert rep.converged == rec["converged"] and rep.diverged == rec["diverged"]
    assert [float(x).hex() for x in rep.residual_history] == rec["residual_history"]
    assert sha(u) == rec["u_sha256"]
    for F, g in zip(H.factors(), rec["factors"]):
        L, U, perm = F.export()
        st = F.stats()
        assert (st["nnz_L"], st["nnz_U"], st["levels_L"], st["levels_U"]) == \
               (g["nnz_L"], g["nnz_U"], g["levels_L"], g["levels_U"])
        assert sha(L.rowptr, L.col, L.val) == g["sha_L"]
        assert sha(U.rowptr, U.col, U.val) == g["sha_U"]
    return rep


@pytest.mark.slow
def test_config4_lshape_against_golden():
    check_against_golden(P.build(4), "config4/ilut/none", "ilut")


@pytest.mark.slow
def test_config5_ilut_against_golden():
    rep = check_against_golden(P.build(5), "config5/ilut/none", "ilut")
    assert rep.converged


@pytest.mark.slow
def test_config5_gauss_seidel_diverges_like_oracle():
    rep = check_against_golden(P.build(5), "config5/gs/none", "gs")
    assert rep.diverged  # PAPER.md:537 reports divergence for p >= 4 with GS


# ---------------------------------------------------------------- error paths
def test_zero_pivot_row_matches_oracle():
    A = Csr.from_dense(np.array([[1.0, 1, 0, 0], [1, 1, 0, 0], [0, 0, 2, 1], [0, 0, 1, 2]]))
    with pytest.raises(O.OracleError) as eo:
        O.ilut_factorize(A, 0.0, 5.0, O.ORDER_NONE)
    with pytest.raises(pmg.FactorizationError) as eg:
        pmg.ilut_factorize(A, 0.0, 5.0, "none")
    assert eg.value.row == eo.value.row == 1


def test_gs_zero_diagonal_row():
    A = Csr.from_dense(np.array([[2.0, 1, 0], [1, 0, 1], [0, 1, 2]]))
    with pytest.raises(pmg.SmootherError) as e:
        pmg.gauss_seidel_sweep(A, np.zeros(3), np.ones(3))
    assert e.value.row == 1


def test_dimension_mismatch():
    A = Csr.from_dense(np.eye(3))
    with pytest.raises(pmg.DimensionError):
        pmg.spmv(A, np.ones(4))


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 257])
def test_tiny_and_ragged_sizes(n):
    rng = np.random.default_rng(n)
    D = np.diag(rng.uniform(2, 3, n)) + np.diag(rng.uniform(-1, 1, max(n - 1, 0)), 1) + \
        np.diag(rng.uniform(-1, 1, max(n - 1, 0)), -1)
    A = Csr.from_dense(D)
    x = rng.uniform(-1, 1, n)
    assert np.array_equal(pmg.spmv(A, x).view(np.uint64), O.spmv(A, x).view(np.uint64))
    for ordering, oo in (("none", O.ORDER_NONE), ("rcm", O.ORDER_RCM)):
        Fg, Fo = pmg.ilut_factorize(A, 1e-12, 1.0, ordering), O.ilut_factorize(A, 1e-12, 1.0, oo)
        assert np.array_equal(pmg.ilut_apply(Fg, x).view(np.uint64), Fo.apply(x).view(np.uint64))
    assert np.array_equal(pmg.gauss_seidel_sweep(A, x, x).view(np.uint64),
                          O.gauss_seidel_sweep(A, x, x).view(np.uint64))


def test_explicit_zeros_and_empty_rows_in_offdiagonal():
    D = np.array([[4.0, 0.0, 1.0], [0.0, 3.0, 0.0], [1.0, 0.0, 5.0]])
    A = Csr.from_arrays(3, 3, [0, 3, 4, 6], [0, 1, 2, 1, 0, 2], [4.0, 0.0, 1.0, 3.0, 1.0, 5.0])  # explicit 0
    x = np.array([1.0, -2.0, 0.5])
    assert np.array_equal(pmg.spmv(A, x), O.spmv(A, x))
    Fg, Fo = pmg.ilut_factorize(A, 0.0, 3.0, "none"), O.ilut_factorize(A, 0.0, 3.0, O.ORDER_NONE)
    for X, Y in zip(Fg.export()[:2], Fo.export()[:2]):
        assert np.array_equal(X.col, Y.col) and np.array_equal(X.val.view(np.uint64), Y.val.view(np.uint64))
    np.testing.assert_allclose(D @ pmg.ilut_apply(Fg, x), x, rtol=1e-14)


def test_zero_rhs_solve_is_zero():
    pb = P.build(1)
    H = pmg.build_hierarchy(pb)
    u, rep = pmg.solve(H, np.zeros(pb.n), guess=np.zeros(pb.n))
    assert rep.cycles == 0 and rep.converged and not u.any()


def test_transfers_bitwise():
    pb = P.build(P.make_spec("annulus", "one", (3, 2, 1), 4))
    H = pmg.build_hierarchy(pb)
    rng = np.random.default_rng(3)
    for l in range(2):
        fine, coarse = pb.plevels[l], pb.plevels[l + 1]
        vc = rng.uniform(-1, 1, coarse.A.nrows)
        rf = rng.uniform(-1, 1, fine.A.nrows)
        assert np.array_equal(pmg.prolongate(H, l, vc, fine.A.nrows), O.prolongate(fine.P, fine.ML, vc))
        assert np.array_equal(pmg.restrict(H, l, rf, coarse.A.nrows), O.restrict(fine.PT, coarse.ML, rf))


def test_cycle_bitwise_and_deterministic():
    pb = P.build(P.make_spec("square", "one", (3, 2, 1), 5, v=(2, 3), R=3))
    Hg, Ho = pmg.build_hierarchy(pb), O.Hierarchy(pb)
    rng = np.random.default_rng(4)
    u, f = rng.uniform(-1, 1, pb.n), rng.uniform(-1, 1, pb.n)
    a, b = pmg.cycle(Hg, 0, u, f), pmg.cycle(Hg, 0, u, f)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.array_equal(a.view(np.uint64), Ho.cycle(u, f).view(np.uint64))
