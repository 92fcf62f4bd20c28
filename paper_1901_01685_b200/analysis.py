"""Spectral analysis of the p-multigrid cycle (the `analysis` module; PAPER §4;
SURVEY §8(f) F3): the iteration matrix column by column on the GPU, its spectral radius and
eigenvalue cloud, and condition numbers.

    generalized_eigs(A, M)  dense generalized eigenpairs A v = lambda M v by the
                            Cholesky reduction M = C C^T; symmetric or general eigensolve.
    reduction_factors(hier, eig, which)
                            per-mode r_S(v_j) = ||S(v_j)|| / ||v_j|| for one smoothing step or one
                            coarse-grid correction from u0 = v_j, f = 0 (PAPER
                            Eq. (32), Fig. 3), every application a GPU call (pmg_smooth /
                            pmg_coarse_correction), modes spread over host threads.
    iteration_matrix(hier)  column i = one V-cycle from u0 = e_i with f = 0: the
                            stationary error propagator.  Columns are independent, so they are
                            spread over `workers` host threads, each with its own work object
                            (its own vectors and stream) on the shared, immutable hierarchy.
    spectral_radius(M)      complex eigenvalues by a general dense eigensolver; rho = max modulus.
    condition_number(A)     ratio of the extreme singular values (dense SVD).

The cycle is the solve path's own (`pmg_cycle`, bitwise equal to the oracle's), so the matrix is
exactly the oracle's iteration matrix (tests/test_gpu_analysis.py)."""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import pmg


@dataclass
class GeneralizedEigenSystem:
    """A v_i = lambda_i M v_i: eigenvalues ascending (by real part), unit
    2-norm eigenvectors as columns, and the pair (A, M) they satisfy."""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    A: np.ndarray
    M: np.ndarray

    def residuals(self) -> np.ndarray:
        """||A v_i - lambda_i M v_i|| / (||A|| ||v_i||) per pair (the SPEC's invariant)."""
        V, lam = self.eigenvectors, self.eigenvalues
        R = self.A @ V - (self.M @ V) * lam[None, :]
        return np.linalg.norm(R, axis=0) / (np.linalg.norm(self.A, 2) * np.linalg.norm(V, axis=0))


@dataclass
class ReductionProfile:
    """r(v_j) per mode j for one part of the cycle; all factors >= 0."""
    which: str
    modes: np.ndarray      # mode indices j into the eigensystem
    factors: np.ndarray    # ||part(v_j)||_2 / ||v_j||_2


@dataclass
class Spectrum:
    rho: float
    eigenvalues: np.ndarray  # complex, the eigenvalue cloud (PAPER Figs. 5-6)


def generalized_eigs(A, M, max_dof: int = 5000) -> GeneralizedEigenSystem:
    """Full dense generalized eigendecomposition A v = lambda M v.  pre: M SPD,
    N_dof <= max_dof.  M = C C^T (Cholesky); the symmetric problem C^-1 A C^-T w = lambda w is
    solved by a symmetric eigensolver when A is symmetric, by a general one otherwise (complex
    pairs for the convection-dominated operator); v = C^-T w, scaled to unit 2-norm.  M not SPD
    raises ArithmeticError (the SPEC's analysis error)."""
    import scipy.linalg as sl

    Ad = A if isinstance(A, np.ndarray) else _dense(A)
    Md = M if isinstance(M, np.ndarray) else _dense(M)
    Ad, Md = np.asarray(Ad, np.float64), np.asarray(Md, np.float64)
    n = Ad.shape[0]
    if Ad.shape != (n, n) or Md.shape != (n, n):
        raise ValueError(f"generalized_eigs: shapes {Ad.shape} / {Md.shape}")
    if n > max_dof:
        raise ValueError(f"generalized_eigs: {n} DOFs > {max_dof} (dense path)")
    if not np.allclose(Md, Md.T, rtol=0, atol=1e-14 * max(1.0, np.abs(Md).max())):
        raise ArithmeticError("generalized_eigs: M is not symmetric")
    try:
        C = sl.cholesky(Md, lower=True)
    except np.linalg.LinAlgError as e:
        raise ArithmeticError(f"generalized_eigs: M is not positive definite ({e})") from e
    if np.array_equal(Ad, Ad.T):
        lam, V = sl.eigh(Ad, Md)
    else:
        B = sl.solve_triangular(C, sl.solve_triangular(C, Ad, lower=True).T, lower=True).T  # C^-1 A C^-T
        lam, W = sl.eig(B)
        V = sl.solve_triangular(C.T, W, lower=False)
        order = np.lexsort((lam.imag, lam.real))
        lam, V = lam[order], V[:, order]
        if np.all(lam.imag == 0):
            lam, V = lam.real, V.real
    V = V / np.linalg.norm(V, axis=0)[None, :]
    return GeneralizedEigenSystem(lam, V, Ad, Md)


def _reduction(apply, V: np.ndarray, modes, workers: int) -> np.ndarray:
    """factors[k] = ||apply(v_j)|| / ||v_j|| for j = modes[k]; a complex mode is split into its real
    and imaginary parts (the operator is real-linear, so ||S v||^2 = ||S Re v||^2 + ||S Im v||^2)."""
    modes = list(modes)
    out = np.zeros(len(modes))
    errors = []

    def run(ks):
        try:
            for k in ks:
                v = V[:, modes[k]]
                parts = [v.real, v.imag] if np.iscomplexobj(v) else [v]
                num = sum(float(np.dot(w, w)) for w in (apply(np.ascontiguousarray(p)) for p in parts))
                den = sum(float(np.dot(p, p)) for p in parts)
                out[k] = np.sqrt(num / den)
        except Exception as e:  # surfaced after the join
            errors.append(e)

    nw = max(1, min(workers, len(modes)))
    threads = [threading.Thread(target=run, args=(range(q, len(modes), nw),)) for q in range(nw)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out


def reduction_factors(hier: pmg.PmgHierarchy, eig: GeneralizedEigenSystem, which: str = "smoother", level: int = 0,
                      modes=None, workers: int = 4) -> ReductionProfile:
    """Reduction factor of every (or the selected) eigenmode for one smoothing step
    (which="smoother") or one coarse-grid correction (which="cgc": restrict the residual, one
    cycle at level+1, prolongate, update) from u0 = v_j with f = 0 (PAPER Eq. (32)).
    pre: the hierarchy is built for the Laplace problem whose (A, M) gave `eig`."""
    if which not in ("smoother", "cgc"):
        raise ValueError(f"reduction_factors: which must be 'smoother' or 'cgc', not {which!r}")
    n = eig.eigenvectors.shape[0]
    if level != 0 or n != hier.n:  # mismatched problem/eigensystem
        raise ValueError(f"reduction_factors: eigensystem of {n} DOFs at level {level}, hierarchy of {hier.n} "
                         "at level 0")
    modes = np.arange(eig.eigenvectors.shape[1]) if modes is None else np.asarray(modes)
    f = np.zeros(n)
    step = pmg.smooth if which == "smoother" else pmg.coarse_correction
    fac = _reduction(lambda v: step(hier, level, v, f), eig.eigenvectors, modes, workers)
    return ReductionProfile(which, modes, fac)


def iteration_matrix(hier: pmg.PmgHierarchy, max_dof: int = 2500, workers: int = 4) -> np.ndarray:
    """Dense iteration matrix of one p-multigrid cycle.  pre: N_dof <= max_dof
    (SPEC: 2500, dense storage)."""
    n = hier.n
    if n > max_dof:
        raise ValueError(f"iteration_matrix: {n} DOFs > {max_dof} (dense storage)")
    M = np.zeros((n, n))
    L = pmg.lib()
    works = [hier.w]
    try:
        for _ in range(max(1, workers) - 1):
            w = ctypes.c_void_p()
            pmg._raise(L.pmg_work_create(hier.h, ctypes.byref(w)), what="work_create")
            works.append(w.value)
        errors = []

        def run(wk, cols):
            f = np.zeros(n)
            u = np.zeros(n)
            try:
                for i in cols:
                    u[:] = 0.0
                    u[i] = 1.0
                    pmg._raise(L.pmg_cycle(wk, 0, pmg.ptr(u), pmg.ptr(f)), what="cycle")
                    M[:, i] = u
            except Exception as e:  # surfaced after the join
                errors.append(e)

        threads = [threading.Thread(target=run, args=(wk, range(q, n, len(works)))) for q, wk in enumerate(works)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
    finally:
        for wk in works[1:]:
            L.pmg_work_destroy(wk)
    return M


def spectral_radius(M: np.ndarray) -> Spectrum:
    """rho = max |lambda| over the eigenvalues of M."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("spectral_radius: square matrix required")
    if M.size == 0:
        return Spectrum(0.0, np.zeros(0, complex))
    try:
        lam = np.linalg.eigvals(M)
    except np.linalg.LinAlgError as e:  # eigensolver non-convergence -> analysis error
        raise ArithmeticError(f"spectral_radius: eigensolver did not converge ({e})") from e
    return Spectrum(float(np.max(np.abs(lam))), lam)


def condition_number(A, max_dof: int = 5000) -> float:
    """kappa_2 = sigma_max / sigma_min by dense SVD; A: CSR or dense."""
    D = A if isinstance(A, np.ndarray) else _dense(A)
    if D.shape[0] > max_dof:
        raise ValueError(f"condition_number: {D.shape[0]} DOFs > {max_dof}")
    s = np.linalg.svd(D, compute_uv=False)
    return float(s[0] / s[-1]) if s[-1] > 0 else float("inf")


def _dense(A) -> np.ndarray:
    D = np.zeros((A.nrows, A.ncols))
    for i in range(A.nrows):
        D[i, A.col[A.rowptr[i]:A.rowptr[i + 1]]] = A.val[A.rowptr[i]:A.rowptr[i + 1]]
    return D
