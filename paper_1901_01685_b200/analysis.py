"""Spectral analysis of the p-multigrid cycle (the `analysis` module; PAPER §4;
SURVEY §8(f) F3): the iteration matrix column by column on the GPU, its spectral radius and
eigenvalue cloud, and condition numbers.

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
class Spectrum:
    rho: float
    eigenvalues: np.ndarray  # complex, the eigenvalue cloud (PAPER Figs. 5-6)


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
