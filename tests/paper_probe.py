"""Probe of the p-multigrid variants behind the paper's Gauss-Seidel numbers (test infrastructure).

A small, knob-driven restatement of the V-cycle (scipy), used to root-cause the gap between the
oracle's Gauss-Seidel cycle counts and PAPER.md:537-563 / SPEC.md:558-563.  The
knobs are the places where the paper / SPEC leave the algorithm open:

  hmg_smoother   smoother of the p=1 h-multigrid coarse solver: "ilut", "same" (the
                 p-level smoother), or "exact" (direct p=1 solve instead of one h-MG V-cycle)
  hrestrict      scale of the h-MG full-weighting restriction (1 = FE P^T, 0.25 = FD)
  nitsche        multiplier of the Nitsche penalty 4p^2/h
  degrees        "consecutive" p, p-1, ..., 1 (Fig. 1) or "direct" p, 1 (BASELINE configs)
  post           "forward" GS post-smoother or "backward" (symmetric GS V-cycle)

Not part of the product and not of the parity suite: ``python tests/paper_probe.py`` prints the table.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import oracle as O
from paper_1901_01685_b200 import problems as P


def _sp(A):
    return sp.csr_matrix((A.val, A.col, A.rowptr), shape=(A.nrows, A.ncols))


class Probe:
    def __init__(self, spec, smoother="gs", hmg_smoother="ilut", hrestrict=1.0, post="forward", gs_order="x",
                 ilut="spec", ordering=O.ORDER_NONE):
        pb = P.build(spec)
        self.pb = pb
        self.smoother, self.hmg_smoother, self.hrestrict, self.post = smoother, hmg_smoother, hrestrict, post
        self.gs_order = gs_order
        self.pA = [_sp(l.A) for l in pb.plevels]
        self.pML = [l.ML for l in pb.plevels]
        self.pP = [_sp(l.P) if l.P is not None else None for l in pb.plevels]
        self.hA = [_sp(h.A) for h in pb.hlevels]
        self.hP = [_sp(h.P) if h.P is not None else None for h in pb.hlevels]
        fac = (lambda A: O.ilut_factorize(A, 1e-12, 1.0, ordering)) if ilut == "spec" else \
            (lambda A: O.ilut_factorize_eigen(A, 1e-12, 1.0, ordering))
        self.pF = [fac(l.A) if smoother == "ilut" else None for l in pb.plevels[:-1]]
        self.hF = [fac(h.A) if hmg_smoother in ("ilut",) or
                   (hmg_smoother == "same" and smoother == "ilut") else None for h in pb.hlevels[:-1]]
        self.coarse_lu = spla.splu(self.hA[-1].tocsc())
        self.p1_lu = spla.splu(self.pA[-1].tocsc()) if hmg_smoother == "exact" else None
        self.tril = {}

    def _gs(self, A, u, f, backward=False):
        key = (id(A), backward)
        if key not in self.tril:
            self.tril[key] = (sp.triu(A, 0).tocsr(), sp.tril(A, -1).tocsr()) if backward else \
                (sp.tril(A, 0).tocsr(), sp.triu(A, 1).tocsr())
        T, R = self.tril[key]
        return spla.spsolve_triangular(T, f - R @ u, lower=not backward)

    def _gs_perm(self, A, u, f, backward=False):
        """GS in the transposed lexicographic order (y fastest)."""
        n = A.shape[0]
        m = int(round(np.sqrt(n)))
        idx = np.arange(n)
        q = (idx % m) * m + idx // m  # q[new] = old
        key = ("perm", id(A))
        if key not in self.tril:
            self.tril[key] = A[q][:, q].tocsr()
        Ap = self.tril[key]
        return self._gs(Ap, u[q], f[q], backward)[np.argsort(q)]

    def _smooth(self, kind, A, F, u, f, post=False):
        if kind == "gs":
            g = self._gs_perm if self.gs_order == "y" else self._gs
            return g(A, u, f, backward=post and self.post == "backward")
        return u + F.apply(f - A @ u)

    def hmg(self, j, r):
        if j == len(self.hA) - 1:
            return self.coarse_lu.solve(r)
        A = self.hA[j]
        kind = self.smoother if self.hmg_smoother == "same" else "ilut"
        F = self.hF[j]
        e = self._smooth(kind, A, F, np.zeros_like(r), r)
        rc = self.hrestrict * (self.hP[j].T @ (r - A @ e))
        e = e + self.hP[j] @ self.hmg(j + 1, rc)
        return self._smooth(kind, A, F, e, r, post=True)

    def cycle(self, l, u, f):
        if l == len(self.pA) - 1:
            if self.p1_lu is not None:
                return u + self.p1_lu.solve(f - self.pA[l] @ u)
            return u + self.hmg(0, f - self.pA[l] @ u)
        A, F = self.pA[l], self.pF[l]
        u = self._smooth(self.smoother, A, F, u, f)
        rc = (self.pP[l].T @ (f - A @ u)) / self.pML[l + 1]
        ec = self.cycle(l + 1, np.zeros(rc.size), rc)
        u = u + (self.pP[l] @ ec) / self.pML[l]
        return self._smooth(self.smoother, A, F, u, f, post=True)

    def solve(self, tol=1e-8, maxc=200):
        f, u = self.pb.f, self.pb.u0.copy()
        A = self.pA[0]
        n0 = np.linalg.norm(f - A @ u)
        hist = [1.0]
        for c in range(1, maxc + 1):
            u = self.cycle(0, u, f)
            rho = np.linalg.norm(f - A @ u) / n0
            hist.append(rho)
            if rho <= tol:
                return c, "conv", hist
            if not rho <= 1e10:
                return c, "div", hist
        return maxc, "max", hist

    def spectral_radius(self):
        """rho of the iteration matrix (f = 0, columns = one cycle from e_i)."""
        n = self.pA[0].shape[0]
        f = np.zeros(n)
        M = np.empty((n, n))
        for i in range(n):
            e = np.zeros(n)
            e[i] = 1.0
            M[:, i] = self.cycle(0, e, f)
        return float(np.max(np.abs(np.linalg.eigvals(M))))


def spec(bench, p, h_exp, degrees="consecutive", nitsche=1.0, random_guess=True):
    s = P.benchmark_spec(bench, p, h_exp, consecutive=(degrees == "consecutive"))
    s.nitsche_scale = nitsche
    s.random_guess = int(random_guess)
    return s


def eliminate_boundary(pr, nel):
    """Strong Dirichlet elimination (g = 0) on a single tensor patch: drop the boundary DOFs'
    rows and columns from every operator (probe of the BC treatment; SPEC.md:185 uses Nitsche)."""
    def interior(p, n_el):
        n = n_el + p
        idx = np.arange(n * n)
        ix, iy = idx % n, idx // n
        return idx[(ix > 0) & (ix < n - 1) & (iy > 0) & (iy < n - 1)]
    degs = [l.degree for l in pr.pb.plevels]
    keep = [interior(d, nel) for d in degs]
    pr.pA = [A[k][:, k] for A, k in zip(pr.pA, keep)]
    pr.pML = [m[k] for m, k in zip(pr.pML, keep)]
    pr.pP = [P[keep[i]][:, keep[i + 1]] if P is not None else None for i, P in enumerate(pr.pP)]
    hk = [interior(1, nel >> j) for j in range(len(pr.hA))]
    pr.hA = [A[k][:, k] for A, k in zip(pr.hA, hk)]
    pr.hP = [P[hk[j]][:, hk[j + 1]] if P is not None else None for j, P in enumerate(pr.hP)]
    pr.coarse_lu = spla.splu(pr.hA[-1].tocsc())
    pr.p1_lu = spla.splu(pr.pA[-1].tocsc())
    pr.hmg_smoother = "exact"
    pr.pb.f = pr.pb.f[keep[0]]
    pr.pb.u0 = pr.pb.u0[keep[0]]
    if pr.smoother == "ilut":
        from paper_1901_01685_b200._native import Csr
        def tocsr(A):
            A = A.tocsr(); A.sort_indices()
            return Csr(A.shape[0], A.shape[1], A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data.copy())
        pr.pF = [O.ilut_factorize(tocsr(A), 1e-12, 1.0, O.ORDER_NONE) for A in pr.pA[:-1]]
    pr.tril = {}
    return pr


def table():
    """The probe table of DESIGN.md §0a: B1 (quarter annulus) Gauss-Seidel cycles at h = 2^-6."""
    rows = [
        ("oracle (SPEC rules)", {}, {}),
        ("h-MG smoother = GS", {}, dict(hmg_smoother="same")),
        ("exact p=1 solve", {}, dict(hmg_smoother="exact")),
        ("h-MG restriction x0.5", {}, dict(hrestrict=0.5)),
        ("h-MG restriction x0.25", {}, dict(hrestrict=0.25)),
        ("direct p->1 hierarchy", dict(degrees="direct"), {}),
        ("Nitsche penalty x0.25", dict(nitsche=0.25), {}),
        ("Nitsche penalty x4", dict(nitsche=4.0), {}),
        ("backward GS post-smoother", {}, dict(post="backward")),
        ("GS order y fastest", {}, dict(gs_order="y")),
        ("strong Dirichlet elimination", {}, dict(hmg_smoother="exact", _elim=True)),
    ]
    for name, skw, pkw in rows:
        out = []
        for p in (2, 3, 4):
            elim = pkw.pop("_elim", False)
            pr = Probe(spec(1, p, 6, **skw), smoother="gs", **pkw)
            if elim:
                eliminate_boundary(pr, 64)
                pkw["_elim"] = True
            c, st, _ = pr.solve()
            out.append(f"{c}" + ("" if st == "conv" else f" ({st})"))
        print(f"| {name} | " + " | ".join(out) + " |", flush=True)


if __name__ == "__main__":
    table()
