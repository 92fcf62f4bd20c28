"""ctypes bindings of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg -- never by the product package.
See oracle.h for the algorithm and its citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

PMG_OK, PMG_ZERO_PIVOT, PMG_ZERO_DIAG = 0, 1, 2
ILUT, GS = 0, 1
ORDER_NONE, ORDER_RCM = 0, 1


class CsrView(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int32), ("ncols", ctypes.c_int32), ("rowptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class HierDesc(ctypes.Structure):
    _fields_ = [("n_plevels", ctypes.c_int), ("degrees", ctypes.c_void_p), ("A", ctypes.c_void_p),
                ("ML", ctypes.c_void_p), ("P", ctypes.c_void_p), ("PT", ctypes.c_void_p),
                ("n_hlevels", ctypes.c_int), ("HA", ctypes.c_void_p), ("HP", ctypes.c_void_p),
                ("HPT", ctypes.c_void_p), ("smoother", ctypes.c_int), ("nu1", ctypes.c_int), ("nu2", ctypes.c_int),
                ("tau", ctypes.c_double), ("fillfactor", ctypes.c_double), ("ordering", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
        L = ctypes.CDLL(LIB)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_norm2.restype = dbl
        L.orc_norm2.argtypes = [vp, i64]
        for fn in ("orc_spmv",):
            getattr(L, fn).argtypes = [vp, vp, vp]
        L.orc_residual.argtypes = [vp, vp, vp, vp]
        L.orc_gs_sweep.argtypes = [vp, vp, vp, vp]
        L.orc_rcm.argtypes = [vp, vp]
        L.orc_ilut.argtypes = [vp, dbl, dbl, ctypes.c_int, ctypes.POINTER(vp), vp]
        L.orc_ilut_eigen.argtypes = [vp, dbl, dbl, ctypes.c_int, ctypes.POINTER(vp)]
        L.orc_factor_from_arrays.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(vp)]
        L.orc_factor_free.argtypes = [vp]
        L.orc_factor_stats.argtypes = [vp, vp, vp, vp, vp]
        L.orc_factor_export.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_ilut_apply.argtypes = [vp, vp, vp]
        L.orc_prolongate.argtypes = [vp, vp, vp, vp]
        L.orc_restrict.argtypes = [vp, vp, vp, vp]
        L.orc_hier_create.argtypes = [vp, vp, ctypes.POINTER(vp), vp, vp]
        L.orc_hier_free.argtypes = [vp]
        L.orc_hier_num_factors.argtypes = [vp]
        L.orc_hier_factor.argtypes = [vp, ctypes.c_int]
        L.orc_hier_factor.restype = vp
        L.orc_solve.argtypes = [vp, vp, vp, dbl, ctypes.c_int, vp, vp, vp, vp, vp]
        L.orc_cycle.argtypes = [vp, ctypes.c_int, vp, vp]
        L.orc_smooth.argtypes = [vp, ctypes.c_int, vp, vp]
        L.orc_coarse_correction.argtypes = [vp, ctypes.c_int, vp, vp]
        L.orc_bicgstab.argtypes = [vp, vp, vp, dbl, ctypes.c_int, vp, vp, vp, vp]
        L.orc_bicgstab_plain.argtypes = [vp, vp, vp, dbl, ctypes.c_int, vp, vp, vp]
        L.orc_dot.restype = dbl
        L.orc_dot.argtypes = [vp, vp, i64]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def view(A) -> CsrView:
    v = CsrView(A.nrows, A.ncols, _p(A.rowptr), _p(A.col), _p(A.val))
    v._keep = A
    return v


class OracleError(RuntimeError):
    def __init__(self, status, row=-1, level=-1):
        super().__init__(f"oracle status {status} row {row} level {level}")
        self.status, self.row, self.level = status, row, level


def set_threads(n: int) -> None:
    """Host threads for the oracle's row-independent loops and ILUT rows (results unchanged)."""
    lib().orc_set_threads(int(n))


def spmv(A, x):
    y = np.empty(A.nrows)
    lib().orc_spmv(ctypes.byref(view(A)), _p(np.ascontiguousarray(x, float)), _p(y))
    return y


def residual(A, x, f):
    r = np.empty(A.nrows)
    lib().orc_residual(ctypes.byref(view(A)), _p(np.ascontiguousarray(x, float)), _p(np.ascontiguousarray(f, float)),
                       _p(r))
    return r


def norm2(r):
    r = np.ascontiguousarray(r, float)
    return lib().orc_norm2(_p(r), r.size)


def dot(x, y):
    x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
    return lib().orc_dot(_p(x), _p(y), x.size)


def _krylov_report(iters, hist, flags, seconds=None):
    it = iters.value
    return dict(iterations=it, residual_history=hist[: it + 1].copy(), converged=bool(flags.value & 1),
                diverged=bool(flags.value & 2), breakdown=bool(flags.value & 4), solve_seconds=seconds)


def bicgstab_plain(A, f, u0=None, tol=1e-8, max_iter=200):
    """Unpreconditioned BiCGSTAB, same arithmetic as the preconditioned one."""
    f = np.ascontiguousarray(f, float)
    u = np.zeros(f.size) if u0 is None else np.array(u0, dtype=float, copy=True)
    hist = np.zeros(max_iter + 1)
    it, flags = ctypes.c_int(), ctypes.c_int()
    st = lib().orc_bicgstab_plain(ctypes.byref(view(A)), _p(f), _p(u), tol, max_iter, _p(hist), ctypes.byref(it),
                                  ctypes.byref(flags))
    if st != PMG_OK:
        raise OracleError(st)
    return u, _krylov_report(it, hist, flags)


def gauss_seidel_sweep(A, u, f):
    u = np.array(u, dtype=float, copy=True)
    row = ctypes.c_int64(-1)
    st = lib().orc_gs_sweep(ctypes.byref(view(A)), _p(u), _p(np.ascontiguousarray(f, float)), ctypes.byref(row))
    if st != PMG_OK:
        raise OracleError(st, row.value)
    return u


def rcm_ordering(A):
    perm = np.empty(A.nrows, np.int32)
    lib().orc_rcm(ctypes.byref(view(A)), _p(perm))
    return perm


class Factor:
    def __init__(self, handle, owner=None):
        self.h = handle
        self._owner = owner

    def __del__(self):
        if self.h and lib is not None:
            lib().orc_factor_free(self.h)
            self.h = None

    def stats(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        c, d = ctypes.c_int32(), ctypes.c_int32()
        lib().orc_factor_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d))
        return dict(nnz_L=a.value, nnz_U=b.value, levels_L=c.value, levels_U=d.value)

    def export(self):
        from paper_1901_01685_b200._native import Csr
        s = self.stats()
        n = self.n
        Lrp = np.empty(n + 1, np.int32); Lc = np.empty(s["nnz_L"], np.int32); Lv = np.empty(s["nnz_L"])
        Urp = np.empty(n + 1, np.int32); Uc = np.empty(s["nnz_U"], np.int32); Uv = np.empty(s["nnz_U"])
        perm = np.empty(n, np.int32)
        lib().orc_factor_export(self.h, _p(Lrp), _p(Lc), _p(Lv), _p(Urp), _p(Uc), _p(Uv), _p(perm))
        return Csr(n, n, Lrp, Lc, Lv), Csr(n, n, Urp, Uc, Uv), perm

    def apply(self, r):
        e = np.empty(self.n)
        lib().orc_ilut_apply(self.h, _p(np.ascontiguousarray(r, float)), _p(e))
        return e

    @classmethod
    def from_arrays(cls, L, U, perm=None):
        h = ctypes.c_void_p()
        lib().orc_factor_from_arrays(L.nrows, _p(L.rowptr), _p(L.col), _p(L.val), _p(U.rowptr), _p(U.col),
                                     _p(U.val), _p(None if perm is None else np.ascontiguousarray(perm, np.int32)),
                                     ctypes.byref(h))
        f = cls(h.value)
        f.n = L.nrows
        return f


def ilut_factorize(A, tau=1e-12, fillfactor=1.0, ordering=ORDER_RCM) -> Factor:
    h = ctypes.c_void_p()
    row = ctypes.c_int64(-1)
    st = lib().orc_ilut(ctypes.byref(view(A)), tau, fillfactor, ordering, ctypes.byref(h), ctypes.byref(row))
    if st != PMG_OK:
        raise OracleError(st, row.value)
    f = Factor(h.value)
    f.n = A.nrows
    return f


def ilut_factorize_eigen(A, tau=1e-12, fillfactor=1.0, ordering=ORDER_NONE) -> Factor:
    """PROBE ONLY: the paper library's ILUT rule (oracle.cpp ilut_eigen)."""
    h = ctypes.c_void_p()
    lib().orc_ilut_eigen(ctypes.byref(view(A)), tau, fillfactor, ordering, ctypes.byref(h))
    f = Factor(h.value)
    f.n = A.nrows
    return f


def prolongate(P, ML, vc):
    vf = np.empty(P.nrows)
    lib().orc_prolongate(ctypes.byref(view(P)), _p(np.ascontiguousarray(ML, float)), _p(np.ascontiguousarray(vc, float)),
                         _p(vf))
    return vf


def restrict(PT, MLc, rf):
    rc = np.empty(PT.nrows)
    lib().orc_restrict(ctypes.byref(view(PT)), _p(np.ascontiguousarray(MLc, float)),
                       _p(np.ascontiguousarray(rf, float)), _p(rc))
    return rc


def make_desc(problem, smoother=ILUT, nu1=1, nu2=1, tau=1e-12, fillfactor=1.0, ordering=ORDER_NONE):
    """pmg_hier_desc for a paper_1901_01685_b200.problems.Problem; returns (desc, keepalive)."""
    pl, hl = problem.plevels, problem.hlevels
    keep = []
    degrees = np.array([l.degree for l in pl], np.int32)
    A = (CsrView * len(pl))(*[view(l.A) for l in pl])
    ML = (ctypes.c_void_p * len(pl))(*[_p(l.ML) for l in pl])
    npt = max(len(pl) - 1, 1)
    P = (CsrView * npt)(*[view(l.P) for l in pl[:-1]])
    PT = (CsrView * npt)(*[view(l.PT) for l in pl[:-1]])
    HA = (CsrView * len(hl))(*[view(h.A) for h in hl])
    nht = max(len(hl) - 1, 1)
    HP = (CsrView * nht)(*[view(h.P) for h in hl[:-1]])
    HPT = (CsrView * nht)(*[view(h.PT) for h in hl[:-1]])
    keep += [degrees, A, ML, P, PT, HA, HP, HPT, problem]
    d = HierDesc(len(pl), _p(degrees), ctypes.addressof(A), ctypes.addressof(ML), ctypes.addressof(P),
                 ctypes.addressof(PT), len(hl), ctypes.addressof(HA), ctypes.addressof(HP), ctypes.addressof(HPT),
                 smoother, nu1, nu2, tau, fillfactor, ordering)
    return d, keep


class Hierarchy:
    """Oracle p-multigrid hierarchy and solve."""

    def __init__(self, problem, smoother=ILUT, nu1=1, nu2=1, tau=1e-12, fillfactor=1.0, ordering=ORDER_NONE,
                 factors=None):
        self.desc, self._keep = make_desc(problem, smoother, nu1, nu2, tau, fillfactor, ordering)
        self.n = problem.n
        self._sizes = ([l.A.nrows for l in problem.plevels[:-1]] if smoother == ILUT else []) + \
                      [h.A.nrows for h in problem.hlevels[:-1]]
        h = ctypes.c_void_p()
        lvl, row = ctypes.c_int(-1), ctypes.c_int64(-1)
        ext = None
        if factors is not None:
            ext = (ctypes.c_void_p * len(factors))(*[f.h for f in factors])
            self._keep.append((ext, factors))
        st = lib().orc_hier_create(ctypes.byref(self.desc), None if ext is None else ctypes.addressof(ext),
                                   ctypes.byref(h), ctypes.byref(lvl), ctypes.byref(row))
        if st != PMG_OK:
            raise OracleError(st, row.value, lvl.value)
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_hier_free(self.h)
            self.h = None

    def factors(self):
        out = []
        for k in range(lib().orc_hier_num_factors(self.h)):
            f = Factor(lib().orc_hier_factor(self.h, k), owner=self)
            f.n = self._sizes[k]
            out.append(f)
        return out

    def solve(self, f, u0, tol=1e-8, max_cycles=200):
        u = np.array(u0, dtype=float, copy=True)
        hist = np.zeros(max_cycles + 1)
        cyc, flags = ctypes.c_int(), ctypes.c_int()
        ts, tsu = ctypes.c_double(), ctypes.c_double()
        st = lib().orc_solve(self.h, _p(np.ascontiguousarray(f, float)), _p(u), tol, max_cycles, _p(hist),
                             ctypes.byref(cyc), ctypes.byref(flags), ctypes.byref(ts), ctypes.byref(tsu))
        if st != PMG_OK:
            raise OracleError(st)
        c = cyc.value
        return u, dict(cycles=c, residual_history=hist[: c + 1].copy(), converged=bool(flags.value & 1),
                       diverged=bool(flags.value & 2), solve_seconds=ts.value, setup_seconds=tsu.value)

    def bicgstab(self, f, u0, tol=1e-8, max_iter=200):
        """BiCGSTAB preconditioned by one V-cycle from zero."""
        u = np.array(u0, dtype=float, copy=True)
        hist = np.zeros(max_iter + 1)
        it, flags, ts = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        st = lib().orc_bicgstab(self.h, _p(np.ascontiguousarray(f, float)), _p(u), tol, max_iter, _p(hist),
                                ctypes.byref(it), ctypes.byref(flags), ctypes.byref(ts))
        if st != PMG_OK:
            raise OracleError(st)
        return u, _krylov_report(it, hist, flags, ts.value)

    def cycle(self, u, f, level=0):
        u = np.array(u, dtype=float, copy=True)
        lib().orc_cycle(self.h, level, _p(u), _p(np.ascontiguousarray(f, float)))
        return u

    def smooth(self, u, f, level=0):
        """One smoothing step at p-level `level` (reduction_factors)."""
        u = np.array(u, dtype=float, copy=True)
        st = lib().orc_smooth(self.h, level, _p(u), _p(np.ascontiguousarray(f, float)))
        if st != PMG_OK:
            raise OracleError(st)
        return u

    def coarse_correction(self, u, f, level=0):
        """One coarse-grid correction at p-level `level` (PAPER §4 steps 2-4)."""
        u = np.array(u, dtype=float, copy=True)
        st = lib().orc_coarse_correction(self.h, level, _p(u), _p(np.ascontiguousarray(f, float)))
        if st != PMG_OK:
            raise OracleError(st)
        return u
