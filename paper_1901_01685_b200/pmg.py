"""Python mirror of the reference's solver API, bound to the C ABI of libpmg_cuda.so.

The names, argument meanings and error behaviour follow SPEC.md's ``sparselin`` and
``pmg`` operations in the conventions of proj/include/iga/types.hpp
(``FactorizationError`` carries ``row``; divergence is a report flag, not an error).
Every operation runs on the GPU through ``include/pmg_cuda.h``; there is no CPU path --
if the CUDA library cannot run, the call raises :class:`CudaError`.

    spmv(A, x)
    gauss_seidel_sweep(A, u, f)
    rcm_ordering(A)
    ilut_factorize(A, tau, fillfactor, ordering) SPEC.md:251-259
    ilut_apply(fac, r)
    build_hierarchy(problem, smoother, ...)
    prolongate / restrict
    cycle(hier, level, u, f)
    solve(hier, f, tol, max_cycles, guess)
"""
from __future__ import annotations

import contextlib
import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from ._native import Csr, load, ptr

PMG_OK, PMG_ZERO_PIVOT, PMG_ZERO_DIAG, PMG_ERR_DIM, PMG_ERR_CUDA, PMG_ERR_OOM, PMG_ERR_ARG = range(7)
SMOOTHERS = {"ilut": 0, "gs": 1}
ORDERINGS = {"none": 0, "rcm": 1}


# ---- errors (types.hpp:23-42 conventions) ----
class PmgError(RuntimeError):
    status = -1


class FactorizationError(PmgError):
    """Zero pivot in ILUT; ``row`` is the failing (permuted) row."""

    def __init__(self, msg, row, level=-1):
        super().__init__(f"{msg} (row {row}, level {level})")
        self.row, self.level = row, level


class SmootherError(PmgError):
    """Gauss-Seidel on a zero/missing diagonal."""

    def __init__(self, msg, row, level=-1):
        super().__init__(f"{msg} (row {row}, level {level})")
        self.row, self.level = row, level


class DimensionError(PmgError, ValueError):
    pass


class CudaError(PmgError):
    pass


class CsrView(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int32), ("ncols", ctypes.c_int32), ("rowptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class HierDesc(ctypes.Structure):
    _fields_ = [("n_plevels", ctypes.c_int), ("degrees", ctypes.c_void_p), ("A", ctypes.c_void_p),
                ("ML", ctypes.c_void_p), ("P", ctypes.c_void_p), ("PT", ctypes.c_void_p),
                ("n_hlevels", ctypes.c_int), ("HA", ctypes.c_void_p), ("HP", ctypes.c_void_p),
                ("HPT", ctypes.c_void_p), ("smoother", ctypes.c_int), ("nu1", ctypes.c_int), ("nu2", ctypes.c_int),
                ("tau", ctypes.c_double), ("fillfactor", ctypes.c_double), ("ordering", ctypes.c_int)]


class HierStats(ctypes.Structure):
    _fields_ = [("setup_seconds", ctypes.c_double), ("ilut_seconds", ctypes.c_double),
                ("device_bytes", ctypes.c_int64)]


_typed = False


def lib():
    global _typed
    L = load("libpmg_cuda.so")
    if not _typed:
        vp, i32, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        P = ctypes.POINTER
        L.pmg_last_error.restype = ctypes.c_char_p
        L.pmg_status_string.restype = ctypes.c_char_p
        L.pmg_device_info.argtypes = [vp, vp, vp]
        L.pmg_csr_create.argtypes = [vp, P(vp)]
        L.pmg_csr_destroy.argtypes = [vp]
        L.pmg_spmv.argtypes = [vp, vp, vp]
        L.pmg_residual.argtypes = [vp, vp, vp, vp, vp]
        L.pmg_gs_sweep.argtypes = [vp, vp, vp, vp]
        L.pmg_rcm_ordering.argtypes = [vp, vp]
        L.pmg_ilut_factorize.argtypes = [vp, dbl, dbl, ci, P(vp), vp]
        L.pmg_factor_destroy.argtypes = [vp]
        L.pmg_ilut_apply.argtypes = [vp, vp, vp]
        L.pmg_factor_stats.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.pmg_factor_sweep_info.argtypes = [vp, vp, vp, vp, vp]
        L.pmg_factor_export.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.pmg_hier_create.argtypes = [vp, P(vp), vp, vp]
        L.pmg_hier_destroy.argtypes = [vp]
        L.pmg_hier_get_stats.argtypes = [vp, vp]
        L.pmg_hier_factor.argtypes = [vp, ci, P(vp)]
        L.pmg_work_create.argtypes = [vp, P(vp)]
        L.pmg_work_destroy.argtypes = [vp]
        L.pmg_solve.argtypes = [vp, vp, vp, dbl, ci, vp, vp, vp, vp]
        L.pmg_solve_device.argtypes = [vp, vp, vp, dbl, ci, vp, vp, vp, vp]
        L.pmg_cycle.argtypes = [vp, ci, vp, vp]
        L.pmg_smooth.argtypes = [vp, ci, vp, vp]
        L.pmg_coarse_correction.argtypes = [vp, ci, vp, vp]
        L.pmg_bicgstab.argtypes = [vp, vp, vp, dbl, ci, vp, vp, vp, vp]
        L.pmg_bicgstab_device.argtypes = [vp, vp, vp, dbl, ci, vp, vp, vp, vp]
        L.pmg_prolongate.argtypes = [vp, ci, vp, vp]
        L.pmg_restrict.argtypes = [vp, ci, vp, vp]
        L.pmg_work_kernel_times.argtypes = [vp, vp, ci]
        _typed = True
    return L


def _raise(st, row=-1, level=-1, what=""):
    if st == PMG_OK:
        return
    msg = lib().pmg_last_error().decode() or lib().pmg_status_string(st).decode()
    if st == PMG_ZERO_PIVOT:
        raise FactorizationError(f"{what}: zero pivot", row, level)
    if st == PMG_ZERO_DIAG:
        raise SmootherError(f"{what}: zero diagonal", row, level)
    if st == PMG_ERR_DIM:
        raise DimensionError(f"{what}: {msg}")
    if st == PMG_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    e = CudaError(f"{what}: {msg}")
    e.status = st
    raise e


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise DimensionError(f"expected a vector of length {n}, got shape {a.shape}")
    return a


def view(A: Csr) -> CsrView:
    v = CsrView(A.nrows, A.ncols, ptr(A.rowptr), ptr(A.col), ptr(A.val))
    v._keep = A
    return v


def device_info():
    sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _raise(lib().pmg_device_info(ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi)), what="device_info")
    return dict(sm_count=sm.value, cc=(ma.value, mi.value))


# =========================================================== sparselin
class CsrMatrix:
    """Device-resident SparseMatrixCsr."""

    def __init__(self, A: Csr):
        self.host = A
        self.nrows, self.ncols = A.nrows, A.ncols
        h = ctypes.c_void_p()
        _raise(lib().pmg_csr_create(ctypes.byref(view(A)), ctypes.byref(h)), what="csr_create")
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().pmg_csr_destroy(self.h)
            self.h = None


def _dev(A) -> CsrMatrix:
    return A if isinstance(A, CsrMatrix) else CsrMatrix(A)


def spmv(A, x):
    A = _dev(A)
    x = _f64(x, A.ncols)
    y = np.empty(A.nrows)
    _raise(lib().pmg_spmv(A.h, ptr(x), ptr(y)), what="spmv")
    return y


def residual(A, x, f):
    """r = f - A x and its canonical 2-norm."""
    A = _dev(A)
    x, f = _f64(x, A.ncols), _f64(f, A.nrows)
    r = np.empty(A.nrows)
    nrm = ctypes.c_double()
    _raise(lib().pmg_residual(A.h, ptr(x), ptr(f), ptr(r), ctypes.byref(nrm)), what="residual")
    return r, nrm.value


def gauss_seidel_sweep(A, u, f):
    A = _dev(A)
    if A.nrows != A.ncols:
        raise DimensionError("gauss_seidel_sweep: matrix not square")
    u = np.array(_f64(u, A.nrows), copy=True)
    row = ctypes.c_int64(-1)
    _raise(lib().pmg_gs_sweep(A.h, ptr(u), ptr(_f64(f, A.nrows)), ctypes.byref(row)), row.value,
           what="gauss_seidel_sweep")
    return u


def rcm_ordering(A: Csr):
    perm = np.empty(A.nrows, np.int32)
    _raise(lib().pmg_rcm_ordering(ctypes.byref(view(A)), ptr(perm)), what="rcm_ordering")
    return perm


class IlutFactorization:
    """L (unit lower, implicit diagonal), U, perm / perm_inverse, tau, fillfactor."""

    def __init__(self, handle, n, tau, fillfactor, owner=None):
        self.h, self.n, self.tau, self.fillfactor = handle, n, tau, fillfactor
        self._owner = owner

    def __del__(self):
        if self._owner is None and getattr(self, "h", None):
            lib().pmg_factor_destroy(self.h)
            self.h = None

    def stats(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        c, d, e, f = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        lib().pmg_factor_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d),
                               ctypes.byref(e), ctypes.byref(f))
        n = self.n
        k, sg, dl, du = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        lib().pmg_factor_sweep_info(self.h, ctypes.byref(k), ctypes.byref(sg), ctypes.byref(dl), ctypes.byref(du))
        return dict(nnz_L=a.value, nnz_U=b.value, levels_L=c.value, levels_U=d.value,
                    rows_per_level_L=n / max(c.value, 1), rows_per_level_U=n / max(d.value, 1),
                    max_row_L=e.value, max_row_U=f.value,
                    sweep=("levels", "chain", "skew", "wave")[k.value], segment=sg.value, skew_D=(dl.value, du.value))

    def export(self):
        s = self.stats()
        n = self.n
        Lrp = np.empty(n + 1, np.int32); Lc = np.empty(s["nnz_L"], np.int32); Lv = np.empty(s["nnz_L"])
        Urp = np.empty(n + 1, np.int32); Uc = np.empty(s["nnz_U"], np.int32); Uv = np.empty(s["nnz_U"])
        perm = np.empty(n, np.int32)
        _raise(lib().pmg_factor_export(self.h, ptr(Lrp), ptr(Lc), ptr(Lv), ptr(Urp), ptr(Uc), ptr(Uv), ptr(perm)),
               what="factor_export")
        return Csr(n, n, Lrp, Lc, Lv), Csr(n, n, Urp, Uc, Uv), perm

    @property
    def perm(self):
        return self.export()[2]

    @property
    def perm_inverse(self):
        p = self.perm
        inv = np.empty_like(p)
        inv[p] = np.arange(p.size, dtype=p.dtype)
        return inv


def ilut_factorize(A, tau=1e-12, fillfactor=1.0, ordering="rcm") -> IlutFactorization:
    A = _dev(A)
    if A.nrows != A.ncols:
        raise DimensionError("ilut_factorize: matrix not square")
    h = ctypes.c_void_p()
    row = ctypes.c_int64(-1)
    _raise(lib().pmg_ilut_factorize(A.h, tau, fillfactor, ORDERINGS[ordering], ctypes.byref(h), ctypes.byref(row)),
           row.value, what="ilut_factorize")
    return IlutFactorization(h.value, A.nrows, tau, fillfactor)


def ilut_apply(fac: IlutFactorization, r):
    r = _f64(r, fac.n)
    e = np.empty(fac.n)
    _raise(lib().pmg_ilut_apply(fac.h, ptr(r), ptr(e)), what="ilut_apply")
    return e


# =========================================================== pmg
@dataclass
class SolveReport:
    """cycles, residual_history, converged / diverged, setup / solve seconds."""

    cycles: int
    residual_history: np.ndarray
    converged: bool
    diverged: bool
    setup_seconds: float
    solve_seconds: float
    extra: dict = field(default_factory=dict)


@dataclass
class KrylovReport:
    """iterations, residual_history ([0] = 1), converged, breakdown."""

    iterations: int
    residual_history: np.ndarray
    converged: bool
    diverged: bool
    breakdown: bool
    solve_seconds: float


class PmgHierarchy:
    """Immutable device hierarchy: p-levels with smoother state and lumped
    L2 transfers, and the p=1 h-multigrid chain with a dense coarsest solve."""

    def __init__(self, problem, smoother="ilut", nu1=1, nu2=1, tau=1e-12, fillfactor=1.0, ordering="none"):
        pl, hl = problem.plevels, problem.hlevels
        self.problem_name = problem.name
        self.n = pl[0].A.nrows
        self.degrees = [l.degree for l in pl]
        self.smoother = smoother
        keep = []
        degrees = np.array(self.degrees, np.int32)
        A = (CsrView * len(pl))(*[view(l.A) for l in pl])
        ML = (ctypes.c_void_p * len(pl))(*[ptr(l.ML) for l in pl])
        npt = max(len(pl) - 1, 1)
        P = (CsrView * npt)(*[view(l.P) for l in pl[:-1]])
        PT = (CsrView * npt)(*[view(l.PT) for l in pl[:-1]])
        HA = (CsrView * len(hl))(*[view(h.A) for h in hl])
        nht = max(len(hl) - 1, 1)
        HP = (CsrView * nht)(*[view(h.P) for h in hl[:-1]])
        HPT = (CsrView * nht)(*[view(h.PT) for h in hl[:-1]])
        keep += [degrees, A, ML, P, PT, HA, HP, HPT, problem]
        d = HierDesc(len(pl), ptr(degrees), ctypes.addressof(A), ctypes.addressof(ML), ctypes.addressof(P),
                     ctypes.addressof(PT), len(hl), ctypes.addressof(HA), ctypes.addressof(HP),
                     ctypes.addressof(HPT), SMOOTHERS[smoother], nu1, nu2, tau, fillfactor, ORDERINGS[ordering])
        h = ctypes.c_void_p()
        lvl, row = ctypes.c_int(-1), ctypes.c_int64(-1)
        st = lib().pmg_hier_create(ctypes.byref(d), ctypes.byref(h), ctypes.byref(lvl), ctypes.byref(row))
        _raise(st, row.value, lvl.value, what="build_hierarchy")
        self.h = h.value
        # per-solve state lives in work objects (vectors, stream, scratch); the hierarchy itself
        # is immutable, so concurrent solves from several host threads each
        # take a work object of their own from this pool
        self.w = self._new_work()
        self._free = [self.w]
        self._all = [self.w]
        self._lock = threading.Lock()
        s = HierStats()
        lib().pmg_hier_get_stats(self.h, ctypes.byref(s))
        self.setup_seconds, self.ilut_seconds, self.device_bytes = s.setup_seconds, s.ilut_seconds, s.device_bytes
        self.nfactors = (len(pl) - 1 if smoother == "ilut" else 0) + len(hl) - 1

    def _new_work(self):
        w = ctypes.c_void_p()
        _raise(lib().pmg_work_create(self.h, ctypes.byref(w)), what="work_create")
        return w.value

    @contextlib.contextmanager
    def work(self):
        """A work object for one call: the primary one when free, else a new pooled one."""
        with self._lock:
            w = self._free.pop() if self._free else None
        if w is None:
            w = self._new_work()
            with self._lock:
                self._all.append(w)
        try:
            yield w
        finally:
            with self._lock:
                self._free.append(w)

    def __del__(self):
        for w in getattr(self, "_all", []):
            lib().pmg_work_destroy(w)
        self._all = []
        self.w = None
        if getattr(self, "h", None):
            lib().pmg_hier_destroy(self.h)
            self.h = None

    def factors(self):
        out = []
        np_ = len(self.degrees)
        ids = ([l for l in range(np_ - 1)] if self.smoother == "ilut" else []) + \
              [np_ - 1 + j for j in range(self.nfactors - (np_ - 1 if self.smoother == "ilut" else 0))]
        for pos, k in enumerate(ids):
            h = ctypes.c_void_p()
            _raise(lib().pmg_hier_factor(self.h, k, ctypes.byref(h)), what="hier_factor")
            out.append(IlutFactorization(h.value, self._sizes[pos], None, None, owner=self))
        return out

    def kernel_times(self, enable=None):
        """Per-class device ms: resid(A_p), L(p), U(p), GS(p), transfers, coarse, misc."""
        L = lib()
        if enable is not None:
            _raise(L.pmg_work_kernel_times(self.w, None, -1 if enable else -2), what="kernel_times")
            return None
        out = np.zeros(15)
        _raise(L.pmg_work_kernel_times(self.w, ptr(out), out.size), what="kernel_times")
        names = ["resid_fine", "lsolve_fine", "usolve_fine", "gs_fine", "transfer", "coarse", "misc"]
        return dict(ms=dict(zip(names, out[:7].tolist())), launches=int(out[7]),
                    launches_by_class=dict(zip(names, out[8:15].astype(int).tolist())))


def build_hierarchy(problem, smoother="ilut", nu1=1, nu2=1, tau=1e-12, fillfactor=1.0, ordering="none"):
    """SPEC.md:327-335 (the degree list and h-chain come from the assembled ``problem``)."""
    H = PmgHierarchy(problem, smoother, nu1, nu2, tau, fillfactor, ordering)
    sizes = []
    if smoother == "ilut":
        sizes += [l.A.nrows for l in problem.plevels[:-1]]
    sizes += [h.A.nrows for h in problem.hlevels[:-1]]
    H._sizes = sizes
    return H


def prolongate(hier: PmgHierarchy, level: int, v, n_fine: int):
    v = _f64(v)
    out = np.empty(n_fine)
    _raise(lib().pmg_prolongate(hier.h, level, ptr(v), ptr(out)), what="prolongate")
    return out


def restrict(hier: PmgHierarchy, level: int, r, n_coarse: int):
    r = _f64(r)
    out = np.empty(n_coarse)
    _raise(lib().pmg_restrict(hier.h, level, ptr(r), ptr(out)), what="restrict")
    return out


def cycle(hier: PmgHierarchy, level: int, u, f):
    u = np.array(_f64(u), copy=True)
    with hier.work() as w:
        _raise(lib().pmg_cycle(w, level, ptr(u), ptr(_f64(f, u.size))), what="cycle")
    return u


def smooth(hier: PmgHierarchy, level: int, u, f):
    """One smoothing step at p-level `level` (the hierarchy's smoother; the building block of
    reduction_factors)."""
    u = np.array(_f64(u), copy=True)
    with hier.work() as w:
        _raise(lib().pmg_smooth(w, level, ptr(u), ptr(_f64(f, u.size))), what="smooth")
    return u


def coarse_correction(hier: PmgHierarchy, level: int, u, f):
    """One coarse-grid correction at p-level `level`: restrict f - A u, one cycle at level+1 from
    zero, prolongate and add (PAPER §4, steps 2-4 of the cycle)."""
    u = np.array(_f64(u), copy=True)
    with hier.work() as w:
        _raise(lib().pmg_coarse_correction(w, level, ptr(u), ptr(_f64(f, u.size))), what="coarse_correction")
    return u


def solve(hier: PmgHierarchy, f, tol=1e-8, max_cycles=200, guess=None):
    """Stand-alone p-multigrid solve. Returns (u, SolveReport)."""
    f = _f64(f, hier.n)
    u = np.zeros(hier.n) if guess is None else np.array(_f64(guess, hier.n), copy=True)
    hist = np.zeros(max_cycles + 1)
    cyc, flags, secs = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    with hier.work() as w:
        st = lib().pmg_solve(w, ptr(f), ptr(u), tol, max_cycles, ptr(hist), ctypes.byref(cyc), ctypes.byref(flags),
                             ctypes.byref(secs))
    _raise(st, what="solve")
    c = cyc.value
    return u, SolveReport(c, hist[: c + 1].copy(), bool(flags.value & 1), bool(flags.value & 2), hier.setup_seconds,
                          secs.value)


def bicgstab(hier: PmgHierarchy, f, tol=1e-8, max_iter=200, guess=None):
    """BiCGSTAB preconditioned by one V-cycle of `hier` (SPEC.md:269-277 with
    as_preconditioner). Returns (u, KrylovReport)."""
    f = _f64(f, hier.n)
    u = np.zeros(hier.n) if guess is None else np.array(_f64(guess, hier.n), copy=True)
    hist = np.zeros(max_iter + 1)
    it, flags, secs = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    with hier.work() as w:
        st = lib().pmg_bicgstab(w, ptr(f), ptr(u), tol, max_iter, ptr(hist), ctypes.byref(it), ctypes.byref(flags),
                                ctypes.byref(secs))
    _raise(st, what="bicgstab")
    k = it.value
    return u, KrylovReport(k, hist[: k + 1].copy(), bool(flags.value & 1), bool(flags.value & 2),
                           bool(flags.value & 4), secs.value)


def bicgstab_device(hier: PmgHierarchy, d_f: int, d_u: int, tol=1e-8, max_iter=200):
    """BiCGSTAB on device-resident vectors (raw device pointers)."""
    hist = np.zeros(max_iter + 1)
    it, flags, secs = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    with hier.work() as w:
        st = lib().pmg_bicgstab_device(w, ctypes.c_void_p(d_f), ctypes.c_void_p(d_u), tol, max_iter, ptr(hist),
                                       ctypes.byref(it), ctypes.byref(flags), ctypes.byref(secs))
    _raise(st, what="bicgstab_device")
    k = it.value
    return KrylovReport(k, hist[: k + 1].copy(), bool(flags.value & 1), bool(flags.value & 2), bool(flags.value & 4),
                        secs.value)


def solve_device(hier: PmgHierarchy, d_f: int, d_u: int, tol=1e-8, max_cycles=200):
    """Solve on device-resident vectors (raw device pointers, e.g. ``torch_tensor.data_ptr()``)."""
    hist = np.zeros(max_cycles + 1)
    cyc, flags, secs = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    with hier.work() as w:
        st = lib().pmg_solve_device(w, ctypes.c_void_p(d_f), ctypes.c_void_p(d_u), tol, max_cycles, ptr(hist),
                                    ctypes.byref(cyc), ctypes.byref(flags), ctypes.byref(secs))
    _raise(st, what="solve_device")
    c = cyc.value
    return SolveReport(c, hist[: c + 1].copy(), bool(flags.value & 1), bool(flags.value & 2), hier.setup_seconds,
                       secs.value)
