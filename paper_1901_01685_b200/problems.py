"""Problem / hierarchy inputs (``libiga_host.so``; matrix values optionally from the GPU).

The BASELINE.json configs 1-5 and the paper's Benchmarks 1-3.
Assembly is setup, not the solve path; it produces the FP64 CSR
operators both the CUDA path and the CPU oracle consume.  ``assembly="gpu"`` (F2,
SPEC.md:132-167) has ``libpmg_cuda.so``'s ``pmg_asm_values`` produce the values of every A_k,
M_k and P^k_j; the result equals the host element loop bit for bit.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._native import Csr, load, ptr

GEOM = {"square": 0, "annulus": 1, "lshape": 2}
RHS = {"sinsin": 0, "annulus": 1, "one": 2, "b1": 3, "b2": 4, "b3": 5}
MAT_A, MAT_P, MAT_PT, MAT_HA, MAT_HP, MAT_HPT = range(6)
VEC_ML, VEC_F, VEC_U0 = range(3)


class ProblemSpec(ctypes.Structure):
    _fields_ = [
        ("geometry", ctypes.c_int), ("rhs", ctypes.c_int), ("D", ctypes.c_double * 4),
        ("v", ctypes.c_double * 2), ("R", ctypes.c_double), ("h_exp", ctypes.c_int),
        ("coarsest_h_exp", ctypes.c_int), ("n_degrees", ctypes.c_int), ("degrees", ctypes.c_int * 8),
        ("random_guess", ctypes.c_int), ("seed", ctypes.c_uint64), ("nitsche_scale", ctypes.c_double),
        ("numbering", ctypes.c_int),
    ]


def _host():
    lib = load("libiga_host.so")
    if not getattr(lib, "_typed", False):
        lib.iga_last_error.restype = ctypes.c_char_p
        lib.iga_problem_build.argtypes = [ctypes.POINTER(ProblemSpec), ctypes.POINTER(ctypes.c_void_p)]
        lib.iga_problem_build_with.argtypes = [ctypes.POINTER(ProblemSpec), ctypes.c_void_p,
                                               ctypes.POINTER(ctypes.c_void_p)]
        lib.iga_problem_free.argtypes = [ctypes.c_void_p]
        for fn in ("iga_problem_num_plevels", "iga_problem_num_hlevels"):
            getattr(lib, fn).argtypes = [ctypes.c_void_p]
        lib.iga_problem_degree.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.iga_problem_csr_shape.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                              ctypes.POINTER(ctypes.c_int64)]
        lib.iga_problem_csr_copy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.iga_problem_csr_arrays.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_void_p)] * 3
        lib.iga_problem_vec_len.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.iga_problem_vec_copy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        lib.iga_config_spec.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ProblemSpec)]
        lib.iga_eval_basis.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_void_p]
        lib.iga_geometry_map.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_void_p]
        lib.iga_set_num_threads.argtypes = [ctypes.c_int]
        lib.iga_matrix_build.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                         ctypes.POINTER(ctypes.c_void_p)]
        lib.iga_matrix_build_with.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        lib._typed = True
    return lib


def _check(rc):
    if rc != 0:
        raise RuntimeError(_host().iga_last_error().decode())


def values_hook(assembly):
    """The ``pmg_asm_values_fn`` (include/pmg_asm.h) that produces matrix values: None / "host" =
    the host element loop, "gpu" = ``pmg_asm_values`` of libpmg_cuda.so (no fallback: a missing
    library or device raises), or a ctypes function pointer (tests)."""
    if assembly is None or assembly == "host":
        return None
    if assembly == "gpu":
        return ctypes.cast(load("libpmg_cuda.so").pmg_asm_values, ctypes.c_void_p)
    return ctypes.cast(assembly, ctypes.c_void_p)


@dataclass
class PLevel:
    degree: int
    A: Csr
    ML: np.ndarray
    P: Csr | None = None   # prolongation from the next (lower-degree) level to this one
    PT: Csr | None = None


@dataclass
class HLevel:
    A: Csr
    P: Csr | None = None   # prolongation from the next coarser h-level
    PT: Csr | None = None


@dataclass
class Problem:
    name: str
    spec: dict
    plevels: list[PLevel]
    hlevels: list[HLevel]   # hlevels[0].A is plevels[-1].A
    f: np.ndarray
    u0: np.ndarray
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.plevels[0].A.nrows


def config_spec(config: int, degree: int = 0) -> ProblemSpec:
    s = ProblemSpec()
    _check(_host().iga_config_spec(config, degree, ctypes.byref(s)))
    return s


NUMBERING = {"patch": 0, "rowmajor": 1}


def make_spec(geometry="square", rhs="one", degrees=(2, 1), h_exp=4, D=(1, 0, 0, 1), v=(0, 0), R=0.0,
              random_guess=False, seed=42, coarsest_h_exp=2, numbering="patch") -> ProblemSpec:
    s = ProblemSpec()
    s.geometry = GEOM[geometry]
    s.rhs = RHS[rhs]
    for i, d in enumerate(D):
        s.D[i] = d
    s.v[0], s.v[1] = v
    s.R = R
    s.h_exp = h_exp
    s.coarsest_h_exp = coarsest_h_exp
    s.n_degrees = len(degrees)
    for i, d in enumerate(degrees):
        s.degrees[i] = d
    s.random_guess = int(bool(random_guess))
    s.seed = seed
    s.numbering = NUMBERING[numbering]
    return s


def benchmark_spec(bench: int, p: int, h_exp: int, consecutive=True, seed=42) -> ProblemSpec:
    """Paper Benchmarks 1-3 with the paper's random initial guess.
    Benchmark 3 is the L-shape as 3 conforming patches with inhomogeneous Dirichlet
    data g = u_exact imposed through Nitsche and f = 0 (u_exact is harmonic)."""
    degrees = tuple(range(p, 0, -1)) if consecutive else (p, 1)
    if bench == 1:
        return make_spec("annulus", "b1", degrees, h_exp, random_guess=True, seed=seed)
    if bench == 2:
        return make_spec("square", "b2", degrees, h_exp, D=(1.2, -0.7, -0.4, 0.9), v=(0.4, -0.2), R=0.3,
                         random_guess=True, seed=seed)
    if bench == 3:
        return make_spec("lshape", "b3", degrees, h_exp, random_guess=True, seed=seed)
    raise ValueError(bench)


def set_threads(n: int) -> None:
    _host().iga_set_num_threads(n)


class _Owner:
    """Keeps a host problem alive while numpy arrays view its memory."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if self.h:
            self.lib.iga_problem_free(self.h)
            self.h = None


def _view(owner, address, ctype, n, dtype):
    if n == 0:
        return np.empty(0, dtype)
    buf = (ctype * n).from_address(address)
    buf._owner = owner  # the array's base chain reaches the owner
    return np.frombuffer(buf, dtype=dtype)


def _csr(lib, h, kind, l, owner=None) -> Csr:
    nr, nc, nnz = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    _check(lib.iga_problem_csr_shape(h, kind, l, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nnz)))
    if owner is not None and nnz.value <= np.iinfo(np.int32).max:
        # zero-copy views of columns and values (the big arrays); offsets converted to int32
        rp, ci, va = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.iga_problem_csr_arrays(h, kind, l, ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(va)))
        rowptr = _view(owner, rp.value, ctypes.c_int64, nr.value + 1, np.int64).astype(np.int32)
        return Csr(nr.value, nc.value, rowptr, _view(owner, ci.value, ctypes.c_int32, nnz.value, np.int32),
                   _view(owner, va.value, ctypes.c_double, nnz.value, np.float64))
    rowptr = np.empty(nr.value + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    _check(lib.iga_problem_csr_copy(h, kind, l, ptr(rowptr), ptr(col), ptr(val)))
    return Csr(nr.value, nc.value, rowptr, col, val)


def _vec(lib, h, kind, l) -> np.ndarray:
    n = lib.iga_problem_vec_len(h, kind, l)
    out = np.empty(n, np.float64)
    _check(lib.iga_problem_vec_copy(h, kind, l, ptr(out)))
    return out


def build(spec: ProblemSpec | int, degree: int = 0, name: str | None = None, assembly=None) -> Problem:
    """Assemble a problem: ``spec`` is a ProblemSpec or a BASELINE config number 1..5;
    ``assembly`` selects who produces the matrix values (see ``values_hook``)."""
    if isinstance(spec, int):
        name = name or (f"config{spec}" + (f"_p{degree}" if spec == 2 else ""))
        spec = config_spec(spec, degree)
    lib = _host()
    h = ctypes.c_void_p()
    _check(lib.iga_problem_build_with(ctypes.byref(spec), values_hook(assembly), ctypes.byref(h)))
    owner = _Owner(lib, h)  # frees the host problem once the last array viewing it is gone
    npl = lib.iga_problem_num_plevels(h)
    nhl = lib.iga_problem_num_hlevels(h)
    pl = []
    for l in range(npl):
        lev = PLevel(lib.iga_problem_degree(h, l), _csr(lib, h, MAT_A, l, owner), _vec(lib, h, VEC_ML, l))
        if l + 1 < npl:
            lev.P = _csr(lib, h, MAT_P, l, owner)
            lev.PT = _csr(lib, h, MAT_PT, l, owner)
        pl.append(lev)
    hl = []
    for j in range(nhl):
        A = pl[-1].A if j == 0 else _csr(lib, h, MAT_HA, j, owner)
        lev = HLevel(A)
        if j + 1 < nhl:
            lev.P = _csr(lib, h, MAT_HP, j, owner)
            lev.PT = _csr(lib, h, MAT_HPT, j, owner)
        hl.append(lev)
    f = _vec(lib, h, VEC_F, 0)
    u0 = _vec(lib, h, VEC_U0, 0)
    sd = {k: (list(getattr(spec, k)) if k in ("D", "v", "degrees") else getattr(spec, k)) for k, _ in spec._fields_}
    sd["degrees"] = sd["degrees"][: spec.n_degrees]
    return Problem(name or "custom", sd, pl, hl, f, u0)


def matrix(kind: str, geometry: str = "square", p: int = 1, nel: int = 1, p2: int = 1, D=(1, 0, 0, 1), v=(0, 0),
           R: float = 0.0, nitsche_scale: float = 0.0, assembly=None):
    """One assembled operator: kind in {"A", "M", "P", "ML"}.
    Returns a Csr (and, for "A", the load vector f = (1, v); for "ML", the lumped mass)."""
    lib = _host()
    k = {"A": 0, "M": 1, "P": 2, "ML": 3}[kind]
    Dv = np.ascontiguousarray(D, np.float64)
    vv = np.ascontiguousarray(v, np.float64)
    h = ctypes.c_void_p()
    _check(lib.iga_matrix_build_with(k, GEOM[geometry], p, p2, nel, ptr(Dv), ptr(vv), R, nitsche_scale,
                                     values_hook(assembly), ctypes.byref(h)))
    try:
        M = _csr(lib, h, MAT_A, 0)
        if kind == "A":
            return M, _vec(lib, h, VEC_F, 0)
        if kind == "ML":
            return M, _vec(lib, h, VEC_ML, 0)
        return M
    finally:
        lib.iga_problem_free(h)


def eval_basis(p: int, spans: int, x: float, deriv: bool = False):
    N = np.zeros(p + 1)
    dN = np.zeros(p + 1)
    first = _host().iga_eval_basis(p, spans, x, int(deriv), ptr(N), ptr(dN))
    if first < 0:
        raise ValueError(_host().iga_last_error().decode())
    return (first, N, dN) if deriv else (first, N)


def geometry_map(geometry: str, patch: int, xi: float, eta: float):
    X = np.zeros(2)
    J = np.zeros(4)
    _check(_host().iga_geometry_map(GEOM[geometry], patch, xi, eta, ptr(X), ptr(J)))
    return X, J.reshape(2, 2)
