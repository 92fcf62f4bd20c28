"""MatrixMarket import / export over the host library's C ABI
(include/iga_host.h): CSR matrices <-> `matrix coordinate real general` files, vectors <->
one-column `array` files or plain text.  Values are written with %.17g, so a write / read round
trip is exact."""
from __future__ import annotations

import ctypes

import numpy as np

from ._native import Csr, ptr
from .problems import _host

_i32p, _i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)


def _lib():
    L = _host()
    if not getattr(L, "_mm_ready", False):
        vp, cp = ctypes.c_void_p, ctypes.c_char_p
        L.iga_mm_last_error.restype = cp
        L.iga_mm_read_shape.argtypes = [cp, _i32p, _i32p, _i64p]
        L.iga_mm_read.argtypes = [cp, vp, vp, vp]
        L.iga_mm_write.argtypes = [cp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, cp]
        L.iga_mm_write_vector.argtypes = [cp, ctypes.c_int32, vp]
        L.iga_mm_read_vector_len.argtypes = [cp, _i32p]
        L.iga_mm_read_vector.argtypes = [cp, vp]
        L._mm_ready = True
    return L


def _check(L, rc):
    if rc != 0:
        raise OSError(L.iga_mm_last_error().decode())


def read_matrix(path) -> Csr:
    L = _lib()
    p = str(path).encode()
    m, n, nnz = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    _check(L, L.iga_mm_read_shape(p, ctypes.byref(m), ctypes.byref(n), ctypes.byref(nnz)))
    rp = np.empty(m.value + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    _check(L, L.iga_mm_read(p, ptr(rp), ptr(col), ptr(val)))
    return Csr(m.value, n.value, rp, col, val)


def write_matrix(path, A: Csr, comment: str | None = None) -> None:
    L = _lib()
    rp = np.ascontiguousarray(A.rowptr, np.int32)
    col = np.ascontiguousarray(A.col, np.int32)
    val = np.ascontiguousarray(A.val, np.float64)
    _check(L, L.iga_mm_write(str(path).encode(), A.nrows, A.ncols, ptr(rp), ptr(col), ptr(val),
                             comment.encode() if comment else None))


def write_vector(path, v) -> None:
    L = _lib()
    v = np.ascontiguousarray(v, np.float64)
    _check(L, L.iga_mm_write_vector(str(path).encode(), v.size, ptr(v)))


def read_vector(path) -> np.ndarray:
    L = _lib()
    p = str(path).encode()
    n = ctypes.c_int32()
    _check(L, L.iga_mm_read_vector_len(p, ctypes.byref(n)))
    v = np.empty(n.value, np.float64)
    _check(L, L.iga_mm_read_vector(p, ptr(v)))
    return v
