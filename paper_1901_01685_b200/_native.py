"""ctypes loader for the in-tree native libraries.

``libpmg_cuda.so``  -- the CUDA solve path behind the C ABI of ``include/pmg_cuda.h``
``libiga_host.so``  -- host-side discretization (input generation, ``include/iga_host.h``)

Both are built in-tree by ``__graft_entry__.build()`` (``make``).  Nothing here falls
back to a CPU path: a missing library raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

LIBDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")

_libs: dict[str, ctypes.CDLL] = {}


def load(name: str) -> ctypes.CDLL:
    lib = _libs.get(name)
    if lib is None:
        # experiments: PMG_CUDA_LIB selects an alternative build of the CUDA library in LIBDIR
        alt = os.environ.get("PMG_CUDA_LIB") if name == "libpmg_cuda.so" else None
        path = os.path.join(LIBDIR, alt or name)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing -- run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
        _libs[name] = lib
    return lib


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Csr:
    """Host CSR: int32 row offsets and columns (sorted, unique), float64 values."""

    nrows: int
    ncols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    @classmethod
    def from_arrays(cls, nrows, ncols, rowptr, col, val) -> "Csr":
        return cls(int(nrows), int(ncols), np.ascontiguousarray(rowptr, dtype=np.int32),
                   np.ascontiguousarray(col, dtype=np.int32), np.ascontiguousarray(val, dtype=np.float64))

    @classmethod
    def from_dense(cls, M) -> "Csr":
        M = np.asarray(M, dtype=np.float64)
        rows, cols = np.nonzero(M)
        rowptr = np.zeros(M.shape[0] + 1, dtype=np.int32)
        np.add.at(rowptr, rows + 1, 1)
        return cls.from_arrays(M.shape[0], M.shape[1], np.cumsum(rowptr), cols, M[rows, cols])

    @classmethod
    def from_scipy(cls, S) -> "Csr":
        S = S.tocsr()
        S.sort_indices()
        return cls.from_arrays(S.shape[0], S.shape[1], S.indptr, S.indices, S.data)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.nrows, self.ncols))

    def to_dense(self) -> np.ndarray:
        D = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.rowptr[i], self.rowptr[i + 1]
            D[i, self.col[s:e]] = self.val[s:e]
        return D
