"""The drop-in boundary without a GPU: every symbol declared in include/*.h is exported by
the in-tree libraries, the C++ API compiles against include/iga/pmg.hpp, and with no CUDA
device the product path fails loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1901_01685_b200", "lib")


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:pmg|iga)_[a-z0-9_]+)\s*\(", src)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(LIB, lib)], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


@pytest.mark.parametrize("header,lib", [("pmg_cuda.h", "libpmg_cuda.so"), ("iga_host.h", "libiga_host.so")])
def test_every_declared_symbol_is_exported(header, lib):
    names = declared(header)
    assert len(names) > 10
    missing = [n for n in names if n not in exported(lib)]
    assert not missing, missing


def test_libraries_load():
    for lib in ("libpmg_cuda.so", "libiga_host.so", "libiga_pmg.so"):
        ctypes.CDLL(os.path.join(LIB, lib))


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(LIB, "libpmg_cuda.so")], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_cpp_api_compiles(tmp_path):
    src = tmp_path / "use_api.cpp"
    src.write_text(r'''
#include "iga/pmg.hpp"
#include <cstdio>
int main() {
    iga::CsrMatrix A;
    A.nrows = A.ncols = 2;
    A.row_offsets = {0, 2, 4};
    A.col_indices = {0, 1, 0, 1};
    A.values = {4, 1, 1, 3};
    try {
        auto fac = iga::ilut_factorize(A, 0.0, 10.0, iga::Ordering::none);   // SPEC.md:258
        auto e = iga::ilut_apply(fac, {5.0, 4.0});                          // SPEC.md:267
        std::printf("%.17g %.17g\n", e[0], e[1]);
    } catch (const iga::FactorizationError& err) {
        std::printf("zero pivot at row %lld\n", (long long)err.row);
        return 2;
    } catch (const iga::DeviceError& err) {
        std::printf("device: %s\n", err.what());
        return 3;
    }
    return 0;
}
''')
    exe = tmp_path / "use_api"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", LIB, "-liga_pmg", "-lpmg_cuda", f"-Wl,-rpath,{LIB}"], check=True)
    assert exe.exists()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    from paper_1901_01685_b200 import pmg
    from paper_1901_01685_b200._native import Csr
    with pytest.raises(pmg.CudaError):
        pmg.device_info()
    with pytest.raises(pmg.CudaError):
        pmg.spmv(Csr.from_dense(np.eye(3)), np.ones(3))


def test_rcm_product_matches_oracle():
    """The product's host RCM (setup) and the oracle's restatement give the same permutation."""
    from oracle import oracle as O
    from paper_1901_01685_b200 import pmg
    from paper_1901_01685_b200 import problems as P
    for geometry, p, nel in (("annulus", 3, 8), ("lshape", 2, 8), ("square", 4, 16)):
        A, _ = P.matrix("A", geometry, p=p, nel=nel)
        np.testing.assert_array_equal(pmg.rcm_ordering(A), O.rcm_ordering(A))


def test_invalid_csr_rejected():
    from paper_1901_01685_b200 import pmg
    from paper_1901_01685_b200._native import Csr
    bad = Csr(2, 2, np.array([0, 2, 3], np.int32), np.array([1, 0, 1], np.int32), np.ones(3))  # unsorted row
    with pytest.raises(ValueError):
        pmg.rcm_ordering(bad)
