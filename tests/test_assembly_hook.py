"""F2 plumbing on the CPU: the host library hands the matrix values of every operator to a
`pmg_asm_values_fn` (include/pmg_asm.h).  Here the producer is tests/cpp/asm_emulate.cpp, which runs
the GPU assembler's own per-phase code (csrc/cuda/asm_core.cuh, __host__ __device__) serially, so
the request, the index logic and the canonical accumulation order are checked bit for bit against
the host element loop without a GPU.  The CUDA kernels themselves: tests/test_gpu_assembly.py."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_1901_01685_b200 import problems as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("asm") / "libasm_emulate.so")
    cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-shared", "-o", so,
           os.path.join(ROOT, "tests", "cpp", "asm_emulate.cpp")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    return ctypes.CDLL(so).asm_emulate_values


def same(a, b):
    return a.shape == b.shape and bool((a.view(np.uint64) == b.view(np.uint64)).all())


def same_problem(a, b):
    for la, lb in zip(a.plevels, b.plevels):
        assert same(la.A.val, lb.A.val) and same(la.ML, lb.ML)
        assert (la.A.col == lb.A.col).all() and (la.A.rowptr == lb.A.rowptr).all()
        if la.P is not None:
            assert same(la.P.val, lb.P.val) and same(la.PT.val, lb.PT.val)
    for la, lb in zip(a.hlevels, b.hlevels):
        assert same(la.A.val, lb.A.val)
    assert same(a.f, b.f) and same(a.u0, b.u0)


@pytest.mark.parametrize("geom", ["square", "annulus", "lshape"])
@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_single_operators_bitwise(emu, geom, p):
    for nel in (1, 2, 5, 7):
        if p == 5 and nel > 5:
            continue
        kw = dict(D=(1.0, 0.3, 0.2, 1.5), v=(2, 3), R=3.0)
        A, f = P.matrix("A", geom, p, nel, **kw)
        A2, f2 = P.matrix("A", geom, p, nel, assembly=emu, **kw)
        assert same(A.val, A2.val) and same(f, f2)
        assert same(P.matrix("M", geom, p, nel).val, P.matrix("M", geom, p, nel, assembly=emu).val)
        if p > 1:
            for p2 in (1, p - 1):
                assert same(P.matrix("P", geom, p, nel, p2=p2).val, P.matrix("P", geom, p, nel, p2=p2, assembly=emu).val)


def test_problems_bitwise(emu):
    c4 = P.config_spec(4)
    c4.h_exp = 4  # config 4's L-shape in global row-major numbering, small
    for spec in (1, P.make_spec("annulus", "annulus", (3, 2, 1), 4), P.make_spec("lshape", "one", (4, 1), 3), c4):
        same_problem(P.build(spec), P.build(spec, assembly=emu))


def test_geometry_error_is_reported(emu):
    """status 1 of the producer maps to the host's geometry error"""
    bad = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)(lambda rq: 1)
    with pytest.raises(RuntimeError, match="Jacobian"):
        P.matrix("M", "square", 2, 2, assembly=bad)
    fail = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)(lambda rq: 3)
    with pytest.raises(RuntimeError, match="external assembler"):
        P.matrix("A", "square", 2, 2, assembly=fail)


def test_structure_is_independent_of_the_thread_count(emu):
    """patterns, transposes, load vector and values are bit-reproducible for any
    number of host workers -- host loop and external producer alike."""
    spec = P.make_spec("annulus", "annulus", (3, 2, 1), 4)
    ref = None
    try:
        for nt in (1, 3, 8):
            P.set_threads(nt)
            for asm in (None, emu):
                pb = P.build(spec, assembly=asm)
                if ref is None:
                    ref = pb
                else:
                    same_problem(ref, pb)
                    for la, lb in zip(ref.plevels, pb.plevels):
                        if la.PT is not None:
                            assert (la.PT.col == lb.PT.col).all() and (la.PT.rowptr == lb.PT.rowptr).all()
    finally:
        P.set_threads(0)
