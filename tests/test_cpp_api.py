"""The C++ solver API (include/iga/pmg.hpp over libiga_pmg.so, the reference's language) compiled
and RUN on config 1 (tests/cpp/api_config1.cpp): every result equals the CPU oracle bit for bit."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1901_01685_b200", "lib")


def _compile(tmp_path):
    exe = str(tmp_path / "api_config1")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "api_config1.cpp"),
           "-L", LIB, "-liga_pmg", "-liga_host", "-lpmg_cuda", f"-Wl,-rpath,{LIB}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    return exe


def test_cpp_api_compiles(tmp_path):
    """CPU: the C++ program links against the three in-tree libraries."""
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_cpp_api_config1_bitwise(tmp_path):
    from oracle import oracle as O
    from paper_1901_01685_b200 import problems as P
    exe = _compile(tmp_path)
    res = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    info = json.loads(res.stdout.strip().splitlines()[-1])
    rd = lambda name: np.fromfile(tmp_path / name, dtype=np.float64)
    bits = lambda a: np.ascontiguousarray(a, np.float64).view(np.uint64)

    pb = P.build(1)
    H = O.Hierarchy(pb, smoother=O.ILUT)
    uo, ro = H.solve(pb.f, pb.u0)
    assert info["converged"] == 1 and info["cycles"] == ro["cycles"]
    assert (bits(rd("solve_u.bin")) == bits(uo)).all()
    assert (bits(rd("solve_hist.bin")) == bits(ro["residual_history"])).all()

    Fo = O.ilut_factorize(pb.plevels[0].A, 1e-12, 1.0, O.ORDER_NONE)
    assert (bits(rd("ilut_apply.bin")) == bits(Fo.apply(pb.f))).all()

    ub, kr = H.bicgstab(pb.f, pb.u0)
    assert info["bicgstab_iterations"] == kr["iterations"]
    assert (bits(rd("bicgstab_u.bin")) == bits(ub)).all()
    assert (bits(rd("bicgstab_hist.bin")) == bits(kr["residual_history"])).all()

    l0 = pb.plevels[0]
    rc = O.restrict(l0.PT, pb.plevels[1].ML, pb.f)
    assert (bits(rd("restrict.bin")) == bits(rc)).all()
    assert (bits(rd("prolongate.bin")) == bits(O.prolongate(l0.P, l0.ML, rc))).all()
    assert info["zero_pivot_row"] == 0
