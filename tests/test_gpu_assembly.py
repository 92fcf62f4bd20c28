"""F2: GPU assembly (pmg_asm_values, csrc/cuda/assemble.cu) against the host element loop of
libiga_host.so -- the CPU implementation of SPEC.md:132-167 in this repository (the reference has
no assembler).  Bar: bit-exact values of every A_k, M_k (through the lumped masses),
P^k_j and the p=1 h-chain operators; patterns and the load vector come from the host either way."""
import numpy as np
import pytest

from paper_1901_01685_b200 import pmg, problems as P

pytestmark = pytest.mark.gpu


def same(a, b):
    return a.shape == b.shape and bool((a.view(np.uint64) == b.view(np.uint64)).all())


def same_problem(a, b):
    for la, lb in zip(a.plevels, b.plevels):
        assert same(la.A.val, lb.A.val) and same(la.ML, lb.ML)
        if la.P is not None:
            assert same(la.P.val, lb.P.val) and same(la.PT.val, lb.PT.val)
    for la, lb in zip(a.hlevels, b.hlevels):
        assert same(la.A.val, lb.A.val)
    assert same(a.f, b.f)


@pytest.mark.parametrize("geom", ["square", "annulus", "lshape"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_single_operators_bitwise(geom, p):
    kw = dict(D=(1.0, 0.3, 0.2, 1.5), v=(2, 3), R=3.0)
    for nel in (1, 2, 7, 16):
        A, f = P.matrix("A", geom, p, nel, **kw)
        A2, f2 = P.matrix("A", geom, p, nel, assembly="gpu", **kw)
        assert same(A.val, A2.val) and same(f, f2), (geom, p, nel, float(np.abs(A.val - A2.val).max()))
        assert same(P.matrix("M", geom, p, nel).val, P.matrix("M", geom, p, nel, assembly="gpu").val)
        if p > 1:
            for p2 in {1, p - 1}:
                assert same(P.matrix("P", geom, p, nel, p2=p2).val, P.matrix("P", geom, p, nel, p2=p2, assembly="gpu").val)


def test_chunked_buffer_bitwise(monkeypatch):
    """element matrices staged through a buffer smaller than the patch: several chunks of DOF rows"""
    import subprocess, sys, os
    code = ("import numpy as np; from paper_1901_01685_b200 import problems as P;"
            "A,_=P.matrix('A','annulus',3,64); B,_=P.matrix('A','annulus',3,64,assembly='gpu');"
            "T=P.matrix('P','annulus',4,64,p2=1); T2=P.matrix('P','annulus',4,64,p2=1,assembly='gpu');"
            "assert (A.val.view(np.uint64)==B.val.view(np.uint64)).all();"
            "assert (T.val.view(np.uint64)==T2.val.view(np.uint64)).all(); print('ok')")
    env = dict(os.environ, PMG_ASM_CHUNK_MB="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]


@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_configs_bitwise(config):
    same_problem(P.build(config), P.build(config, assembly="gpu"))


def test_spec_invariants_on_gpu_values():
    """mass entries >= 0 with sum = area; transfer preserves constants"""
    M = P.matrix("M", "annulus", 3, 16, assembly="gpu")
    assert (M.val >= 0).all() and abs(M.val.sum() - 0.75 * np.pi) < 1e-10
    _, ML = P.matrix("ML", "annulus", 3, 16, assembly="gpu")
    T = P.matrix("P", "annulus", 3, 16, p2=2, assembly="gpu")
    ones = np.add.reduceat(T.val, T.rowptr[:-1]) / ML
    assert np.abs(ones - 1).max() < 1e-10


def test_gpu_assembled_solve_matches_host_assembled():
    pb = P.build(2, 3, assembly="gpu")
    ph = P.build(2, 3)
    H = pmg.build_hierarchy(pb, smoother="ilut")
    u, rep = pmg.solve(H, pb.f, guess=pb.u0)
    Hh = pmg.build_hierarchy(ph, smoother="ilut")
    uh, reph = pmg.solve(Hh, ph.f, guess=ph.u0)
    assert rep.cycles == reph.cycles and same(u, uh)


@pytest.mark.slow
def test_config5_bitwise():
    same_problem(P.build(5), P.build(5, assembly="gpu"))
