"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit for bit.

Bar (BASELINE.json north_star): identical V-cycle counts, per-cycle relative residuals within
1e-10 relative, final solution within 1e-12 relative in l2.  The kernels reproduce the
oracle's per-row operation order, so these tests assert BITWISE equality,
which implies every tolerance; the tolerance checks are kept explicitly as well.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_01685_b200 import pmg
from paper_1901_01685_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["wave", "skew", "chain", "levelsched"])
def sweep_path(request, monkeypatch):
    """Every sweep implementation must match the oracle: the default rotating-lane kernel
    (wave.cu), the skewed-warp kernel (PMG_WAVE=0), the chained-segment kernel (PMG_WAVE=0,
    PMG_SKEW=0) and the level-scheduled fallback."""
    monkeypatch.delenv("PMG_FORCE_LEVELSCHED", raising=False)
    monkeypatch.delenv("PMG_SKEW", raising=False)
    monkeypatch.delenv("PMG_WAVE", raising=False)
    if request.param == "levelsched":
        monkeypatch.setenv("PMG_FORCE_LEVELSCHED", "1")
    elif request.param == "chain":
        monkeypatch.setenv("PMG_WAVE", "0")
        monkeypatch.setenv("PMG_SKEW", "0")
    elif request.param == "skew":
        monkeypatch.setenv("PMG_WAVE", "0")
    return request.param


@pytest.fixture(params=["wave", "skew"])
def engine(request, monkeypatch):
    """The two wavefront kernels for tensor-grid factors: rotating lanes (wave.cu, default) and
    skewed warps (skew.cu, PMG_WAVE=0)."""
    monkeypatch.delenv("PMG_SKEW", raising=False)
    monkeypatch.delenv("PMG_FORCE_LEVELSCHED", raising=False)
    monkeypatch.delenv("PMG_WAVE", raising=False)
    if request.param == "skew":
        monkeypatch.setenv("PMG_WAVE", "0")
    return request.param

RTOL_RHO = 1e-10
RTOL_U = 1e-12


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, what
    bad = np.nonzero(bits(a) != bits(b))[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


_cache = {}


def problem(cfg, degree=0):
    key = (cfg, degree)
    if key not in _cache:
        _cache[key] = P.build(cfg, degree)
    return _cache[key]


@pytest.fixture(scope="module")
def cfg1():
    return problem(1)


def test_device_is_b200():
    info = pmg.device_info()
    assert info["cc"] == (10, 0), info


def test_spmv_residual_bitwise(cfg1):
    rng = np.random.default_rng(0)
    for lev in cfg1.plevels:
        A = lev.A
        x = rng.uniform(-1, 1, A.ncols)
        f = rng.uniform(-1, 1, A.nrows)
        assert_bitwise(pmg.spmv(A, x), O.spmv(A, x), "spmv")
        r, nrm = pmg.residual(A, x, f)
        ro = O.residual(A, x, f)
        assert_bitwise(r, ro, "residual")
        assert_bitwise([nrm], [O.norm2(ro)], "norm")


@pytest.mark.parametrize("ordering", ["none", "rcm"])
def test_ilut_factors_bitwise(cfg1, ordering, sweep_path):
    for lev in cfg1.plevels:
        A = lev.A
        Fg = pmg.ilut_factorize(A, 1e-12, 1.0, ordering)
        Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_RCM if ordering == "rcm" else O.ORDER_NONE)
        Lg, Ug, pg = Fg.export()
        Lo, Uo, po = Fo.export()
        np.testing.assert_array_equal(pg, po)
        for X, Y, nm in ((Lg, Lo, "L"), (Ug, Uo, "U")):
            np.testing.assert_array_equal(X.rowptr, Y.rowptr, err_msg=nm)
            np.testing.assert_array_equal(X.col, Y.col, err_msg=nm)
            assert_bitwise(X.val, Y.val, nm)
        so, sg = Fo.stats(), Fg.stats()
        assert sg["levels_L"] == so["levels_L"] and sg["levels_U"] == so["levels_U"]
        r = np.random.default_rng(1).uniform(-1, 1, A.nrows)
        assert_bitwise(pmg.ilut_apply(Fg, r), Fo.apply(r), "ilut_apply")


def test_gs_sweep_bitwise(cfg1, sweep_path):
    A = cfg1.plevels[0].A
    rng = np.random.default_rng(2)
    u = rng.uniform(-1, 1, A.nrows)
    f = rng.uniform(-1, 1, A.nrows)
    assert_bitwise(pmg.gauss_seidel_sweep(A, u, f), O.gauss_seidel_sweep(A, u, f), "gs")


def _solve_parity(pb, smoother="ilut", ordering="none"):
    Hg = pmg.build_hierarchy(pb, smoother=smoother, ordering=ordering)
    ug, rep = pmg.solve(Hg, pb.f, guess=pb.u0)
    Ho = O.Hierarchy(pb, smoother=O.GS if smoother == "gs" else O.ILUT,
                     ordering=O.ORDER_RCM if ordering == "rcm" else O.ORDER_NONE)
    uo, ro = Ho.solve(pb.f, pb.u0)
    assert rep.cycles == ro["cycles"], (rep.cycles, ro["cycles"])
    assert rep.converged == ro["converged"] and rep.diverged == ro["diverged"]
    np.testing.assert_allclose(rep.residual_history, ro["residual_history"], rtol=RTOL_RHO, atol=0)
    assert np.linalg.norm(ug - uo) <= RTOL_U * np.linalg.norm(uo)
    assert_bitwise(rep.residual_history, ro["residual_history"], "history")
    assert_bitwise(ug, uo, "solution")
    return rep, ro


@pytest.mark.parametrize("ordering", ["none", "rcm"])
def test_solve_config1(cfg1, ordering, sweep_path):
    rep, ro = _solve_parity(cfg1, "ilut", ordering)
    assert rep.converged


@pytest.mark.parametrize("degree", [2, 3, 4])
@pytest.mark.parametrize("smoother", ["ilut", "gs"])
def test_solve_config2(degree, smoother, sweep_path):
    _solve_parity(problem(2, degree), smoother)


def test_solve_config3(sweep_path):
    rep, _ = _solve_parity(problem(3), "ilut")
    assert rep.converged


@pytest.mark.parametrize("h_exp", [4, 5, 6, 8])
@pytest.mark.parametrize("geometry", ["square", "annulus"])
def test_skew_sweeps_p1(h_exp, geometry, engine):
    """The wavefront sweeps on p=1 factors: one 8-segment warp block (h=2^-4: 17 segments ->
    3 blocks), many blocks with halo hand-offs (2^-5 .. 2^-8), bitwise against the oracle."""
    spec = P.make_spec(geometry=geometry, rhs="one", degrees=(2, 1), h_exp=h_exp)
    A = P.build(spec).hlevels[0].A
    Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
    st = Fg.stats()
    assert st["sweep"] == engine, st
    Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE)
    rng = np.random.default_rng(h_exp)
    for _ in range(3):
        r = rng.uniform(-1, 1, A.nrows)
        assert_bitwise(pmg.ilut_apply(Fg, r), Fo.apply(r), "skew ilut_apply")


@pytest.mark.parametrize("env", [{"PMG_WAVE": "0", "PMG_SKEW_GRID": "3"}, {"PMG_WAVE_GRID": "3"},
                                 {"PMG_WAVE_GRID": "2", "PMG_WAVE_W": "1"}])
def test_skew_sweeps_cta_loops(env):
    """Fewer CTAs than warp blocks (PMG_SKEW_GRID / PMG_WAVE_GRID, read once per process): CTAs
    claim blocks in order and re-arm their barriers per block; also one sweep warp per CTA
    (PMG_WAVE_W=1).  Run in a subprocess so the settings stay local."""
    import os, subprocess, sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, '.');"
        "from oracle import oracle as O; from paper_1901_01685_b200 import pmg, problems as P;"
        "A = P.build(P.make_spec(geometry='annulus', rhs='one', degrees=(2, 1), h_exp=7)).hlevels[0].A;"
        "F = pmg.ilut_factorize(A, 1e-12, 1.0, 'none'); assert F.stats()['sweep'] == sys.argv[1];"
        "Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE);"
        "r = np.random.default_rng(3).uniform(-1, 1, A.nrows);"
        "e, eo = pmg.ilut_apply(F, r), Fo.apply(r);"
        "assert (e.view(np.uint64) == eo.view(np.uint64)).all(), 'mismatch'"
    )
    engine = "skew" if env.get("PMG_WAVE") == "0" else "wave"
    env = dict(os.environ, **env)
    env.pop("PMG_SKEW", None)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code, engine], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]


@pytest.mark.parametrize("p,h_exp", [(1, 5), (2, 6), (3, 6), (4, 6), (5, 6), (5, 7)])
def test_gs_sweep_skew_degrees(p, h_exp, engine):
    """Gauss-Seidel through the wavefront kernels (lower entries as terms, upper sums over the
    old values by a pre-pass) on A_p of every degree, bitwise against the oracle's sweep."""
    pb = P.build(P.make_spec(geometry="annulus", rhs="one", degrees=(max(p, 2), 1), h_exp=h_exp))
    A = pb.hlevels[0].A if p == 1 else pb.plevels[0].A
    rng = np.random.default_rng(p)
    u = rng.uniform(-1, 1, A.nrows)
    f = rng.uniform(-1, 1, A.nrows)
    assert_bitwise(pmg.gauss_seidel_sweep(A, u, f), O.gauss_seidel_sweep(A, u, f), "gs skew")


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_skew_sweeps_long_rows(p, engine):
    """The wavefront layouts for long rows (8x4, 16x4, 32x3, 32x4 lanes x terms; up to five
    segments back): ilut_apply on the p-level factor, bitwise against the oracle."""
    pb = P.build(P.make_spec(geometry="annulus", rhs="one", degrees=(p, 1), h_exp=6))
    A = pb.plevels[0].A
    Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
    assert Fg.stats()["sweep"] == engine
    Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE)
    r = np.random.default_rng(p).uniform(-1, 1, A.nrows)
    assert_bitwise(pmg.ilut_apply(Fg, r), Fo.apply(r), "skew ilut_apply")


def test_concurrent_solves_share_a_hierarchy():
    """the hierarchy is immutable and shareable, each solve owns its vectors.
    Two host threads solve on one hierarchy through two work objects at once (their sweeps run
    concurrently on two streams); both must equal the oracle bit for bit."""
    import ctypes
    import threading
    pb = P.build(P.make_spec(geometry="annulus", rhs="annulus", degrees=(3, 1), h_exp=6))
    Hg = pmg.build_hierarchy(pb, smoother="ilut")
    uo, ro = O.Hierarchy(pb, smoother=O.ILUT).solve(pb.f, pb.u0)
    L = pmg.lib()
    w2 = ctypes.c_void_p()
    assert L.pmg_work_create(Hg.h, ctypes.byref(w2)) == 0
    results = {}

    def run(tag, work):
        u = np.array(pb.u0, dtype=np.float64, copy=True)
        hist = np.zeros(201)
        cyc, flags, secs = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        for _ in range(3):
            u[:] = pb.u0
            st = L.pmg_solve(work, pmg.ptr(np.ascontiguousarray(pb.f)), pmg.ptr(u), 1e-8, 200, pmg.ptr(hist),
                             ctypes.byref(cyc), ctypes.byref(flags), ctypes.byref(secs))
            assert st == 0
        results[tag] = (u.copy(), cyc.value)

    try:
        ts = [threading.Thread(target=run, args=("a", Hg.w)), threading.Thread(target=run, args=("b", w2.value))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        L.pmg_work_destroy(w2.value)
    for tag in ("a", "b"):
        u, c = results[tag]
        assert c == ro["cycles"]
        assert_bitwise(u, uo, f"concurrent solve {tag}")


def test_concurrent_python_solves_share_a_hierarchy():
    """pmg.solve from two Python threads on one PmgHierarchy (ctypes releases the GIL)
    takes a work object per call from the hierarchy's pool; both results equal the oracle."""
    import threading
    pb = P.build(P.make_spec(geometry="annulus", rhs="annulus", degrees=(3, 1), h_exp=6))
    Hg = pmg.build_hierarchy(pb, smoother="ilut")
    uo, ro = O.Hierarchy(pb, smoother=O.ILUT).solve(pb.f, pb.u0)
    results, errors = {}, []

    def run(tag):
        try:
            for _ in range(4):
                u, rep = pmg.solve(Hg, pb.f, guess=pb.u0)
            results[tag] = (u, rep.cycles)
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=run, args=(t,)) for t in "ab"]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for tag in "ab":
        u, c = results[tag]
        assert c == ro["cycles"]
        assert_bitwise(u, uo, f"python concurrent solve {tag}")


def test_p1_only_hierarchy_converges():
    """degrees (1,) -- the hierarchy is the h-multigrid solver alone.
    Each cycle corrects the current iterate (e = hmg(f - A u), u += e) and converges like the
    oracle, bit for bit."""
    pb = P.build(P.make_spec(geometry="square", rhs="one", degrees=(1,), h_exp=5))
    Hg = pmg.build_hierarchy(pb, smoother="ilut")
    u, rep = pmg.solve(Hg, pb.f, guess=pb.u0)
    uo, ro = O.Hierarchy(pb, smoother=O.ILUT).solve(pb.f, pb.u0)
    assert ro["converged"] and rep.converged
    assert rep.cycles == ro["cycles"] < 20
    assert_bitwise(u, uo, "p=1-only solve")


@pytest.mark.parametrize("p,h_exp", [(1, 5), (2, 5), (4, 5), (4, 6)])
def test_wave_variable_segments_lshape(p, h_exp):
    """Rotating-lane sweeps on grid rows of different lengths: the L-shape (3 patches) in global
    row-major numbering has rows of 2n-1 DOFs below y = 0 and n above (segments detected from the
    pattern).  ILUT apply and the GS sweep, bitwise against the oracle."""
    pb = P.build(P.make_spec(geometry="lshape", rhs="one", degrees=(max(p, 2), 1), h_exp=h_exp, numbering="rowmajor"))
    A = pb.hlevels[0].A if p == 1 else pb.plevels[0].A
    Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
    assert Fg.stats()["sweep"] == "wave", Fg.stats()
    Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE)
    rng = np.random.default_rng(p)
    r = rng.uniform(-1, 1, A.nrows)
    assert_bitwise(pmg.ilut_apply(Fg, r), Fo.apply(r), "wave ilut_apply (variable segments)")
    u, f = rng.uniform(-1, 1, A.nrows), rng.uniform(-1, 1, A.nrows)
    assert_bitwise(pmg.gauss_seidel_sweep(A, u, f), O.gauss_seidel_sweep(A, u, f), "wave GS (variable segments)")


def test_solve_lshape_rowmajor():
    """A whole p-MG solve on the row-major L-shape (config 4's numbering at h = 2^-5), bitwise."""
    pb = P.build(P.make_spec(geometry="lshape", rhs="one", degrees=(4, 1), h_exp=5, numbering="rowmajor"))
    Hg = pmg.build_hierarchy(pb, smoother="ilut")
    assert all(F.stats()["sweep"] == "wave" for F in Hg.factors())
    u, rep = pmg.solve(Hg, pb.f, guess=pb.u0)
    uo, ro = O.Hierarchy(pb, smoother=O.ILUT).solve(pb.f, pb.u0)
    assert rep.cycles == ro["cycles"] and rep.converged
    assert_bitwise(u, uo, "L-shape row-major solve")
