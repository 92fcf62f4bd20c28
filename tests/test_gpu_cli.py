"""F4 on the GPU: `iga-pmg run` over a small Benchmark-1 sweep; the cycle counts and residual
histories equal the oracle's, reruns give byte-identical results apart from the timing columns
(SPEC.md:480)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_01685_b200 import cli
from paper_1901_01685_b200 import problems as P

pytestmark = pytest.mark.gpu


def _strip_times(text):
    return [",".join(l.split(",")[:7]) for l in text.splitlines()]


def test_cli_standalone_sweep(tmp_path):
    cfg_file = tmp_path / "t.cfg"
    cfg_file.write_text("mode = standalone\nbenchmark = 1\np = 2, 3\nh_exp = 3, 4\nsmoother = ilut, gs\n")
    assert cli.main(["run", str(cfg_file), "--out", str(tmp_path / "a")]) == 0
    assert cli.main(["table", str(cfg_file), "--out", str(tmp_path / "b")]) == 0
    a = (tmp_path / "a" / "results.csv").read_text()
    assert _strip_times(a) == _strip_times((tmp_path / "b" / "results.csv").read_text())
    rows = [l.split(",") for l in a.splitlines()[1:]]
    assert len(rows) == 8
    for b, p, h, s, mode, value, status, *_ in rows:
        pb = P.build(P.benchmark_spec(int(b), int(p), int(h), seed=42))
        Ho = O.Hierarchy(pb, smoother=O.ILUT if s == "ilut" else O.GS)
        _, ro = Ho.solve(pb.f, pb.u0)
        assert int(value) == ro["cycles"] and status == "converged"
        hist = np.loadtxt(tmp_path / "a" / f"residuals_b{b}_p{p}_h{h}_{s}_{mode}.txt")
        np.testing.assert_array_equal(hist, ro["residual_history"])


def test_cli_spectrum_and_bicgstab(tmp_path):
    for mode in ("spectrum", "bicgstab"):
        f = tmp_path / f"{mode}.cfg"
        f.write_text(f"mode = {mode}\nbenchmark = 2\np = 2\nh_exp = 3\nsmoother = ilut\n")
        assert cli.main(["run", str(f), "--out", str(tmp_path / mode)]) == 0
        row = (tmp_path / mode / "results.csv").read_text().splitlines()[1].split(",")
        assert row[6] in ("ok", "converged"), row
        if mode == "spectrum":
            assert 0 < float(row[5]) < 0.2
