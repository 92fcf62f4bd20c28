"""F4: the `iga-pmg run | table` surface: config parsing, the deterministic
results.csv / results.md / residuals_<cell>.txt outputs, failures recorded in-row.  The sweep
itself runs on the GPU (tests/test_gpu_cli.py); here the cell runner is a stub."""
import glob
import os

import numpy as np
import pytest

from paper_1901_01685_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse_config_and_errors():
    c = cli.parse_config("# comment\nmode = bicgstab\nbenchmark = 2, 1\np = 3,2\nh_exp = 5\n"
                         "smoother = ILUT, gs  # trailing\nseed = 0x10\ntol = 1e-6\n")
    assert (c.mode, c.benchmark, c.p, c.h_exp, c.smoother, c.seed, c.tol) == \
        ("bicgstab", [2, 1], [3, 2], [5], ["ilut", "gs"], 16, 1e-6)
    assert c.cells()[0] == (1, 2, 5, "ilut") and c.cells()[-1] == (2, 3, 5, "gs")
    for bad in ("mode = wcycle", "p = two", "colour = red", "benchmark = 4", "smoother = jacobi",
                "p = 2\np = 3", "just words", "tol = 0"):
        with pytest.raises(cli.ConfigError):
            cli.parse_config(bad)


def test_shipped_table_configs_parse():
    files = sorted(glob.glob(os.path.join(ROOT, "tables", "*.cfg")))
    assert len(files) == 8
    for f in files:
        with open(f) as fh:
            c = cli.parse_config(fh.read())
        assert c.cells()


def _stub(cfg):
    def cell(b, p, h, s):
        if p == 3 and s == "gs":
            return cli.Row(b, p, h, s, cfg.mode, "", "error: RuntimeError: boom", 0.1, 0.0)
        if s == "gs":
            return cli.Row(b, p, h, s, cfg.mode, "200", "diverged", 0.1, 0.2, np.array([1.0, 3.0, 1e11]))
        return cli.Row(b, p, h, s, cfg.mode, str(p + h), "converged", 0.1, 0.2, np.array([1.0, 0.1 / 3, 1e-9]))
    return cell


def test_run_writes_deterministic_outputs(tmp_path):
    cfg = cli.parse_config("benchmark = 1\np = 2, 3\nh_exp = 4, 5\nsmoother = ilut, gs\n")
    rows = cli.run(cfg, str(tmp_path), cell_fn=_stub(cfg))
    assert len(rows) == 8
    csv = (tmp_path / "results.csv").read_text().splitlines()
    assert csv[0] == "benchmark,p,h_exp,smoother,mode,value,status,setup_s,solve_s"
    assert csv[1] == "1,2,4,ilut,standalone,6,converged,0.100,0.200"
    assert any(",error: RuntimeError: boom," in l for l in csv)  # recorded in-row, sweep continued
    md = (tmp_path / "results.md").read_text()
    assert "| 2^-4 | 6 | 7 |" in md and "| 2^-5 | - | - |" in md  # GS diverged / failed -> "-"
    hist = (tmp_path / "residuals_b1_p2_h4_ilut_standalone.txt").read_text().splitlines()
    assert [float(x) for x in hist] == [1.0, 0.1 / 3, 1e-9]  # %.17g round-trips exactly
    assert not (tmp_path / "residuals_b1_p3_h4_gs_standalone.txt").exists()
    cli.run(cfg, str(tmp_path / "again"), cell_fn=_stub(cfg))
    assert (tmp_path / "again" / "results.csv").read_text() == (tmp_path / "results.csv").read_text()


def test_main_bad_config_exit_code(tmp_path, capsys):
    p = tmp_path / "bad.cfg"
    p.write_text("mode = nope\n")
    assert cli.main(["run", str(p), "--out", str(tmp_path / "o")]) == 2
    assert "mode must be" in capsys.readouterr().err
