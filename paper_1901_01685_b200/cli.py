"""`iga-pmg run | table` -- the experiment sweep surface of the reference (F4 of
SURVEY §8(f)), on the GPU solve path.

    python -m paper_1901_01685_b200.cli run   <config-file> [--out DIR] [--seed U64] [--threads N]
    python -m paper_1901_01685_b200.cli table <config-file> [--out DIR] [--seed U64] [--threads N]

A config file is flat `key = value` text, lists comma-separated, `#` comments:

    mode      = standalone | bicgstab | spectrum
    benchmark = 1, 2, 3
    p         = 2, 3, 4, 5
    h_exp     = 6, 7                                  (h = 2^-h_exp)
    smoother  = ilut, gs
    hierarchy = consecutive | direct                  (degree list p, p-1, .., 1 or p, 1)
    tol = 1e-8   max_cycles = 200   seed = 42        (seed default 42)

`run` sweeps every (benchmark, p, h_exp, smoother) cell -- build the problem and the hierarchy,
run the mode -- and writes into --out:

    results.csv              benchmark,p,h_exp,smoother,mode,value,status,setup_s,solve_s
    results.md               one table per (benchmark, smoother, mode): rows h, columns p,
                             divergence and failures rendered as "-"
    residuals_<cell>.txt     the residual history, one value per line (%.17g)

Rows are ordered by (benchmark, p, h_exp, smoother) whatever the completion order; a failing cell
is recorded in its row (status column) and never aborts the sweep; divergence is data, exit code 0
(SPEC.md:474, :488).  Reruns give byte-identical files apart from the timing columns (fixed seed,
deterministic kernels: every GPU result is bitwise reproducible).  `table` runs the sweep the same
way and prints results.md.  Every value is computed on the GPU (pmg.solve / pmg.bicgstab /
analysis.iteration_matrix); there is no CPU path."""
from __future__ import annotations

import argparse
import csv
import io
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

MODES = ("standalone", "bicgstab", "spectrum")
HEADER = ["benchmark", "p", "h_exp", "smoother", "mode", "value", "status", "setup_s", "solve_s"]


class ConfigError(ValueError):
    """A malformed config file (types.hpp's ConfigError convention)."""


@dataclass
class Config:
    mode: str = "standalone"
    benchmark: list = field(default_factory=lambda: [1])
    p: list = field(default_factory=lambda: [2])
    h_exp: list = field(default_factory=lambda: [4])
    smoother: list = field(default_factory=lambda: ["ilut"])
    hierarchy: str = "consecutive"
    tol: float = 1e-8
    max_cycles: int = 200
    seed: int = 42

    def cells(self):
        """(benchmark, p, h_exp, smoother) in the deterministic output order."""
        return [(b, p, h, s) for b in sorted(self.benchmark) for p in sorted(self.p) for h in sorted(self.h_exp)
                for s in self.smoother]


_INT_LISTS = ("benchmark", "p", "h_exp")


def parse_config(text: str) -> Config:
    c = Config()
    seen = set()
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {ln}: expected 'key = value': {raw!r}")
        k, v = (x.strip() for x in line.split("=", 1))
        if k in seen:
            raise ConfigError(f"line {ln}: duplicate key {k!r}")
        seen.add(k)
        items = [x.strip() for x in v.split(",") if x.strip()]
        try:
            if k in _INT_LISTS:
                setattr(c, k, [int(x) for x in items])
            elif k == "smoother":
                c.smoother = [x.lower() for x in items]
            elif k in ("mode", "hierarchy"):
                setattr(c, k, v.lower())
            elif k == "tol":
                c.tol = float(v)
            elif k in ("max_cycles", "seed"):
                setattr(c, k, int(v, 0))
            else:
                raise ConfigError(f"line {ln}: unknown key {k!r}")
        except ValueError as e:
            if isinstance(e, ConfigError):
                raise
            raise ConfigError(f"line {ln}: bad value for {k!r}: {v!r}") from e
    if c.mode not in MODES:
        raise ConfigError(f"mode must be one of {MODES}, not {c.mode!r}")
    if c.hierarchy not in ("consecutive", "direct"):
        raise ConfigError(f"hierarchy must be 'consecutive' or 'direct', not {c.hierarchy!r}")
    for s in c.smoother:
        if s not in ("ilut", "gs"):
            raise ConfigError(f"smoother must be ilut or gs, not {s!r}")
    if any(b not in (1, 2, 3) for b in c.benchmark):
        raise ConfigError(f"benchmark must be 1, 2 or 3: {c.benchmark}")
    if any(p < 1 or p > 7 for p in c.p) or any(h < 2 or h > 12 for h in c.h_exp):
        raise ConfigError(f"p in 1..7 and h_exp in 2..12 required: p={c.p} h_exp={c.h_exp}")
    if not (c.tol > 0) or c.max_cycles < 1:
        raise ConfigError("tol > 0 and max_cycles >= 1 required")
    return c


@dataclass
class Row:
    benchmark: int
    p: int
    h_exp: int
    smoother: str
    mode: str
    value: str          # cycles / iterations (int) or rho (%.6g); "" on failure
    status: str         # converged | diverged | not_converged | ok | error: <message>
    setup_s: float
    solve_s: float
    history: np.ndarray | None = None


def run_cell(cfg: Config, bench: int, p: int, h_exp: int, smoother: str, threads: int = 4) -> Row:
    """Build and run one cell on the GPU (any exception becomes the row's status)."""
    from . import analysis, pmg
    from . import problems as P

    t0 = time.perf_counter()
    try:
        spec = P.benchmark_spec(bench, p, h_exp, consecutive=cfg.hierarchy == "consecutive", seed=cfg.seed)
        pb = P.build(spec)
        H = pmg.build_hierarchy(pb, smoother=smoother)
        setup = time.perf_counter() - t0
        t1 = time.perf_counter()
        if cfg.mode == "standalone":
            _, rep = pmg.solve(H, pb.f, tol=cfg.tol, max_cycles=cfg.max_cycles, guess=pb.u0)
            status = "converged" if rep.converged else ("diverged" if rep.diverged else "not_converged")
            return Row(bench, p, h_exp, smoother, cfg.mode, str(rep.cycles), status, setup,
                       time.perf_counter() - t1, rep.residual_history)
        if cfg.mode == "bicgstab":
            _, rep = pmg.bicgstab(H, pb.f, tol=cfg.tol, max_iter=cfg.max_cycles, guess=pb.u0)
            status = ("converged" if rep.converged else "breakdown" if rep.breakdown
                      else "diverged" if rep.diverged else "not_converged")
            return Row(bench, p, h_exp, smoother, cfg.mode, str(rep.iterations), status, setup,
                       time.perf_counter() - t1, rep.residual_history)
        rho = analysis.spectral_radius(analysis.iteration_matrix(H, workers=threads)).rho
        return Row(bench, p, h_exp, smoother, cfg.mode, f"{rho:.6g}", "ok", setup, time.perf_counter() - t1)
    except Exception as e:  # recorded in-row, never aborts the sweep
        msg = " ".join(str(e).split())[:200]
        return Row(bench, p, h_exp, smoother, cfg.mode, "", f"error: {type(e).__name__}: {msg}",
                   time.perf_counter() - t0, 0.0)


def cell_name(r: Row) -> str:
    return f"b{r.benchmark}_p{r.p}_h{r.h_exp}_{r.smoother}_{r.mode}"


def to_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for r in rows:
        w.writerow([r.benchmark, r.p, r.h_exp, r.smoother, r.mode, r.value, r.status, f"{r.setup_s:.3f}",
                    f"{r.solve_s:.3f}"])
    return buf.getvalue()


def to_markdown(rows) -> str:
    """One table per (benchmark, smoother, mode): rows h = 2^-h_exp, columns p (the paper's layout);
    a diverged, unconverged or failed cell is "-"."""
    out = []
    groups = sorted({(r.benchmark, r.smoother, r.mode) for r in rows})
    for b, s, m in groups:
        g = [r for r in rows if (r.benchmark, r.smoother, r.mode) == (b, s, m)]
        ps = sorted({r.p for r in g})
        hs = sorted({r.h_exp for r in g})
        what = {"standalone": "V-cycles", "bicgstab": "BiCGSTAB iterations", "spectrum": "spectral radius"}[m]
        out.append(f"### Benchmark {b}, {s.upper() if s == 'gs' else 'ILUT'} smoother: {what}\n")
        out.append("| h | " + " | ".join(f"p = {p}" for p in ps) + " |")
        out.append("|---|" + "---|" * len(ps))
        cell = {(r.p, r.h_exp): r for r in g}
        for h in hs:
            vals = []
            for p in ps:
                r = cell.get((p, h))
                ok = r is not None and r.status in ("converged", "ok")
                vals.append(r.value if ok else "-")
            out.append(f"| 2^-{h} | " + " | ".join(vals) + " |")
        out.append("")
    return "\n".join(out)


def run(cfg: Config, out_dir: str, threads: int = 4, cell_fn=None) -> list[Row]:
    """Sweep every cell (sequentially: one GPU, cells already saturate it) and write the outputs."""
    cell_fn = cell_fn or (lambda b, p, h, s: run_cell(cfg, b, p, h, s, threads))
    rows = [cell_fn(b, p, h, s) for b, p, h, s in cfg.cells()]
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "results.csv"), "w") as fh:
        fh.write(to_csv(rows))
    with open(os.path.join(out_dir, "results.md"), "w") as fh:
        fh.write(to_markdown(rows))
    for r in rows:
        if r.history is not None:
            with open(os.path.join(out_dir, f"residuals_{cell_name(r)}.txt"), "w") as fh:
                fh.write("".join(f"{x:.17g}\n" for x in np.asarray(r.history, np.float64)))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="iga-pmg", description=__doc__.split("\n\n")[0])
    ap.add_argument("command", choices=("run", "table"))
    ap.add_argument("config")
    ap.add_argument("--out", default="results")
    ap.add_argument("--seed", type=lambda s: int(s, 0), default=None)
    ap.add_argument("--threads", type=int, default=4)
    a = ap.parse_args(argv)
    try:
        with open(a.config) as fh:
            cfg = parse_config(fh.read())
    except (OSError, ConfigError) as e:
        print(f"iga-pmg: {e}", file=sys.stderr)
        return 2
    if a.seed is not None:
        cfg.seed = a.seed
    from . import problems as P
    P.set_threads(max(1, a.threads))
    rows = run(cfg, a.out, a.threads)
    if a.command == "table":
        sys.stdout.write(to_markdown(rows))
    else:
        for r in rows:
            print(f"{cell_name(r)}: {r.value or '-'} ({r.status}) setup {r.setup_s:.2f}s solve {r.solve_s:.3f}s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
