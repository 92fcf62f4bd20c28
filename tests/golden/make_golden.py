"""Generate tests/golden/golden.json with the CPU oracle (run here, offline; ~20 min for config 5).

For every BASELINE config run (and BiCGSTAB with the p-MG preconditioner): V-cycle count, convergence flags, the residual history as
hex floats, SHA-256 + l2 norm of the solution, and per ILUT factor its nnz, level counts
and SHA-256 (rowptr|col|val bytes).  The GPU parity tests compare against these when the
oracle itself would be too slow to rerun on the GPU box (config 5), and the CPU tests pin
the oracle against them (regression).

The reference has no fixtures or golden vectors of its own; these are the
oracle's outputs, i.e. "parity unpinned by the reference".

    python tests/golden/make_golden.py [--skip5]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1901_01685_b200 import problems as P  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def factor_record(F):
    L, U, perm = F.export()
    st = F.stats()
    return dict(nnz_L=st["nnz_L"], nnz_U=st["nnz_U"], levels_L=st["levels_L"], levels_U=st["levels_U"],
                sha_L=sha(L.rowptr, L.col, L.val), sha_U=sha(U.rowptr, U.col, U.val), sha_perm=sha(perm))


def run(pb, smoother, ordering):
    t0 = time.time()
    H = O.Hierarchy(pb, smoother=O.GS if smoother == "gs" else O.ILUT,
                    ordering=O.ORDER_RCM if ordering == "rcm" else O.ORDER_NONE)
    setup = time.time() - t0
    u, rep = H.solve(pb.f, pb.u0)
    rec = dict(cycles=rep["cycles"], converged=rep["converged"], diverged=rep["diverged"],
               residual_history=[float(x).hex() for x in rep["residual_history"]],
               u_sha256=sha(u), u_l2=float(np.linalg.norm(u)).hex(),
               factors=[factor_record(F) for F in H.factors()],
               oracle_setup_s=round(setup, 2), oracle_solve_s=round(rep["solve_seconds"], 3))
    print(f"  {smoother}/{ordering}: {rep['cycles']} cycles conv={rep['converged']} div={rep['diverged']} "
          f"setup {setup:.1f}s solve {rep['solve_seconds']:.2f}s", flush=True)
    return rec


def run_bicgstab(pb):
    t0 = time.time()
    H = O.Hierarchy(pb)
    setup = time.time() - t0
    u, rep = H.bicgstab(pb.f, pb.u0)
    rec = dict(iterations=rep["iterations"], converged=rep["converged"], breakdown=rep["breakdown"],
               residual_history=[float(x).hex() for x in rep["residual_history"]], u_sha256=sha(u),
               oracle_setup_s=round(setup, 2), oracle_solve_s=round(rep["solve_seconds"], 3))
    print(f"  bicgstab: {rep['iterations']} iterations conv={rep['converged']} setup {setup:.1f}s "
          f"solve {rep['solve_seconds']:.2f}s", flush=True)
    return rec


def main():
    runs = [(1, 0, "ilut", "none"), (1, 0, "ilut", "rcm"),
            (2, 2, "ilut", "none"), (2, 3, "ilut", "none"), (2, 4, "ilut", "none"),
            (2, 2, "gs", "none"), (2, 3, "gs", "none"), (2, 4, "gs", "none"),
            (3, 0, "ilut", "none"), (4, 0, "ilut", "none")]
    runs += [(1, 0, "bicgstab", "none"), (2, 3, "bicgstab", "none"), (3, 0, "bicgstab", "none"),
             (4, 0, "bicgstab", "none")]
    if "--skip5" not in sys.argv:
        runs += [(5, 0, "ilut", "none"), (5, 0, "gs", "none"), (5, 0, "bicgstab", "none")]
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    golden = {}
    if os.path.exists(out_path):
        with open(out_path) as fh:
            golden = json.load(fh)
    cache = {}
    for cfg, deg, smoother, ordering in runs:
        key = f"config{cfg}" + (f"_p{deg}" if cfg == 2 else "") + (
            "/ilut/none/bicgstab" if smoother == "bicgstab" else f"/{smoother}/{ordering}")
        if key in golden:
            continue
        print(key, flush=True)
        if (cfg, deg) not in cache:
            cache.clear()
            cache[(cfg, deg)] = P.build(cfg, deg)
        if smoother == "bicgstab":
            golden[key] = run_bicgstab(cache[(cfg, deg)])
        else:
            golden[key] = run(cache[(cfg, deg)], smoother, ordering)
        with open(out_path, "w") as fh:
            json.dump(golden, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    O.set_threads(os.cpu_count() or 1)
    main()
