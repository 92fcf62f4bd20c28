"""Small driver for compute-sanitizer runs: config 1 (ILUT and GS solves, the
GPU ILUT factorization, BiCGSTAB) and one p=5 factor sweep at h=2^-5, through the C ABI.
Each engine is exercised: rotating-lane (default), skewed-warp (PMG_WAVE=0), chained
(PMG_WAVE=0 PMG_SKEW=0) and level-scheduled (PMG_FORCE_LEVELSCHED=1) -- chosen by the caller's env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1901_01685_b200 import pmg, problems as P

pb = P.build(1)
for sm in ("ilut", "gs"):
    H = pmg.build_hierarchy(pb, smoother=sm)
    u, rep = pmg.solve(H, pb.f, guess=pb.u0)
    print(sm, "cycles", rep.cycles, "converged", rep.converged, flush=True)
H = pmg.build_hierarchy(pb, smoother="ilut")
u, kr = pmg.bicgstab(H, pb.f, guess=pb.u0)
print("bicgstab", kr.iterations, kr.converged, flush=True)
A = P.build(P.make_spec("annulus", "one", (5, 1), 5)).plevels[0].A
F = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
e = pmg.ilut_apply(F, np.ones(A.nrows))
print("p5 factor", F.stats()["sweep"], float(np.abs(e).max()), flush=True)
