"""Sweep-kernel experiment (diagnostics): per-class device times of one solve on a p-MG
hierarchy, under the PMG_* settings of the environment.  usage: wave_exp.py p h_exp [smoother]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1901_01685_b200 import pmg, problems as P

p, h = int(sys.argv[1]), int(sys.argv[2])
sm = sys.argv[3] if len(sys.argv) > 3 else "ilut"
pb = P.build(P.make_spec("annulus", "annulus", (p, 1), h))
H = pmg.build_hierarchy(pb, smoother=sm)
for _ in range(2):
    u, rep = pmg.solve(H, pb.f, guess=pb.u0)
H.kernel_times(enable=False)
t = []
for _ in range(3):
    u, rep = pmg.solve(H, pb.f, guess=pb.u0)
    t.append(rep.solve_seconds)
H.kernel_times(enable=True)
u, rep = pmg.solve(H, pb.f, guess=pb.u0)
kt = H.kernel_times()
H.kernel_times(enable=False)
c = rep.cycles
st = H.factors()[0].stats() if sm == "ilut" else {}
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("PMG_")}, "p": p, "h": h, "n": pb.n, "cycles": c,
       "ms_solve": 1e3 * min(t), "ms_per_sweep": {k: v / max(1, 2 * c) for k, v in kt["ms"].items() if k.endswith("_fine") and v},
       "coarse_ms_per_cycle": kt["ms"]["coarse"] / c, "sweep": st.get("sweep"), "lead": st.get("skew_D")}
print(json.dumps(out), flush=True)
