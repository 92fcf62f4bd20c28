# F3: spectral radii of the GPU p-multigrid cycle for the paper's benchmarks (SPEC.md:443-458,
# PAPER Tables 2-3 for comparison; our Nitsche constant and problems follow DESIGN.md §0)
import json, sys, time
sys.path.insert(0, '.')
from paper_1901_01685_b200 import analysis, pmg, problems as P
rows = []
for bench, p, h, sm in [(1, 2, 4, "gs"), (1, 2, 4, "ilut"), (1, 3, 4, "ilut"), (1, 4, 5, "ilut"), (2, 4, 5, "ilut"),
                        (1, 4, 5, "gs")]:
    pb = P.build(P.benchmark_spec(bench, p, h))
    if pb.n > 2500:
        continue
    H = pmg.build_hierarchy(pb, smoother=sm)
    t0 = time.perf_counter()
    M = analysis.iteration_matrix(H, workers=8)
    s = analysis.spectral_radius(M)
    rows.append({"benchmark": bench, "p": p, "h_exp": h, "smoother": sm, "n_dof": pb.n, "rho": s.rho,
                 "seconds": round(time.perf_counter() - t0, 2)})
    print(json.dumps(rows[-1]), flush=True)
