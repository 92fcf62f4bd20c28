# debug: Gauss-Seidel sweep (skewed-warp kernel) vs the oracle on A_p at h = 2^-argv[1], p = argv[2]
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
h, p = int(sys.argv[1]), int(sys.argv[2])
pb = P.build(P.make_spec(geometry="annulus", rhs="one", degrees=(max(p, 2), 1), h_exp=h))
A = pb.hlevels[0].A if p == 1 else pb.plevels[0].A
rng = np.random.default_rng(2)
u = rng.uniform(-1, 1, A.nrows); f = rng.uniform(-1, 1, A.nrows)
g = pmg.gauss_seidel_sweep(A, u, f); o = O.gauss_seidel_sweep(A, u, f)
print(f"GS p={p} h=2^-{h} n={A.nrows} mismatches", int(np.sum(g.view(np.uint64) != o.view(np.uint64))))
