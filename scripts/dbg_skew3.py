import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
mode = sys.argv[1]
pb = P.build(1)
A = pb.plevels[1].A
if mode == "p2first":
    F2 = pmg.ilut_factorize(pb.plevels[0].A, 1e-12, 1.0, "none")
if mode == "apply2":
    F2 = pmg.ilut_factorize(pb.plevels[0].A, 1e-12, 1.0, "none")
    pmg.ilut_apply(F2, np.ones(pb.plevels[0].A.nrows))
Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
r = np.random.default_rng(1).uniform(-1, 1, A.nrows)
for i in range(3):
    e = pmg.ilut_apply(Fg, r)
print(mode, "ok", flush=True)
