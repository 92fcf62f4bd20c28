import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
pb = P.build(1)
for lev in pb.plevels:
    A = lev.A
    Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
    print(A.nrows, Fg.stats(), flush=True)
    r = np.random.default_rng(1).uniform(-1, 1, A.nrows)
    e = pmg.ilut_apply(Fg, r)
    print("ok", flush=True)
