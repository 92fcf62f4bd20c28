# debug: skewed-warp sweeps vs the oracle on the factor of a p-level (p = argv[2]) at h = 2^-argv[1]
import sys, time, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
h = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1
geo = sys.argv[3] if len(sys.argv) > 3 else "square"
spec = P.make_spec(geometry=geo, rhs="one", degrees=(max(p, 2), 1), h_exp=h)
pb = P.build(spec)
A = pb.hlevels[0].A if p == 1 else pb.plevels[0].A
n = A.nrows
Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
st = Fg.stats()
print({k: st[k] for k in ("max_row_L", "max_row_U", "sweep", "segment", "skew_D")})
t0 = time.time()
Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE)
r = np.random.default_rng(0).uniform(-1, 1, n)
eg = pmg.ilut_apply(Fg, r)
eo = Fo.apply(r)
bad = np.nonzero(eg.view(np.uint64) != eo.view(np.uint64))[0]
S = st["segment"]
print(f"p={p} h=2^-{h} n={n} mismatches {bad.size}", [(int(b) // S, int(b) % S) for b in bad[:6]] if bad.size else "")
