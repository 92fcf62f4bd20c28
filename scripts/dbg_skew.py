# debug: skew sweeps vs oracle on a small p=1 factor; prints where results differ
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
h = int(sys.argv[1]) if len(sys.argv) > 1 else 5
spec = P.make_spec(geometry="square", rhs="one", degrees=(2, 1), h_exp=h)
A = P.build(spec).hlevels[0].A
n = A.nrows
Fg = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
print(Fg.stats())
Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE); Fo.n = n
L, U, _ = Fo.export()
r = np.random.default_rng(0).uniform(-1, 1, n)
eg = pmg.ilut_apply(Fg, r)
eo = Fo.apply(r)
# oracle L solve alone
import scipy.sparse as sp
Lm = sp.csr_matrix((L.val, L.col, L.rowptr), shape=(n, n))
y = np.zeros(n)
for i in range(n):
    s = 0.0
    for k in range(L.rowptr[i], L.rowptr[i+1]):
        s = s + L.val[k] * y[L.col[k]]
    y[i] = r[i] - s
bad = np.nonzero(eg != eo)[0]
print("mismatches", bad.size, "first", bad[:20], "seg", int(round(np.sqrt(n))))
if bad.size:
    S = int(round(np.sqrt(n)))
    print("first bad rows (seg, ix):", [(int(b)//S, int(b)%S) for b in bad[:10]])
    print("last bad:", [(int(b)//S, int(b)%S) for b in bad[-5:]])
    print(eg[bad[:5]], eo[bad[:5]])
    print("any nan", np.isnan(eg).sum())
