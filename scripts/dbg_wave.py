"""Debug: where a wave ilut_apply differs from the oracle (segment, row) for a p=1 factor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from oracle import oracle as O
from paper_1901_01685_b200 import pmg, problems as P
h = int(sys.argv[1]) if len(sys.argv) > 1 else 4
geo = sys.argv[2] if len(sys.argv) > 2 else "square"
deg = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pb = P.build(P.make_spec(geometry=geo, rhs="one", degrees=(max(deg, 2), 1), h_exp=h))
A = pb.hlevels[0].A if deg == 1 else pb.plevels[0].A
F = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
st = F.stats()
Fo = O.ilut_factorize(A, 1e-12, 1.0, O.ORDER_NONE)
r = np.random.default_rng(0).uniform(-1, 1, A.nrows)
e, eo = pmg.ilut_apply(F, r), Fo.apply(r)
bad = np.nonzero(e.view(np.uint64) != eo.view(np.uint64))[0]
seg = st["segment"]
print(os.environ.get("PMG_CUDA_LIB"), st["sweep"], "n", A.nrows, "seg", seg, "bad", bad.size)
L, U, perm = Fo.export()
n = A.nrows
Ls = sp.csr_matrix((L.val, L.col, L.rowptr), shape=(n, n)) + sp.identity(n)
Us = sp.csr_matrix((U.val, U.col, U.rowptr), shape=(n, n))
y_o = sp.linalg.spsolve_triangular(Ls.tocsr(), r, lower=True)
y_g = Us @ e
dy = np.abs(y_g - y_o) / (np.abs(y_o) + 1e-30)
print("L part max rel diff (y = U e vs L^-1 r):", dy.max(), "rows with >1e-8:", np.nonzero(dy > 1e-8)[0][:10])
segs = sorted(set(int(b) // seg for b in bad))
print("bad segments (natural):", segs)
import ctypes
Lb = pmg.lib()
Lb.pmg_debug_wave_dump.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
Lb.pmg_debug_wave_dump(1, None, 0)
pmg.ilut_apply(F, r)
yg = np.empty(n); xg = np.empty(n)
Lb.pmg_debug_wave_dump(2, yg.ctypes.data, n)
Lb.pmg_debug_wave_dump(3, xg.ctypes.data, n)
dyy = np.abs(yg - y_o) / (np.abs(y_o) + 1e-30)
print("GPU L output y vs oracle L^-1 r: rows > 1e-12:", np.nonzero(dyy > 1e-12)[0][:12])
# U sweep in v-order: x[v] for v = n-1-row, input y[n-1-v]
x_o = sp.linalg.spsolve_triangular(Us.tocsr(), yg, lower=False)
xv = xg[::-1]
dxx = np.abs(xv - x_o) / (np.abs(x_o) + 1e-30)
print("GPU U output (from the GPU's own y) vs exact: rows > 1e-10:", np.nonzero(dxx > 1e-10)[0][:12])
