# diagnostics: time the skewed-warp vs chained sweeps on a p=1 factor, trace one skew sweep
import ctypes, sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1901_01685_b200 import pmg, problems as P
h = int(sys.argv[1]) if len(sys.argv) > 1 else 10
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L = pmg.lib()
L.pmg_debug_skew_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
spec = P.make_spec(geometry="annulus", rhs="one", degrees=(max(deg, 2), 1), h_exp=h)
pb = P.build(spec)
A = pb.hlevels[0].A if deg == 1 else pb.plevels[0].A
n = A.nrows
F = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
print(F.stats())
r = np.random.default_rng(0).uniform(-1, 1, n)
for _ in range(3): pmg.ilut_apply(F, r)
t0 = time.perf_counter(); K = 10
for _ in range(K): pmg.ilut_apply(F, r)
print("ilut_apply (L+U sweeps + copies) ms", (time.perf_counter() - t0) / K * 1e3)
L.pmg_debug_skew_trace(1, None, 0)
pmg.ilut_apply(F, r)
buf = (ctypes.c_ulonglong * 65536)()
nb = L.pmg_debug_skew_trace(-1, buf, 65536)
tr = np.array(buf[:8 * nb], dtype=np.int64).reshape(nb, 8)
t0 = tr[:, 0].min()
print("blocks", nb, "sweep span us", (tr[:, 1].max() - t0) / 1e3)
for b in range(0, nb, max(1, nb // 12)):
    if b + 1 < nb and tr[b, 4]:
        print(f"  hop at row 200: store->bridge sees {(tr[b,5]-tr[b,4])/1e3:.2f} us, ->published {(tr[b,6]-tr[b,4])/1e3:.2f} us, ->next block at row 154 {(tr[b,7]-tr[b,4])/1e3:.2f} us")
    print(f"blk {b}: claim {(tr[b,0]-t0)/1e3:9.1f} us end {(tr[b,1]-t0)/1e3:9.1f} us dur {(tr[b,1]-tr[b,0])/1e3:8.1f} halo wait {tr[b,2]/1965:.1f} us bridge polls {tr[b,3]}")

import os
if int(os.environ.get("PMG_SKEW_DBG", "0")) & 16:
    a, b = int(tr[0, 2]), int(tr[0, 3])
    print("block 0 cycles: issue+group wait", a >> 32, "rhs wait", a & 0xffffffff, "halo+sync", b >> 32, "compute+store", b & 0xffffffff)
