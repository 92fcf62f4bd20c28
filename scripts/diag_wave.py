"""Diagnostics: trace one rotating-lane L sweep (wave.cu) of a p-level ILUT factor and print the
lags between consecutive warp blocks (inside a CTA vs across CTAs) and the step rate.
usage: diag_wave.py h_exp degree"""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_01685_b200 import pmg, problems as P

h = int(sys.argv[1]) if len(sys.argv) > 1 else 9
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
L = pmg.lib()
L.pmg_debug_wave_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
pb = P.build(P.make_spec(geometry="annulus", rhs="one", degrees=(max(deg, 2), 1), h_exp=h))
A = pb.hlevels[0].A if deg == 1 else pb.plevels[0].A
n = A.nrows
F = pmg.ilut_factorize(A, 1e-12, 1.0, "none")
st = F.stats()
print({k: st[k] for k in ("sweep", "segment", "skew_D", "levels_L")})
r = np.random.default_rng(0).uniform(-1, 1, n)
for _ in range(3):
    pmg.ilut_apply(F, r)
L.pmg_debug_wave_trace(1, None, 0)
pmg.ilut_apply(F, r)
buf = (ctypes.c_ulonglong * (1 << 20))()
nb = L.pmg_debug_wave_trace(-1, buf, 1 << 20)
tr = np.array(buf[:4 * nb], dtype=np.int64).reshape(nb, 4)
t0 = tr[:, 0].min()
span = (tr[:, 2].max() - t0) / 1e3
seg = st["segment"]
lead = st["skew_D"][0]
print(f"blocks {nb} span {span:.1f} us")
task = tr[:, 3]
lag = np.diff(tr[:, 0]) / 1e3
same = task[1:] == task[:-1]
print(f"lag between consecutive blocks: same CTA {np.median(lag[same]) if same.any() else float('nan'):.2f} us, "
      f"across CTAs {np.median(lag[~same]) if (~same).any() else float('nan'):.2f} us  (lead {lead} steps)")
lag_end = np.diff(tr[:, 2]) / 1e3
print(f"lag between consecutive blocks at their last step: same CTA {np.median(lag_end[same]) if same.any() else float('nan'):.2f} us, "
      f"across CTAs {np.median(lag_end[~same]) if (~same).any() else float('nan'):.2f} us")
lag_mid = np.diff(tr[:, 1]) / 1e3
print(f"lag at step 192: same CTA {np.median(lag_mid[same]) if same.any() else float('nan'):.2f} us, "
      f"across CTAs {np.median(lag_mid[~same]) if (~same).any() else float('nan'):.2f} us")
ok = tr[:, 1] > 0
rate = (tr[ok, 2] - tr[ok, 1]) / 1e3  # us from step 192 to the end
print("median block duration us", np.median((tr[:, 2] - tr[:, 0]) / 1e3), "median us from step 192 to end", np.median(rate))
for b in range(0, nb, max(1, nb // 10)):
    print(f"blk {b} task {task[b]}: start {(tr[b,0]-t0)/1e3:9.2f} s192 {(tr[b,1]-t0)/1e3:9.2f} end {(tr[b,2]-t0)/1e3:9.2f} us")
