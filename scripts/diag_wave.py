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
tr = np.array(buf[:8 * nb], dtype=np.int64).reshape(nb, 8)
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
# crossing anatomy (first block of a CTA b, its producer b-1 in another CTA): the producer passes
# step 32 (row 0 final at step 31) -> the bridge sees row 0's first values -> the bridge publishes
# enough virtual progress for step 0 (needs row 14: 13 steps more) -> the sweep warp starts
cross = np.where(~same)[0] + 1
cross = cross[(tr[cross, 4] > 0) & (tr[cross, 5] > 0) & (tr[cross - 1, 6] > 0)]
if len(cross):
    seen = (tr[cross, 4] - tr[cross - 1, 6]) / 1e3
    pubd = (tr[cross, 5] - tr[cross - 1, 6]) / 1e3
    start = (tr[cross, 0] - tr[cross - 1, 6]) / 1e3
    dur = (tr[cross - 1, 2] - tr[cross, 4]) / 1e3  # the nearest row streams in until its producer ends
    print(f"crossing anatomy (medians over {len(cross)} crossings, us after the producer's step 32): bridge sees "
          f"row 0 {np.median(seen):.2f}, bridge publishes the start {np.median(pubd):.2f}, sweep warp starts "
          f"{np.median(start):.2f}; bridge pass {1e3 * np.median(dur / np.maximum(tr[cross, 7], 1)):.0f} ns "
          f"({np.median(tr[cross, 7]):.0f} passes while the nearest row streams in)")
ok = tr[:, 1] > 0
rate = (tr[ok, 2] - tr[ok, 1]) / 1e3  # us from step 192 to the end
print("median block duration us", np.median((tr[:, 2] - tr[:, 0]) / 1e3), "median us from step 192 to end", np.median(rate))
for b in range(0, nb, max(1, nb // 10)):
    print(f"blk {b} task {task[b]}: start {(tr[b,0]-t0)/1e3:9.2f} s192 {(tr[b,1]-t0)/1e3:9.2f} end {(tr[b,2]-t0)/1e3:9.2f} us")
