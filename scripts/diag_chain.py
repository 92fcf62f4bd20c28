"""Per-segment timing trace of the chained sweeps (diagnostics)."""
import ctypes, sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_01685_b200 import pmg, problems as P

L = pmg.lib()
L.pmg_debug_chain_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
h_exp = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s = P.make_spec('annulus', 'annulus', (p, 1), h_exp)
pb = P.build(s)
for lev, A in (('p', pb.plevels[0].A), ('p1', pb.plevels[1].A)):
    t = time.time(); F = pmg.ilut_factorize(A, 1e-12, 1.0, 'none'); tf = time.time() - t
    r = np.random.default_rng(0).uniform(-1, 1, A.nrows)
    e = pmg.ilut_apply(F, r)
    L.pmg_debug_chain_trace(1, None, 0)
    t = time.time(); e = pmg.ilut_apply(F, r); ta = time.time() - t
    buf = np.zeros(6 * 5000 + 64 * 5 + 1024, np.uint64)
    nseg = L.pmg_debug_chain_trace(-1, buf.ctypes.data_as(ctypes.c_void_p), buf.size)
    L.pmg_debug_chain_trace(0, None, 0)
    tr = buf[:6 * nseg].reshape(nseg, 6).astype(np.float64)
    t0 = tr[:, 0].min()
    claim, hdone, fs, fe = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3, (tr[:, 3] - t0) / 1e3
    print(f"[{lev}] n={A.nrows} nseg={nseg} factor {tf:.2f}s apply(L+U) wall {ta*1e3:.1f} ms stats {F.stats()}")
    print(f"  L sweep span {fe.max():.1f} us; per-seg fin duration median {np.median(fe-fs):.1f} us; "
          f"lag(fin_end) median {np.median(np.diff(fe)):.2f} us; fin_start lag median {np.median(np.diff(fs)):.2f} us")
    print(f"  helper spins median {np.median(tr[:,4]):.0f} fin batch waits median {np.median(tr[:,5]):.0f}; "
          f"helpers done - fin start median {np.median(hdone-fs):.1f} us")
    bt = buf[6 * nseg: 6 * nseg + 64 * 5].reshape(64, 5).astype(np.float64)
    hp = buf[6 * nseg + 64 * 5: 6 * nseg + 64 * 5 + 1024].astype(np.float64)
    seglen = A.nrows // nseg
    hp = (hp[:seglen] - t0) / 1e3
    print("   seg8 helper prefix ready (us) at rows 0,31,63,95,127,191,255,383,511:", [round(hp[i], 1) for i in (0, 31, 63, 95, 127, 191, 255, 383, 511) if i < seglen])
    print("   seg7 fin_end %.1f, seg8 claim %.1f fin_end %.1f" % (fe[7], claim[8], fe[8]))
    nb = int((bt[:, 0] > 0).sum())
    b0 = t0
    for b in range(min(nb, 6)):
        print(f"   seg8 batch {b}: start {(bt[b,0]-b0)/1e3:.2f} hdr {(bt[b,1]-bt[b,0])/1e3:.2f} cpwait {(bt[b,2]-bt[b,1])/1e3:.2f} "
              f"catchup {(bt[b,3]-bt[b,2])/1e3:.2f} steps {(bt[b,4]-bt[b,3])/1e3:.2f} us")
    for k in list(range(0, 6)) + [nseg // 2, nseg // 2 + 1, nseg - 1]:
        print(f"   seg {k}: claim {claim[k]:.1f} fin_start {fs[k]:.1f} fin_end {fe[k]:.1f} hdone {hdone[k]:.1f} "
              f"spins {tr[k,4]:.0f} waits {tr[k,5]:.0f}")
