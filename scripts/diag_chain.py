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
    buf = np.zeros(6 * 5000 + 640 + 4096 + 64, np.uint64)
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
    ex = buf[6 * nseg: 6 * nseg + 640].reshape(2, 64, 5).astype(np.float64)
    hr = buf[6 * nseg + 640: 6 * nseg + 640 + 4096].reshape(2, 1024, 2).astype(np.float64)
    seglen = A.nrows // nseg
    cts = buf[6 * nseg + 640 + 4096: 6 * nseg + 640 + 4096 + 64].astype(np.float64)
    h0 = hr[1, 160, 0]
    if cts[0] > 0:
        c0 = cts[0]
        print("  seg8 row160 helper: pub %.2f us after start; per chunk [start, S wait done, y ready] cycles from first chunk:"
              % ((hr[1, 160, 1] - h0) / 1e3))
        print("   ", [(int(cts[i] - c0), int(cts[21 + i] - c0), int(cts[42 + i] - c0)) for i in range(21) if cts[i] > 0])
    Lf = F.export()[0]
    need = np.zeros(min(seglen, 1024), np.int64)  # seg-7 row each seg-8 row needs last
    for r in range(len(need)):
        v = 8 * seglen + r
        cols = Lf.col[Lf.rowptr[v]:Lf.rowptr[v + 1]]
        c7 = cols[(cols >= 7 * seglen) & (cols < 8 * seglen)] - 7 * seglen
        need[r] = c7.max() if c7.size else -1
    bs = 8 if max(F.stats()['max_row_L'], F.stats()['max_row_U']) <= 16 else 32
    def fin_time(si, row):  # end of the batch of segment 7+si that finalised `row`
        return ex[si, row // bs, 4]
    print(f"  bs {bs}; seg8 rows need seg7 row up to max {need.max()}")
    print("   row | s7 fin(need) | s8 h.start  h.pub | s8 fin | hop(pub - s7fin)  (us, rel. to s7 fin of row 0)")
    base = ex[0, 0, 4]
    hops = []
    for r in list(range(0, 40, 4)) + list(range(64, min(seglen, 1024), 96)):
        if r >= len(need) or need[r] < 0 or need[r] // bs >= 64 or r // bs >= 64:
            continue
        f7 = fin_time(0, need[r]); hs, hp = hr[1, r]; f8 = fin_time(1, r)
        hops.append(hp - f7)
        print(f"   {r:4d} | {(f7-base)/1e3:9.2f} | {(hs-base)/1e3:9.2f} {(hp-base)/1e3:9.2f} | {(f8-base)/1e3:8.2f} | {(hp-f7)/1e3:7.2f}")
    for k in list(range(0, 6)) + [nseg // 2, nseg // 2 + 1, nseg - 1]:
        print(f"   seg {k}: claim {claim[k]:.1f} fin_start {fs[k]:.1f} fin_end {fe[k]:.1f} hdone {hdone[k]:.1f} "
              f"spins {tr[k,4]:.0f} waits {tr[k,5]:.0f}")
    if os.environ.get("DIAG_BATCHES"):
        print("   b | s7 start hdr_ok end | s8 start hdr_ok end | s8 helper row 32b start / row 32b+31 pub")
        for b in range(min(20, seglen // bs)):
            r0, r1 = b * bs, b * bs + bs - 1
            f = lambda x: (x - base) / 1e3
            print(f"  {b:2d} | {f(ex[0,b,0]):7.2f} {f(ex[0,b,1]):7.2f} {f(ex[0,b,4]):7.2f} | {f(ex[1,b,0]):7.2f} {f(ex[1,b,1]):7.2f} {f(ex[1,b,4]):7.2f} |"
                  f" {f(hr[1,r0,0]):7.2f} {f(hr[1,r1,1]):7.2f}")
