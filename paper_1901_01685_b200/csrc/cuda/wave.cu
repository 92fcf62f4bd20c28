// Rotating-lane wavefront sweeps: L and U solves of the ILUT factors and the lexicographic
// Gauss-Seidel sweep on tensor-grid orderings, bitwise equal to the oracle (SPEC.md:233-241,
// :260-264).
//
// Rows are visited in v-order (L, GS: ascending; U: descending) and cut into segments of one
// grid row.  A row's terms (ascending v-column, the oracle's summation order) are cut from the
// end into chunks: chunk 0 (the last C terms; for U and GS the last C-1, the first slot then
// carries 1/diagonal) and chunks 1, 2, ... of C terms.  NR lanes serve a segment and a warp
// serves SPW = 32/NR consecutive segments (a "block"); the segments of a block are skewed by
// D_b steps.  Lane rl of segment k owns the rows ix == rl (mod NR): it starts row ix at step
// ix + D_b k (chunk P = NR-1), adds one chunk per step, and finalises the row at step
// ix + P + D_b k (chunk 0).  The partial sum never leaves its lane, so a step's only
// cross-lane operation is ONE shuffle broadcasting the value finalised at the previous step.
// The recurrence per step is shfl -> DMUL -> DADD -> DADD (-> DMUL), about 60 cycles.
//
// Everything else is off that chain:
//   * a chunk's values are loaded from shared-memory rings one step ahead (the plan guarantees
//     they were final two steps before use), except a chunk's last term when it is the value
//     finalised at the previous step: the items address it through the XB cell and the lane
//     takes the broadcast instead;
//   * items (4 coefficients + 4 byte offsets = 48 B per lane and step) are fetched two steps
//     ahead from a ring that bulk copies (cp.async.bulk + mbarrier) fill 32 steps at a time;
//   * right-hand sides come from a ring that a stager warp fills.
// A CTA runs W consecutive blocks in W sweep warps; a warp waits for its predecessor through
// a progress counter in shared memory (before step t: prog(b-1) >= t + L_b, L_b from the plan,
// which makes the chain transitive over every block a term reaches).  Values of segments
// before the CTA come from global memory: a bridge warp polls them (NaN-sentinel protocol),
// copies them into halo rings and publishes a virtual progress of the previous block.
// Producers never overwrite ring cells a consumer may still read (back-pressure per group).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "wave.cuh"

namespace pmg {

namespace {

#ifndef PMG_WAVE_ST
#define PMG_WAVE_ST 0
#endif
#ifndef PMG_WAVE_BRIDGE_REL
#define PMG_WAVE_BRIDGE_REL 1
#endif
#ifndef PMG_WAVE_G
#define PMG_WAVE_G 32
#endif
#ifndef PMG_WAVE_WMAX
#define PMG_WAVE_WMAX 2
#endif
constexpr int G = PMG_WAVE_G;   // steps per bulk copy = unroll of the step loop
constexpr int NG = 2;           // item groups in flight
constexpr int PF = G * NG;      // item ring steps
constexpr int NRH = 4;          // right-hand-side ring groups
constexpr int STEP_BYTES = 3 * 32 * 16;
constexpr int MAXD = 8;         // segments back a term may reach
constexpr int EMAX = 8;         // blocks back a term may reach
constexpr int WMAX = PMG_WAVE_WMAX;  // sweep warps per CTA
#ifndef PMG_WAVE_CHK
#define PMG_WAVE_CHK 2
#endif
// steps per progress test / publication: a test is a branch, which splits the unrolled step
// sequence into basic blocks the scheduler cannot overlap; testing every CHK steps (for the
// needs of all CHK) costs at most CHK-1 steps of extra lag per warp hand-off
constexpr int CHK = PMG_WAVE_CHK;
static_assert(G % CHK == 0, "CHK divides the group");
constexpr int INF = INT_MAX / 2;
#ifndef PMG_WAVE_BRIDGE_AHEAD
#define PMG_WAVE_BRIDGE_AHEAD 64
#endif
constexpr int kBridgeAhead = PMG_WAVE_BRIDGE_AHEAD;  // 0: poll every halo row in every iteration
constexpr unsigned FULL = 0xffffffffu;

struct Layout {
    int item, rhs, su, ring, xb, bar, rfull, rempty, prog, rdp, vprog, task, total;
    int nrings;
};

// byte offsets of the dynamic shared memory regions
Layout layout(int W, int SPW, int DM, int RY, bool gs) {
    Layout L{};
    int o = 0;
    L.item = o;
    o += W * PF * STEP_BYTES;
    L.rhs = o;
    o += W * NRH * G * SPW * 8;
    L.su = o;
    if (gs) o += W * NRH * G * SPW * 8;
    L.nrings = DM + W * SPW;
    L.ring = o;
    o += L.nrings * (RY + 1) * 8;
    L.xb = o;
    o += 8;
    o = (o + 15) & ~15;
    L.bar = o;
    o += W * NG * 8;
    L.rfull = o;
    o += W * NRH * 8;
    L.rempty = o;
    o += W * NRH * 8;
    L.prog = o;
    o += W * 4;
    L.rdp = o;
    o += W * 4;
    L.vprog = o;
    o += 4;
    L.task = o;
    o += 4;
    L.total = (o + 127) & ~127;
    return L;
}

struct WaveArgs {
    const int32_t* starts;  // [nseg+1] first v-row of every segment (grid row)
    const uint4* item;
    const double* rhs;
    const double* su;
    double* out;
    const int32_t* Db;
    const int32_t* Lb;
    const int32_t* bp;
    const int32_t* hoff;
    const int32_t* hrb;
    const int32_t* hsl;
    const int64_t* off;
    unsigned sbase;  // shared-window address of the dynamic shared memory the items were built for
    int32_t n, seg, nseg, nblk, ntask, W, dm, ry;
    int32_t slack;   // extra steps of lead over the plan's L_b (see wave_sweep)
    unsigned long long* trace;  // diagnostics (null: off): 8 per block [start, step 192, end, task, bridge: first value
                                // of the nearest row seen, start published, (sweep) step 32, bridge passes while that row streams in]
    Layout lay;
    int* ticket;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_u128(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int ld_vol_s(unsigned a) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
// progress reads are acquire loads: on shared memory this is a plain LDS, but the compiler may
// not move the ring loads that follow it above it (a relaxed read lets ptxas hoist them over the
// spin loop, reading values before their producer published them)
__device__ __forceinline__ int ld_acq_s(unsigned a) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_s(unsigned a, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_vol_s(unsigned a, int v) {
    asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// spin (warp-uniform) until the shared counter at addr reaches need; pv: last value seen
__device__ __forceinline__ int wait_ge(unsigned addr, int pv, int need) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "L:\n\tsetp.ge.s32 p, %0, %2;\n\t@p bra.uni D;\n\t"
        "ld.acquire.cta.shared.b32 %0, [%1];\n\tbra.uni L;\n"
        "D:\n\t}"
        : "+r"(pv)
        : "r"(addr), "r"(need)
        : "memory");
    return pv;
}
__device__ __forceinline__ void bar_init(unsigned b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(b),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ double u2d(unsigned lo, unsigned hi) { return __hiloint2double(int(hi), int(lo)); }

struct Step {  // a lane's item of one step
    double w[4];
    unsigned o[4];
};
__device__ __forceinline__ void fetch_item(unsigned a, Step& s) {
    const uint4 c0 = lds_u128(a), c1 = lds_u128(a + 512), c2 = lds_u128(a + 1024);
    s.w[0] = u2d(c0.x, c0.y);
    s.w[1] = u2d(c0.z, c0.w);
    s.w[2] = u2d(c1.x, c1.y);
    s.w[3] = u2d(c1.z, c1.w);
    s.o[0] = c2.x;
    s.o[1] = c2.y;
    s.o[2] = c2.z;
    s.o[3] = c2.w;
}

template <int K, int NR, int C>
__global__ void __launch_bounds__(32 * (WMAX + 2)) k_wave(WaveArgs a) {
    constexpr int SPW = 32 / NR, P = NR - 1;
    constexpr int DS = 4 - C;  // first used slot; U / GS chunk 0: 1/diagonal there
    extern __shared__ __align__(128) unsigned char wave_smem[];
    const unsigned sb = smem_u32(wave_smem);
    if (sb != a.sbase) __trap();  // the items hold absolute shared-memory addresses
    const Layout& ly = a.lay;
    const int W = a.W, DM = a.dm, RY = a.ry, RYS = a.ry + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = a.n;
    const int32_t* starts = a.starts;
    const unsigned s_prog = sb + ly.prog, s_vprog = sb + ly.vprog;
    int* task_p = reinterpret_cast<int*>(wave_smem + ly.task);
    double* rings = reinterpret_cast<double*>(wave_smem + ly.ring);

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            *task_p = atomicAdd(a.ticket, 1);
            for (int w = 0; w < W; ++w) {
                for (int q = 0; q < NG; ++q) bar_init(sb + ly.bar + (w * NG + q) * 8, 1);
                for (int q = 0; q < NRH; ++q) {
                    bar_init(sb + ly.rfull + (w * NRH + q) * 8, 1);
                    bar_init(sb + ly.rempty + (w * NRH + q) * 8, 1);
                }
                st_vol_s(s_prog + 4 * w, 0);
                st_vol_s(sb + ly.rdp + 4 * w, 0);
            }
            st_vol_s(s_vprog, -INF);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int q = threadIdx.x; q < ly.nrings * RYS + 1; q += blockDim.x) rings[q] = 0.0;
        __syncthreads();
        const int task = *task_p;
        if (task >= a.ntask) break;
        const int b0 = task * W, g0 = b0 * SPW;

        if (warp == W) {
            // ------------------------------------------------------------ stager
            // right-hand sides (and GS upper sums) of the finalised rows, group by group
            int nq[WMAX], Dw[WMAX];
            int maxq = 0;
            for (int w = 0; w < W; ++w) {
                const int b = b0 + w;
                nq[w] = b < a.nblk ? int((a.off[b + 1] - a.off[b]) / G) : 0;
                Dw[w] = b < a.nblk ? a.Db[b] : 0;
                maxq = max(maxq, nq[w]);
            }
            for (int q = 0; q < maxq; ++q) {
                const int slot = q % NRH;
                for (int w = 0; w < W; ++w) {
                    if (q >= nq[w]) continue;
                    if (q >= NRH) bar_wait(sb + ly.rempty + (w * NRH + slot) * 8, ((q / NRH) - 1) & 1);
                    constexpr int PER = (G * SPW + 31) / 32;
                    double v[PER], s2[PER];
#pragma unroll
                    for (int i = 0; i < PER; ++i) {
                        const int e = i * 32 + lane;
                        const int st = q * G + e / SPW, kk = e % SPW;
                        const int gg = (b0 + w) * SPW + kk, ix = st - P - Dw[w] * kk;
                        const bool real = e < G * SPW && gg < a.nseg;
                        const int s0 = real ? starts[gg] : 0, s1 = real ? starts[gg + 1] : 0;
                        const int64_t vv = int64_t(s0) + ix;
                        const bool in = real && ix >= 0 && ix < s1 - s0;
                        v[i] = in ? a.rhs[K == kSkewU ? int64_t(n) - 1 - vv : vv] : 0.0;
                        if (K == kSkewGS) s2[i] = in ? a.su[vv] : 0.0;
                    }
#pragma unroll
                    for (int i = 0; i < PER; ++i) {
                        const int e = i * 32 + lane;
                        if (e < G * SPW) {
                            const int idx = ((w * NRH + slot) * G + e / SPW) * SPW + e % SPW;
                            reinterpret_cast<double*>(wave_smem + ly.rhs)[idx] = v[i];
                            if (K == kSkewGS) reinterpret_cast<double*>(wave_smem + ly.su)[idx] = s2[i];
                        }
                    }
                    __syncwarp();
                    if (lane == 0) bar_arrive(sb + ly.rfull + (w * NRH + slot) * 8);
                }
            }
            continue;
        }
        if (warp == W + 1) {
            // ------------------------------------------------------------ bridge
            // halo segment g0-1-d (d < DM) -> ring d' = DM-1-d; vprog = min_d (f[d] + hoff[d])
            int f[MAXD], ho[MAXD], rows[MAXD], hr[WMAX][MAXD], sl[MAXD], hb[MAXD];
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
                const int gh = g0 - 1 - d;
                ho[d] = d < DM ? a.hoff[task * MAXD + d] : INT_MIN;
                sl[d] = d < DM ? a.hsl[task * MAXD + d] : 0;  // ring slot of row j: (j + sl) mod RY
                hb[d] = gh >= 0 ? starts[gh] : 0;
                rows[d] = gh >= 0 ? starts[gh + 1] - hb[d] : 0;
                f[d] = (d < DM && gh >= 0 && ho[d] > INT_MIN / 2) ? 0 : rows[d];
                for (int w = 0; w < WMAX; ++w) hr[w][d] = (w < W && d < DM) ? a.hrb[(task * W + w) * MAXD + d] : INF;
            }
            int pub = -INF;
            int npass = 0;
            for (;;) {
                if (f[0] > 0 && f[0] < rows[0]) ++npass;  // passes while the nearest row streams in (trace)
                int pr[WMAX];
                for (int w = 0; w < WMAX; ++w)  // a warp that finished its steps reads no ring cell
                    pr[w] = w < W ? max(ld_acq_s(s_prog + 4 * w), ld_acq_s(sb + ly.rdp + 4 * w)) : INF;
                double v[MAXD];
                // the nearest halo row is the one the sweep waits for; an older row is polled only
                // while its virtual progress is less than kBridgeAhead steps ahead of the nearest
                // one's (always at the start of a block, then once per ~32 rows): a short loop keeps
                // the hand-over latency low
                const bool all = f[0] >= rows[0];
                const int near_vp = all ? 0 : f[0] + ho[0] + kBridgeAhead;
                bool polled[MAXD];
#pragma unroll
                for (int d = 0; d < MAXD; ++d) {
                    v[d] = sentinel();
                    polled[d] = f[d] < rows[d] && (d == 0 || all || f[d] + ho[d] < near_vp);
                    int lim = INF;
                    for (int w = 0; w < WMAX; ++w) lim = min(lim, pr[w] >= INF ? INF : pr[w] + hr[w][d]);
                    const int j = f[d] + lane;
                    if (polled[d] && j < rows[d] && j < lim)
                        v[d] = ld_relaxed_nb(a.out + hb[d] + j);
                }
                int vp = INF;
#pragma unroll
                for (int d = 0; d < MAXD; ++d) {
                    if (f[d] < rows[d] && !polled[d]) vp = min(vp, f[d] + ho[d]);
                    if (polled[d]) {
                        const unsigned ok = __ballot_sync(FULL, !is_sentinel(v[d]));
                        const int cnt = ok == FULL ? 32 : __ffs(~ok) - 1;
                        if (lane < cnt) rings[(DM - 1 - d) * RYS + ((f[d] + lane + sl[d]) & (RY - 1))] = v[d];
                        f[d] += cnt;
                        if (f[d] < rows[d]) vp = min(vp, f[d] + ho[d]);
                    }
                }
                if (a.trace && lane == 0 && b0 < a.nblk) {
                    if (f[0] > 0 && a.trace[b0 * 8 + 4] == 0) a.trace[b0 * 8 + 4] = gtimer();
                    if (vp >= a.Lb[b0] + a.slack - 1 && a.trace[b0 * 8 + 5] == 0) a.trace[b0 * 8 + 5] = gtimer();
                }
                __syncwarp();
                if (vp > pub) {
                    // PMG_WAVE_BRIDGE_REL=0 publishes with a plain volatile store (as the sweep warps
                    // publish their progress) and saves the MEMBAR.ALL.CTA of the release: measured,
                    // no effect on the hand-over (142.0 vs 142.2 ms per solve), so the release stays
#if PMG_WAVE_BRIDGE_REL
                    if (lane == 0) st_rel_s(s_vprog, vp);
#else
                    if (lane == 0) st_vol_s(s_vprog, vp);
#endif
                    pub = vp;
                }
                if (vp >= INF) break;
            }
            if (a.trace && lane == 0 && b0 < a.nblk) a.trace[b0 * 8 + 7] = npass;
            continue;
        }

        // ---------------------------------------------------------------- sweep warp
        const int b = b0 + warp;
        const unsigned s_me = s_prog + 4 * warp;
        if (b >= a.nblk) {
            st_vol_s(sb + ly.rdp + 4 * warp, INF);
            st_vol_s(s_me, INF);
            continue;
        }
        const int D = a.Db[b], Lw = a.Lb[b] + a.slack;
        const int NS = int(a.off[b + 1] - a.off[b]);
        const int nq = NS / G;
        const int k = lane / NR, rl = lane % NR, gbase = k * NR;
        const int g = b * SPW + k;
        const int64_t lo = g < a.nseg ? starts[g] : 0;
        const int rows = g < a.nseg ? starts[g + 1] - starts[g] : 0;
        const int phase = (P + D * k + rl) % NR;         // lane finalises at step t <=> t % NR == phase
        const int c0 = ((-1 - P - D * k) % NR + NR) % NR;  // finaliser of step t-1: gbase + ((t + c0) % NR)
        const unsigned pred = warp == 0 ? s_vprog : s_prog + 4 * (warp - 1);
        const unsigned XB = sb + unsigned(ly.xb);
        const int myring = (DM + warp * SPW + k) * RYS;  // own ring (element index)
        const unsigned ibase = sb + ly.item + warp * PF * STEP_BYTES + lane * 16;
        const unsigned rbase = sb + ly.rhs + warp * NRH * G * SPW * 8 + k * 8;
        const unsigned sbase2 = sb + ly.su + warp * NRH * G * SPW * 8 + k * 8;
        const unsigned char* bsrc = reinterpret_cast<const unsigned char*>(a.item) + a.off[b] * STEP_BYTES;
        const int* bpp = a.bp + b * W;
        auto refill = [&](int q) {
            if (lane == 0 && q < nq) {
                const int slot = q % NG;
                bulk_load(sb + ly.item + (warp * PF + slot * G) * STEP_BYTES, bsrc + int64_t(q) * G * STEP_BYTES,
                          G * STEP_BYTES, sb + ly.bar + (warp * NG + slot) * 8);
            }
        };
        auto group_wait = [&](int q) {
            if (q < nq) {
                bar_wait(sb + ly.bar + (warp * NG + q % NG) * 8, (q / NG) & 1);
                bar_wait(sb + ly.rfull + (warp * NRH + q % NRH) * 8, (q / NRH) & 1);
            }
        };
        auto backpressure = [&](int q) {  // ring cells of rows finalised before (q+1)G - RY may be reused
            for (int j = 1; warp + j < W; ++j) {
                const int need = (q + 1) * G + bpp[j];
                if (need > -INF / 2)
                    while (max(ld_acq_s(s_prog + 4 * (warp + j)), ld_acq_s(sb + ly.rdp + 4 * (warp + j))) < need) {
                    }
            }
        };
        for (int q = 0; q < NG; ++q) refill(q);
        group_wait(0);
        int pv = ld_acq_s(pred);
        while (pv < Lw - 1) pv = ld_acq_s(pred);  // the prologue loads below belong to step -1
        // software pipeline: items of step t+1 (cur) and t+2 (nxt); for step t, the products of
        // its first C-1 terms (pc, computed at step t-1 from values loaded at step t-1), its last
        // term's value / coefficient / address (y3, w3, o3) and 1/diagonal (wd)
        Step cur, nxt;
        double pc[3], y3, w3, wd;
        unsigned o3;
        {
            Step now;
            fetch_item(ibase, now);
            fetch_item(ibase + STEP_BYTES, cur);
#pragma unroll
            for (int q = DS; q < 3; ++q) pc[q] = now.w[q] * lds_f64(now.o[q]);
            y3 = lds_f64(now.o[3]);
            w3 = now.w[3];
            o3 = now.o[3];
            wd = now.w[DS];
        }
        double rh = lds_f64(rbase), sr = 0.0;
        if (K == kSkewGS) sr = lds_f64(sbase2);
        double acc = 0.0, x = 0.0;
        double* outp = a.out + lo;
        backpressure(0);
        if (a.trace && lane == 0) {
            a.trace[b * 8 + 0] = gtimer();
            a.trace[b * 8 + 3] = task;
        }
        for (int tb = 0; tb < NS; tb += G) {
            const int qg = tb / G;
            const int rgb = myring + (tb & (RY - 1));  // ring cell of step tb (RY is a multiple of G)
            if (tb == 192 && a.trace && lane == 0) a.trace[b * 8 + 1] = gtimer();
            if (tb == 32 && a.trace && lane == 0) a.trace[b * 8 + 6] = gtimer();  // row 0 is final at step 31
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int t = tb + u;
                // the broadcast first: it heads the step's critical chain and touches no shared
                // memory, so the progress test (a branch) need not come before it
                const double xb = __shfl_sync(FULL, x, gbase + ((u + c0) & (NR - 1)));
                // the predecessor's progress, read a step ago (it only grows, so a stale value is
                // a valid lower bound) and re-read now, off the chain; acquire loads keep the ring
                // loads below after the test
                if (u % CHK == 0) {  // one test covers the loads of steps t .. t+CHK-1
                    pv = wait_ge(pred, pv, t + CHK - 1 + Lw);
                    pv = ld_acq_s(pred);
                }
                if (u == G - 2) group_wait(qg + 1);
                // loads for step t+1 (values, items of t+2, right-hand side); their products are
                // formed at the end of this step, so they are issued early and their latency is
                // hidden behind this step's chain
                double yn[4];
#pragma unroll
                for (int q = DS; q < 4; ++q) yn[q] = lds_f64(cur.o[q]);
                fetch_item(ibase + ((t + 2) % PF) * STEP_BYTES, nxt);
                const int rs = ((t + 1) % (NRH * G)) * SPW * 8;
                const double rhn = lds_f64(rbase + rs);
                double srn = 0.0;
                if (K == kSkewGS) srn = lds_f64(sbase2 + rs);
                // step t: its chunk in the oracle's order, the last term from the broadcast if it
                // is the value finalised at the previous step
                double r = acc;
#pragma unroll
                for (int q = DS; q < 3; ++q) r = r + pc[q];
                r = r + w3 * (o3 == XB ? xb : y3);
                const bool stage0 = (u & (NR - 1)) == phase;
                const int ix = t - P - D * k;
                x = K == kSkewL ? rh - r : K == kSkewU ? (rh - r) * wd : ((rh - r) - sr) * wd;
                // ring cells are indexed by the step that finalised the value (cells of rows
                // outside the segment are never read); the output only for real rows
                if (stage0) rings[rgb + u] = x;
                // the value other CTAs poll for: PMG_WAVE_ST selects the store flavour (0 plain,
                // 1 st.global.cg, 2 st.relaxed.gpu)
#if PMG_WAVE_ST == 1
                if (stage0 && ix >= 0 && ix < rows) __stcg(outp + ix, x);
#elif PMG_WAVE_ST == 2
                if (stage0 && ix >= 0 && ix < rows) st_relaxed_if(outp + ix, x, true);
#else
                if (stage0 && ix >= 0 && ix < rows) outp[ix] = x;
#endif
                acc = stage0 ? 0.0 : r;
                if (u % CHK == CHK - 1) st_vol_s(s_me, t + 1);
                // step t+1's products and last term
#pragma unroll
                for (int q = DS; q < 3; ++q) pc[q] = cur.w[q] * yn[q];
                y3 = yn[3];
                w3 = cur.w[3];
                o3 = cur.o[3];
                wd = cur.w[DS];
                cur = nxt;
                rh = rhn;
                sr = srn;
            }
            __syncwarp();
            if (lane == 0) bar_arrive(sb + ly.rempty + (warp * NRH + qg % NRH) * 8);
            refill(qg + NG);
            backpressure(qg + 1);
        }
        if (a.trace && lane == 0) a.trace[b * 8 + 2] = gtimer();
        // finished: no ring cell is read any more; "done" is published once the predecessor is
        // done (keeps the progress chain valid)
        st_vol_s(sb + ly.rdp + 4 * warp, INF);
        while (ld_acq_s(pred) < INF) {
        }
        st_vol_s(s_me, INF);
    }
}

// The terms of row v (v-order) of S, ascending v-column.
template <int K>
struct RowView {
    const Sell& S;
    int v, n, len;
    int64_t base;
    int li;
    __device__ RowView(const Sell& s, int v_, const int32_t* nlow)
        : S(s), v(v_), n(s.n), len(K == kSkewGS ? nlow[v_] : s.len[v_]), base(s.off[v_ >> 5]), li(v_ & 31) {}
    __device__ int col(int k) const {
        const int c = S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)];
        return K == kSkewU ? n - 1 - c : c;
    }
    __device__ double val(int k) const { return S.val[base + (k >> 1) * 64 + li * 2 + (k & 1)]; }
};

// segment of v-row v: starts[g] <= v < starts[g+1]
__device__ __forceinline__ int seg_of(const int32_t* __restrict__ starts, int nseg, int v) {
    int lo = 0, hi = nseg;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (starts[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// term i of a row with m terms: chunk (stage) and slot
__device__ __forceinline__ void chunk_of(int i, int m, int C, int C0, int& s, int& q) {
    const int r = m - 1 - i;  // 0 = last term
    if (r < C0) {
        s = 0;
        q = 3 - r;
    } else {
        s = 1 + (r - C0) / C;
        q = 3 - (r - C0) % C;
    }
}

struct PlanDev {
    int32_t* Db;     // [nblk]
    int32_t* R;      // [nblk][EMAX] max (producer step + 1 - consumer load step)
    int32_t* Wb;     // [nblk][EMAX] max (consumer load step - producer step)
    int* out;        // [0] fail bits, [1] dm, [2] ring requirement
};

// pass 1: validity, in-block skew D_b, reach
template <int K>
__global__ void k_wave_req(Sell S, const int32_t* nlow, const int32_t* starts, int32_t nseg, int NR, int C,
                           PlanDev p) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int SPW = 32 / NR, P = NR - 1, C0 = K == kSkewL ? C : C - 1;
    const int g = seg_of(starts, nseg, v), ix = v - starts[g], k = g % SPW;
    RowView<K> r(S, v, nlow);
    int dreq = 1, dm = 0, ring = 0, fail = 0, prev = INT_MIN;
    for (int i = 0; i < r.len; ++i) {
        const int c = r.col(i);
        if (c <= prev || c >= v) fail |= 1;
        prev = c;
        int s, q;
        chunk_of(i, r.len, C, C0, s, q);
        if (s > P) fail |= 2;
        const int gc = seg_of(starts, nseg, c), jx = c - starts[gc], d = g - gc;
        if (d > MAXD) fail |= 8;
        dm = max(dm, d);
        if (d == 0) {
            const bool xb = q == 3 && jx == ix - s - 1;
            if (!xb && jx > ix - s - 2) fail |= 4;
            ring = max(ring, ix - s - jx + 2);
        } else if (d <= k) {
            const int need = jx - ix + s + 2;
            if (need > 0) dreq = max(dreq, (need + d - 1) / d);
        }
    }
    atomicMax(p.Db + g / SPW, dreq);
    if (fail) atomicOr(p.out + 0, fail);
    atomicMax(p.out + 1, dm);
    atomicMax(p.out + 2, ring);
}

// pass 2: leads and read-behind between blocks; in-block ring requirement
template <int K>
__global__ void k_wave_req2(Sell S, const int32_t* nlow, const int32_t* starts, int32_t nseg, int NR, int C,
                            PlanDev p) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int SPW = 32 / NR, P = NR - 1, C0 = K == kSkewL ? C : C - 1;
    const int g = seg_of(starts, nseg, v), ix = v - starts[g], k = g % SPW, b = g / SPW;
    const int D = p.Db[b];
    RowView<K> r(S, v, nlow);
    int Rl[EMAX], Wl[EMAX];
    for (int e = 0; e < EMAX; ++e) Rl[e] = Wl[e] = INT_MIN;
    int ring = 0;
    for (int i = 0; i < r.len; ++i) {
        const int c = r.col(i);
        int s, q;
        chunk_of(i, r.len, C, C0, s, q);
        const int gc = seg_of(starts, nseg, c), jx = c - starts[gc], d = g - gc;
        if (d == 0 || d > MAXD) continue;
        const int tload = (ix - s) + P + D * k - 1;
        if (d <= k) {
            ring = max(ring, ix - s + D * d - jx);
        } else {
            const int bp = gc / SPW, kp = gc % SPW, e = b - bp;
            if (e < 1 || e > EMAX) continue;
            const int pstep = jx + P + p.Db[bp] * kp;
            Rl[e - 1] = max(Rl[e - 1], pstep + 1 - tload);
            Wl[e - 1] = max(Wl[e - 1], tload - pstep);
        }
    }
    for (int e = 0; e < EMAX; ++e)
        if (Rl[e] > INT_MIN) {
            atomicMax(p.R + b * EMAX + e, Rl[e]);
            atomicMax(p.Wb + b * EMAX + e, Wl[e]);
        }
    atomicMax(p.out + 2, ring);
}

// pass 3: items, one thread per (step, lane)
template <int K>
__global__ void k_wave_fill(Sell S, const int32_t* __restrict__ nlow, const double* __restrict__ dinv,
                            const int32_t* __restrict__ starts, int32_t nseg, const int32_t* __restrict__ Db, const int64_t* __restrict__ off, int32_t nblk,
                            int NR, int C, int W, int DM, int RY, int ring0, int xb, unsigned sbase,
                            int64_t nsteps, uint4* __restrict__ item) {
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= nsteps * 32) return;
    const int64_t ts = gid >> 5;
    const int lane = int(gid & 31);
    const int SPW = 32 / NR, P = NR - 1, C0 = K == kSkewL ? C : C - 1, DS = 4 - C;
    const int k = lane / NR, rl = lane % NR;
    int lo = 0, hi = nblk;  // the block holding step ts
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= ts) lo = mid;
        else hi = mid;
    }
    const int b = lo, t = int(ts - off[b]), D = Db[b];
    const int g = b * SPW + k;
    const int g0 = (b / W) * W * SPW;  // first segment of the CTA
    const int base = t - P - D * k;    // the segment's stage-0 row at step t
    const int s = ((rl - base) % NR + NR) % NR;
    const int ix = base + s;           // the row this lane works on (chunk s)
    const int RYS = RY + 1;
    const unsigned zero = sbase + ring0 + 8 * RY;
    Step it;
    for (int q = 0; q < 4; ++q) {
        it.w[q] = 0.0;
        it.o[q] = unsigned(zero);
    }
    if (g < nseg && ix >= 0 && ix < starts[g + 1] - starts[g]) {
        const int v = starts[g] + ix;
        RowView<K> r(S, v, nlow);
        if (s == 0 && K != kSkewL) it.w[DS] = dinv[v];
        for (int i = 0; i < r.len; ++i) {
            int si, q;
            chunk_of(i, r.len, C, C0, si, q);
            if (si != s) continue;
            const int c = r.col(i);
            const int gc = seg_of(starts, nseg, c), jx = c - starts[gc], d = g - gc;
            it.w[q] = r.val(i);
            if (d == 0 && q == 3 && jx == ix - s - 1) {
                it.o[q] = sbase + unsigned(xb);
            } else {  // the cell of the step that finalised row jx of segment gc
                const int ridx = DM + (gc - g0);
                const int pstep = jx + P + Db[gc / SPW] * (gc % SPW);
                it.o[q] = sbase + unsigned(ring0 + 8 * (ridx * RYS + (pstep & (RY - 1))));
            }
        }
    }
    uint4 c0, c1, c2;
    c0.x = unsigned(__double_as_longlong(it.w[0]));
    c0.y = unsigned(__double_as_longlong(it.w[0]) >> 32);
    c0.z = unsigned(__double_as_longlong(it.w[1]));
    c0.w = unsigned(__double_as_longlong(it.w[1]) >> 32);
    c1.x = unsigned(__double_as_longlong(it.w[2]));
    c1.y = unsigned(__double_as_longlong(it.w[2]) >> 32);
    c1.z = unsigned(__double_as_longlong(it.w[3]));
    c1.w = unsigned(__double_as_longlong(it.w[3]) >> 32);
    c2 = make_uint4(it.o[0], it.o[1], it.o[2], it.o[3]);
    item[(ts * 3 + 0) * 32 + lane] = c0;
    item[(ts * 3 + 1) * 32 + lane] = c1;
    item[(ts * 3 + 2) * 32 + lane] = c2;
}

// Gauss-Seidel pre-pass: the upper sums over the old values; also prepares the sweep (sentinels in
// its output, claim counter reset) so that a GS sweep is two launches
__global__ void k_wave_gs_su(Sell S, const int32_t* __restrict__ nlow, const double* __restrict__ old,
                             double* __restrict__ su, double* __restrict__ out, int* __restrict__ ticket) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v == 0) *ticket = 0;
    if (v >= S.n) return;
    out[v] = sentinel();
    const int64_t base = S.off[v >> 5];
    const int li = v & 31, len = S.len[v];
    double s = 0.0;
    for (int k = nlow[v]; k < len; ++k)
        s = s + S.val[base + (k >> 1) * 64 + li * 2 + (k & 1)] * old[S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)]];
    su[v] = s;
}

__global__ void k_wave_prep2(double* __restrict__ y, double* __restrict__ x, int32_t n, int* __restrict__ ticket) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v == 0) ticket[0] = ticket[1] = 0;
    if (v >= n) return;
    y[v] = sentinel();
    x[v] = sentinel();
}

__global__ void k_wave_upd(const double* __restrict__ x, double* __restrict__ u, int32_t n) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t i = n - 1 - v;
    u[i] = u[i] + x[v];
}

template <int K>
void launch_req(const Sell& S, const int32_t* nlow, const int32_t* starts, int32_t nseg, int NR, int C,
                const PlanDev& p, bool second, cudaStream_t st) {
    const int nb = ceil_div(S.n, 256);
    if (second) k_wave_req2<K><<<nb, 256, 0, st>>>(S, nlow, starts, nseg, NR, C, p);
    else k_wave_req<K><<<nb, 256, 0, st>>>(S, nlow, starts, nseg, NR, C, p);
    PMG_LAUNCH_CHECK();
}

__global__ void k_sbase(unsigned* out) {
    extern __shared__ __align__(128) unsigned char probe_smem[];
    *out = smem_u32(probe_smem);
}

// shared-window address of a kernel's dynamic shared memory (no static shared memory, no
// cluster): the items are built with it (absolute LDS addresses), k_wave checks it
unsigned dyn_smem_base(cudaStream_t st) {
    static const unsigned base = [st] {
        unsigned* d = nullptr;
        unsigned h = 0;
        PMG_CUDA(cudaMalloc(&d, sizeof(unsigned)));
        k_sbase<<<1, 32, 128, st>>>(d);
        PMG_LAUNCH_CHECK();
        PMG_CUDA(cudaMemcpyAsync(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        PMG_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
        return h;
    }();
    return base;
}

int smem_limit() {
    static const int lim = [] {
        int dev = 0, v = 0;
        PMG_CUDA(cudaGetDevice(&dev));
        PMG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        return v;
    }();
    return lim;
}

}  // namespace

bool g_wave_dump = false;
double* g_wave_dump_buf[3] = {nullptr, nullptr, nullptr};
int g_wave_dump_n[3] = {0, 0, 0};
bool g_wave_trace_on = false;
unsigned long long* g_wave_trace = nullptr;
int g_wave_trace_n = 0;

std::vector<int32_t> uniform_starts(int32_t n, int32_t seg) {
    std::vector<int32_t> v;
    for (int64_t i = 0; i < n; i += seg) v.push_back(int32_t(i));
    v.push_back(n);
    return v;
}

std::vector<int32_t> reversed_starts(const std::vector<int32_t>& s) {
    const int32_t n = s.back();
    std::vector<int32_t> r(s.size());
    for (size_t i = 0; i < s.size(); ++i) r[i] = n - s[s.size() - 1 - i];
    return r;
}

bool wave_plan(const Sell& S, const double* dinv, const std::vector<int32_t>& hstarts, SkewKind kind,
               int32_t max_terms, WavePlan& plan, cudaStream_t st, const int32_t* nlow) {
    wave_plan_free(plan);
    if (S.n == 0 || hstarts.size() < 2 || hstarts.front() != 0 || hstarts.back() != S.n) return false;
    int32_t seg = 0;  // longest segment
    for (size_t i = 0; i + 1 < hstarts.size(); ++i) {
        if (hstarts[i + 1] <= hstarts[i]) return false;
        seg = std::max(seg, hstarts[i + 1] - hstarts[i]);
    }
    static const int lay[][2] = {{4, 3}, {8, 4}, {16, 4}, {32, 3}, {32, 4}};
    const int extra = kind == kSkewL ? 0 : 1;  // chunk 0 carries 1/diagonal
    int NR = 0, C = 0;
    for (auto& l : lay)
        if (l[0] * l[1] - extra >= max_terms) {
            NR = l[0];
            C = l[1];
            break;
        }
    if (!NR) return false;
    const bool verbose = getenv("PMG_VERBOSE") != nullptr;
    const int SPW = 32 / NR, P = NR - 1;
    const int nseg = int(hstarts.size()) - 1;
    const int nblk = ceil_div(nseg, SPW);
    int32_t* starts = nullptr;
    PMG_CUDA(cudaMalloc(&starts, sizeof(int32_t) * (nseg + 1)));
    PMG_CUDA(cudaMemcpyAsync(starts, hstarts.data(), sizeof(int32_t) * (nseg + 1), cudaMemcpyHostToDevice, st));
    PlanDev p{};
    PMG_CUDA(cudaMalloc(&p.Db, sizeof(int32_t) * nblk));
    PMG_CUDA(cudaMalloc(&p.R, sizeof(int32_t) * nblk * EMAX));
    PMG_CUDA(cudaMalloc(&p.Wb, sizeof(int32_t) * nblk * EMAX));
    PMG_CUDA(cudaMalloc(&p.out, sizeof(int) * 4));
    auto release = [&] {
        cudaFree(starts);
        cudaFree(p.Db);
        cudaFree(p.R);
        cudaFree(p.Wb);
        cudaFree(p.out);
    };
    std::vector<int32_t> minus(size_t(nblk) * EMAX, INT_MIN);
    PMG_CUDA(cudaMemsetAsync(p.Db, 0, sizeof(int32_t) * nblk, st));
    PMG_CUDA(cudaMemcpyAsync(p.R, minus.data(), sizeof(int32_t) * minus.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(p.Wb, minus.data(), sizeof(int32_t) * minus.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemsetAsync(p.out, 0, sizeof(int) * 4, st));
    auto req = [&](bool second) {
        if (kind == kSkewL) launch_req<kSkewL>(S, nlow, starts, nseg, NR, C, p, second, st);
        else if (kind == kSkewU) launch_req<kSkewU>(S, nlow, starts, nseg, NR, C, p, second, st);
        else launch_req<kSkewGS>(S, nlow, starts, nseg, NR, C, p, second, st);
    };
    req(false);
    int h[4];
    PMG_CUDA(cudaMemcpyAsync(h, p.out, sizeof(h), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    if (h[0]) {
        if (verbose)
            fprintf(stderr, "[pmg] wave plan rejected (n=%d seg=%d NR=%d): %s%s%s%s\n", S.n, seg, NR,
                    h[0] & 1 ? "unsorted " : "", h[0] & 2 ? "row too long " : "", h[0] & 4 ? "own value late " : "",
                    h[0] & 8 ? "reach beyond 8 segments" : "");
        release();
        return false;
    }
    req(true);
    std::vector<int32_t> hD(nblk), hR(size_t(nblk) * EMAX), hW(size_t(nblk) * EMAX);
    PMG_CUDA(cudaMemcpyAsync(h, p.out, sizeof(h), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hD.data(), p.Db, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hR.data(), p.R, sizeof(int32_t) * hR.size(), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hW.data(), p.Wb, sizeof(int32_t) * hW.size(), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    const int dm = std::max(h[1], 1);
    // leads: L_b = max_e (R[b][e] + (e-1) - sum_{i<e} L_{b-i}), never negative
    std::vector<int64_t> Lb(nblk, 0);
    for (int b = 0; b < nblk; ++b) {
        int64_t L = 0, sum = 0;
        for (int e = 1; e <= EMAX && b - e >= 0; ++e) {
            const int32_t R = hR[size_t(b) * EMAX + e - 1];
            if (R > INT_MIN) L = std::max<int64_t>(L, R + (e - 1) - sum);
            sum += Lb[b - e];
        }
        Lb[b] = L;
    }
    // ring rows: own / in-block requirement, and the cross-block window (lead chain + read-behind)
    int64_t need = h[2];
    for (int b = 0; b < nblk; ++b) {
        int64_t chain = 0;
        for (int e = 1; e <= EMAX && b - e + 1 >= 0; ++e) {
            chain += Lb[b - e + 1];
            const int32_t Wv = hW[size_t(b) * EMAX + e - 1];
            if (Wv > INT_MIN) need = std::max<int64_t>(need, chain + Wv);
        }
    }
    need += 2 * G + EMAX * 8;  // room for the run-time slack (wave_sweep) of up to 8 steps per block
    int ry = 64;
    while (ry < need) ry *= 2;
    // warps per CTA: as many as shared memory holds
    const bool gs = kind == kSkewGS;
    int W = 0;
    for (int w = WMAX; w >= 1; --w)
        if (ry <= 4096 && layout(w, SPW, dm, ry, gs).total <= smem_limit()) {
            W = w;
            break;
        }
    if (const char* e = getenv("PMG_WAVE_W")) W = std::min(W, std::max(1, atoi(e)));
    if (!W) {
        if (verbose)
            fprintf(stderr, "[pmg] wave plan rejected (n=%d seg=%d NR=%d): rings of %d rows exceed shared memory\n",
                    S.n, seg, NR, ry);
        release();
        return false;
    }
    const Layout ly = layout(W, SPW, dm, ry, gs);
    const int ntask = ceil_div(nblk, W);
    // back-pressure: producer b, consumer b+j in the same CTA
    std::vector<int32_t> hbp(size_t(nblk) * W, -INF);
    for (int b = 0; b < nblk; ++b)
        for (int j = 1; j < W; ++j) {
            const int c = b + j;
            if (c >= nblk || c / W != b / W || j > EMAX) continue;
            const int32_t Wv = hW[size_t(c) * EMAX + j - 1];
            if (Wv > INT_MIN) hbp[size_t(b) * W + j] = Wv - ry;
        }
    // bridge data per CTA task and halo distance
    std::vector<int32_t> hho(size_t(ntask) * MAXD, INT_MIN), hhr(size_t(ntask) * W * MAXD, INF),
        hsl(size_t(ntask) * MAXD, 0);
    for (int tk = 0; tk < ntask; ++tk) {
        const int b0 = tk * W, g0 = b0 * SPW;
        for (int d = 0; d < dm; ++d) {
            const int gh = g0 - 1 - d;
            if (gh < 0) continue;
            const int bpd = gh / SPW, kp = gh % SPW, e = b0 - bpd;
            hsl[size_t(tk) * MAXD + d] = int32_t(P + int64_t(hD[bpd]) * kp);
            bool used = false;
            for (int w = 0; w < W && b0 + w < nblk; ++w) {
                const int ee = e + w;
                if (ee > EMAX) continue;
                if (hR[size_t(b0 + w) * EMAX + ee - 1] > INT_MIN) {
                    used = true;
                    const int32_t Wv = hW[size_t(b0 + w) * EMAX + ee - 1];
                    hhr[(size_t(tk) * W + w) * MAXD + d] = int32_t(ry - Wv - P - int64_t(hD[bpd]) * kp);
                }
            }
            if (!used) continue;
            int64_t sum = 0;
            for (int i = 1; i < e; ++i) sum += Lb[b0 - i];
            hho[size_t(tk) * MAXD + d] = int32_t(P + int64_t(hD[bpd]) * kp - sum + (e - 1));
        }
    }
    std::vector<int64_t> hoff(nblk + 1, 0);
    for (int b = 0; b < nblk; ++b) {
        const int kl = std::min(SPW - 1, nseg - 1 - b * SPW);
        int32_t seg = 0;  // the block's longest segment
        for (int k = 0; k <= kl; ++k) seg = std::max(seg, hstarts[b * SPW + k + 1] - hstarts[b * SPW + k]);
        // whole groups, at least NG (the last steps fetch items one group past the end: the
        // ring slot then still holds valid offsets of an earlier group)
        const int64_t ns = std::max<int64_t>(seg + int64_t(kl) * hD[b] + P, NG * G);
        hoff[b + 1] = hoff[b] + (ns + G - 1) / G * G;
    }
    const int64_t nsteps = hoff[nblk];
    std::vector<int32_t> hL(nblk);
    for (int b = 0; b < nblk; ++b) hL[b] = int32_t(std::min<int64_t>(Lb[b], INF));
    int32_t *Lbd = nullptr, *bpd = nullptr, *hod = nullptr, *hrd = nullptr, *hsd = nullptr;
    int64_t* offd = nullptr;
    uint4* item = nullptr;
    PMG_CUDA(cudaMalloc(&Lbd, sizeof(int32_t) * nblk));
    PMG_CUDA(cudaMalloc(&bpd, sizeof(int32_t) * hbp.size()));
    PMG_CUDA(cudaMalloc(&hod, sizeof(int32_t) * hho.size()));
    PMG_CUDA(cudaMalloc(&hrd, sizeof(int32_t) * hhr.size()));
    PMG_CUDA(cudaMalloc(&hsd, sizeof(int32_t) * hsl.size()));
    PMG_CUDA(cudaMemcpyAsync(hsd, hsl.data(), sizeof(int32_t) * hsl.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMalloc(&offd, sizeof(int64_t) * (nblk + 1)));
    PMG_CUDA(cudaMalloc(&item, size_t(nsteps) * STEP_BYTES));
    PMG_CUDA(cudaMemcpyAsync(Lbd, hL.data(), sizeof(int32_t) * nblk, cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(bpd, hbp.data(), sizeof(int32_t) * hbp.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(hod, hho.data(), sizeof(int32_t) * hho.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(hrd, hhr.data(), sizeof(int32_t) * hhr.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(offd, hoff.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, st));
    const int nf = ceil_div(nsteps * 32, 256);
    const unsigned sbase = dyn_smem_base(st);
    if (kind == kSkewL)
        k_wave_fill<kSkewL><<<nf, 256, 0, st>>>(S, nlow, dinv, starts, nseg, p.Db, offd, nblk, NR, C, W, dm, ry, ly.ring,
                                                ly.xb, sbase, nsteps, item);
    else if (kind == kSkewU)
        k_wave_fill<kSkewU><<<nf, 256, 0, st>>>(S, nlow, dinv, starts, nseg, p.Db, offd, nblk, NR, C, W, dm, ry, ly.ring,
                                                ly.xb, sbase, nsteps, item);
    else
        k_wave_fill<kSkewGS><<<nf, 256, 0, st>>>(S, nlow, dinv, starts, nseg, p.Db, offd, nblk, NR, C, W, dm, ry,
                                                 ly.ring, ly.xb, sbase, nsteps, item);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaStreamSynchronize(st));
    cudaFree(p.R);
    cudaFree(p.Wb);
    cudaFree(p.out);
    std::vector<int32_t> sl(hL.begin() + nblk / 4, hL.begin() + std::max(nblk / 4 + 1, 3 * nblk / 4));
    std::sort(sl.begin(), sl.end());
    plan.n = S.n;
    plan.seg = seg;
    plan.nseg = nseg;
    plan.starts = starts;
    plan.nr = NR;
    plan.c = C;
    plan.spw = SPW;
    plan.w = W;
    plan.nblk = nblk;
    plan.ntask = ntask;
    plan.dm = dm;
    plan.ry = ry;
    plan.nsteps = nsteps;
    plan.Db = p.Db;
    plan.Lb = Lbd;
    plan.bp = bpd;
    plan.hoff = hod;
    plan.hrb = hrd;
    plan.hsl = hsd;
    plan.sbase = sbase;
    plan.off = offd;
    plan.item = item;
    plan.lead = sl.empty() ? hL[0] : sl[sl.size() / 2];
    plan.ok = true;
    if (verbose)
        fprintf(stderr, "[pmg] wave plan n=%d seg=%d NRxC %dx%d W %d dm %d ring %d lead %d smem %d\n", S.n, seg, NR, C,
                W, dm, ry, plan.lead, ly.total);
    return true;
}

void wave_plan_free(WavePlan& plan) {
    cudaFree(plan.starts);
    cudaFree(plan.Db);
    cudaFree(plan.Lb);
    cudaFree(plan.bp);
    cudaFree(plan.hoff);
    cudaFree(plan.hrb);
    cudaFree(plan.hsl);
    cudaFree(plan.off);
    cudaFree(plan.item);
    plan = WavePlan{};
}

namespace {
template <int K, int NR, int C>
void launch(const WaveArgs& a, int grid, cudaStream_t st) {
    static const bool attr = [] {
        PMG_CUDA(cudaFuncSetAttribute(k_wave<K, NR, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_limit()));
        return true;
    }();
    (void)attr;
    k_wave<K, NR, C><<<grid, 32 * (a.W + 2), a.lay.total, st>>>(a);
    PMG_LAUNCH_CHECK();
}
template <int K>
void launch_kind(const WavePlan& p, const WaveArgs& a, int grid, cudaStream_t st) {
    if (p.nr == 4) launch<K, 4, 3>(a, grid, st);
    else if (p.nr == 8) launch<K, 8, 4>(a, grid, st);
    else if (p.nr == 16) launch<K, 16, 4>(a, grid, st);
    else if (p.c == 3) launch<K, 32, 3>(a, grid, st);
    else launch<K, 32, 4>(a, grid, st);
}
}  // namespace

void wave_prepare2(double* y, double* x, int32_t n, int* ticket, cudaStream_t st) {
    if (n <= 0) return;
    k_wave_prep2<<<ceil_div(n, 256), 256, 0, st>>>(y, x, n, ticket);
    PMG_LAUNCH_CHECK();
}

void wave_sweep(const WaveOp& op, int* ticket, cudaStream_t st) {
    const WavePlan& p = *op.plan;
    const int32_t n = p.n;
    if (n == 0) return;
    const int nsm = sm_count();
    if (op.kind == kSkewGS) {  // the pre-pass prepares the sweep as well
        k_wave_gs_su<<<ceil_div(n, 256), 256, 0, st>>>(*op.gsS, op.nlow, op.old, op.su, op.out, ticket);
        PMG_LAUNCH_CHECK();
    } else if (!op.prepared) {
        fill_sentinel(op.out, n, st);
        PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    }
    WaveArgs a{};
    a.starts = p.starts;
    a.item = p.item;
    a.rhs = op.rhs;
    a.su = op.su;
    a.out = op.out;
    a.Db = p.Db;
    a.Lb = p.Lb;
    a.bp = p.bp;
    a.hoff = p.hoff;
    a.hrb = p.hrb;
    a.hsl = p.hsl;
    a.sbase = p.sbase;
    // a consumer tests its predecessor's progress with a value read a step earlier; running
    // `slack` steps further behind than the dependencies require lets that stale value pass, so
    // a gated block steps at the free-running rate instead of spinning on every test
    static const int slack = std::max(0, env_int("PMG_WAVE_SLACK", 0));
    a.slack = slack;
    a.trace = nullptr;
    if (g_wave_trace_on) {  // one-shot trace of the next sweep (diagnostics)
        g_wave_trace_on = false;
        cudaFree(g_wave_trace);
        PMG_CUDA(cudaMalloc(&g_wave_trace, sizeof(unsigned long long) * 8 * p.nblk));
        PMG_CUDA(cudaMemsetAsync(g_wave_trace, 0, sizeof(unsigned long long) * 8 * p.nblk, st));
        g_wave_trace_n = p.nblk;
        a.trace = g_wave_trace;
    }
    a.off = p.off;
    a.n = n;
    a.seg = p.seg;
    a.nseg = p.nseg;
    a.nblk = p.nblk;
    a.ntask = p.ntask;
    a.W = p.w;
    a.dm = p.dm;
    a.ry = p.ry;
    a.lay = layout(p.w, p.spw, p.dm, p.ry, op.kind == kSkewGS);
    a.ticket = ticket;
    static const int grid_cap = std::max(0, env_int("PMG_WAVE_GRID", 0));  // tests: fewer CTAs than tasks
    const int grid = std::min(std::min(p.ntask, nsm), grid_cap > 0 ? grid_cap : INT_MAX);
    if (op.kind == kSkewL) launch_kind<kSkewL>(p, a, grid, st);
    else if (op.kind == kSkewU) launch_kind<kSkewU>(p, a, grid, st);
    else launch_kind<kSkewGS>(p, a, grid, st);
    if (g_wave_dump) {  // diagnostics: keep a copy of this sweep's output (v-space), per kind
        double*& d = g_wave_dump_buf[op.kind];
        cudaFree(d);
        PMG_CUDA(cudaMalloc(&d, sizeof(double) * n));
        PMG_CUDA(cudaMemcpyAsync(d, op.out, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        g_wave_dump_n[op.kind] = n;
    }
    if (op.kind == kSkewU) {
        k_wave_upd<<<ceil_div(n, 256), 256, 0, st>>>(op.out, op.upd, n);
        PMG_LAUNCH_CHECK();
    }
}

}  // namespace pmg
