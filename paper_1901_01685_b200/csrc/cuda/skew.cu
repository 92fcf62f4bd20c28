// Skewed-warp wavefront sweeps for sparse triangular solves on tensor-grid orderings.
//
// v-order and segments as in chain.cu (segment = one grid row of S rows; L: ascending rows,
// U: descending rows).  A row's terms (its entries in ascending v-column) are assigned to
// pipeline stages at plan time: stage 0 is the v-1 term, stages 1..P hold C terms each,
// counted back from the end, so stage s is summed s steps before the row is finalised.
// NR = P+1 lanes serve one segment, one per stage; a warp owns SPW = 32/NR consecutive
// segments (a "block") and at step t the stage-s lane of segment k works on row
// ix + s, ix = t - P - k*D.  It adds its stage's terms, in the oracle's ascending order, to
// the partial sum the stage-(s+1) lane handed over (shuffle) at the end of step t-1; the
// stage-0 lane adds the v-1 term (its own previous output, a register) and finalises the row.
// Every value a term needs is already on chip:
//   * own segment: the segment's ring in shared memory;
//   * d segments back inside the block: that segment's ring, written >= 1 step earlier because
//     the lane skew D covers the forward reach (D >= (stage + 1 + jx - ix) / d per term);
//   * d segments back beyond the block: halo rings, filled from global memory by a bridge warp
//     that polls the previous block's last DM segments (NaN-sentinel protocol).
// The per-step static data (coefficients and shared-memory offsets of every lane's terms) is
// stored step-major per block and moved by bulk copies (cp.async.bulk + mbarrier) into a ring;
// a stager warp gathers the right-hand sides.  A sweep costs about nseg * D steps; a step is a
// shuffle plus C dependent adds on its critical path.
//
// Layouts per factor (chosen by skew_plan from the longest row): NR x C = 4 x 3 (p = 1,
// <= 10 terms), 8 x 4 (<= 29), 16 x 4 (<= 61), 32 x 3 (<= 94), 32 x 4 (<= 125).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "skew.cuh"

namespace pmg {

namespace {

constexpr int G = 32;         // steps per bulk copy
constexpr int NG = 2;         // bulk-copy groups in the ring
constexpr int PF = G * NG;    // steps staged
constexpr int ICH = 3;        // 16-B chunks per (step, lane) item
constexpr int STEP_BYTES = ICH * 32 * 16;
constexpr int MAXD = 8;       // segments back a term may reach
constexpr unsigned FULL = 0xffffffffu;
constexpr int NT = 96;        // sweep warp, bridge warp, stager warp

// per (step, lane) item: the lane's stage data for the row it works on at that step
//   stage s >= 1: w[0..3], o[0..3] = coefficients / byte offsets of the stage's terms
//   stage 0     : w[0] = coefficient of the v-1 term, w[1] = 1/diagonal (U), o[0] = 8 if
//                 the row has a v-1 term else 0, o[1..3] = zero cell
struct __align__(16) SkewItem {
    double w[4];
    int32_t o[4];
};
static_assert(sizeof(SkewItem) == ICH * 16, "SkewItem layout");

struct SkewSmem {
    uint4 item[PF][ICH][32];  // [step slot][16-B chunk][lane]: conflict-free 128-bit reads
    double rhs[PF][32];
    double su[PF][32];              // Gauss-Seidel: the rows' upper sums over the old values
    unsigned long long bar[NG];     // items of a group have landed (bulk copy)
    unsigned long long rfull[NG];   // right-hand sides of a group are in (stager warp)
    unsigned long long rempty[NG];  // a group's slots were consumed (sweep warp)
    int halo_ready;           // segment 0 may work on rows < halo_ready + 1 (all halo values it needs are in)
    int cons_ix;              // segment 0's current row (halo ring reuse)
    int blk;
    int pad;
    // followed by double Y[DM + SPW][RY + 1]: rows 0..DM-1 halo (segment g0-DM .. g0-1),
    // row DM + k: segment k of the block; cell RY of every row is a zero
};

struct SkewArgs {
    const uint4* item;
    const double* rhs;
    double* out;
    const int32_t* Db;        // [nblk] lane skew of the block
    const int64_t* off;       // [nblk+1] first step of the block in the item stream
    const int32_t* R;         // [nblk][MAXD] lead (rows) a halo segment needs over segment 0
    const int32_t* W;         // [nblk][MAXD] how far behind segment 0 a halo value is still read
    const double* su;         // Gauss-Seidel upper sums (natural order)
    const int32_t* far_off;   // [nblk+1] far-table entries of the block (terms > MAXD segments back)
    const int32_t* far_idx;   // v-space rows of those values, sorted per block
    const int32_t* far_blk;   // [nblk] the last block the far values come from (-1: none)
    int* done;                // [nblk] block finished (release), reset per sweep
    int32_t n, seg, nseg, dm, ry;
    int* ticket;
    unsigned long long* trace;  // optional: per block [claim, end, halo wait cycles, bridge polls, ...]
};
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int K>
__device__ __forceinline__ int vcol(int c, int n) {
    return K == kSkewU ? n - 1 - c : c;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
// one bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_vol_s(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_shared_if(double* p, double v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f64 [%0], %1;\n\t}" ::"r"(smem_u32(p)),
                 "d"(v), "r"(int(pred))
                 : "memory");
}

template <int K, int NR, int C, bool TR>
__global__ void __launch_bounds__(NT) k_skew(SkewArgs a) {
    constexpr int SPW = 32 / NR, P = NR - 1;
    extern __shared__ __align__(128) unsigned char skew_smem[];
    SkewSmem& sm = *reinterpret_cast<SkewSmem*>(skew_smem);
    const int DM = a.dm, RY = a.ry, RYS = a.ry + 1;
    double* Ybase = reinterpret_cast<double*>(skew_smem + sizeof(SkewSmem));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = a.n, S = a.seg;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            sm.blk = atomicAdd(a.ticket, 1);
            sm.halo_ready = INT_MIN / 2;
            sm.cons_ix = -P;
            // every copy / arrival of the previous block has been waited for or has completed
            for (int q = 0; q < NG; ++q) {
                bar_init(&sm.bar[q]);
                bar_init(&sm.rfull[q]);
                bar_init(&sm.rempty[q]);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int q = threadIdx.x; q < (DM + SPW) * RYS; q += NT) Ybase[q] = 0.0;
        __syncthreads();
        const int blk = sm.blk;
        const int g0 = blk * SPW;
        if (g0 >= a.nseg) break;
        if (TR && a.trace && threadIdx.x == 0) a.trace[blk * 8 + 0] = gtimer();
        const int D = a.Db[blk];
        const int NS = int(a.off[blk + 1] - a.off[blk]);  // steps of this block (t = tau + P)
        const unsigned nq = (NS + G - 1) / G;       // bulk-copy groups of this block

        if (warp == 2) {
            // ---------------------------------------------------------------- stager
            // right-hand sides of the stage-0 rows, group by group, into the rhs ring
            for (unsigned q = 0; q < nq; ++q) {
                const unsigned slot = q % NG, use = q / NG;
                if (use > 0) bar_wait(&sm.rempty[slot], (use - 1) & 1);
#pragma unroll
                for (int e0 = 0; e0 < G * SPW; e0 += 32) {
                    const int e = e0 + lane;
                    if (G * SPW >= 32 || e < G * SPW) {
                        const int st = int(q) * G + e / SPW, kk = e % SPW;
                        const int gg = g0 + kk, ix = st - P - D * kk;
                        const int64_t lo2 = int64_t(gg) * S;
                        const bool in = gg < a.nseg && ix >= 0 && ix < S && lo2 + ix < n;
                        const int64_t v = lo2 + ix;
                        sm.rhs[slot * G + e / SPW][kk * NR] =
                            in ? a.rhs[K == kSkewU ? int64_t(n) - 1 - v : v] : 0.0;
                        if (K == kSkewGS) sm.su[slot * G + e / SPW][kk * NR] = in ? a.su[v] : 0.0;
                    }
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.rfull[slot]);
            }
            continue;
        }
        if (warp == 1) {
            // ---------------------------------------------------------------- bridge
            // the previous block's last DM segments -> halo rings, in order, as values appear.
            // halo_ready = h publishes [0, h + (delta-1)*D) of segment g0-delta for every delta.
            if (g0 > 0) {
                const int f0 = a.far_off[blk], nf = a.far_off[blk + 1] - f0;
                if (nf > 0) {  // far values: once their last block is done, copy them once
                    const int* dn = a.done + a.far_blk[blk];
                    unsigned ns = 64;
                    while (ld_acquire(dn) == 0) {
                        __nanosleep(ns);
                        ns = min(ns * 2, 1024u);
                    }
                    // done[far_blk] does not imply that lower source blocks have finished (a
                    // block with no halo needs can end early): wait on every value
                    double* far = Ybase + (DM + SPW) * RYS;
                    for (int i = lane; i < nf; i += 32) far[i] = wait_value(a.out, a.far_idx[f0 + i]);
                    __syncwarp();
                }
                int f[MAXD], Rq[MAXD], Wq[MAXD];
#pragma unroll
                for (int d = 0; d < MAXD; ++d) {
                    Rq[d] = d < DM ? a.R[blk * MAXD + d] : INT_MIN;
                    Wq[d] = d < DM ? a.W[blk * MAXD + d] : 0;
                    f[d] = (Rq[d] > INT_MIN / 2 && g0 - 1 - d >= 0) ? 0 : S;  // halo rows nobody reads: done
                }
                int pub = INT_MIN / 2, idle = 0;
                unsigned ns = 16;
                while (pub < INT_MAX / 2) {
                    const int cons = ld_vol_s(&sm.cons_ix);
                    // rows further back are polled only while they may bind: their producers ran
                    // earlier, so they are usually far ahead of what segment 0 needs
                    const int lim = f[0] < S ? f[0] - Rq[0] + 32 : INT_MAX / 2;
                    double v[MAXD];
#pragma unroll
                    for (int d = 0; d < MAXD; ++d) {  // halo distance delta = d + 1: all polls in flight at once
                        v[d] = sentinel();
                        const int cap = cons - Wq[d] + RY - f[d];  // ring slots free
                        const int j = f[d] + lane;
                        if (d < DM && f[d] < S && lane < cap && j < S && (d == 0 || f[d] - Rq[d] <= lim))
                            v[d] = ld_relaxed_nb(a.out + int64_t(g0 - 1 - d) * S + j);
                    }
                    bool moved = false;
                    int h = INT_MAX / 2;
#pragma unroll
                    for (int d = 0; d < MAXD; ++d) {
                        if (d < DM && f[d] < S) {
                            const unsigned ok = __ballot_sync(FULL, !is_sentinel(v[d]));
                            const int cnt = ok == FULL ? 32 : __ffs(~ok) - 1;
                            if (lane < cnt) Ybase[(DM - 1 - d) * RYS + ((f[d] + lane) & (RY - 1))] = v[d];
                            if (TR && a.trace && d == 0 && f[d] <= 200 && f[d] + cnt > 200 && lane == 0)
                                a.trace[(blk - 1) * 8 + 5] = gtimer();
                            f[d] += cnt;
                            moved = moved || cnt > 0;
                            if (f[d] < S) h = min(h, f[d] - Rq[d]);
                        }
                    }
                    __syncwarp();
                    if (h > pub) {
                        if (lane == 0) st_rel_cta(&sm.halo_ready, h);
                        if (TR && a.trace && lane == 0 && f[0] > 200 && a.trace[(blk - 1) * 8 + 6] == 0)
                            a.trace[(blk - 1) * 8 + 6] = gtimer();
                        pub = h;
                    }
                    if (moved) {  // spin while values flow (this warp has its own scheduler slot)
                        ns = 16;
                        idle = 0;
                    } else if (++idle > 8 && pub >= cons) {  // sleep only while segment 0 is not waiting
                        __nanosleep(ns);
                        ns = min(ns * 2, 256u);
                    }
                    if (TR && a.trace && lane == 0) a.trace[blk * 8 + 3]++;
                }
            }
            continue;
        }

        // -------------------------------------------------------------------- sweep warp
        const int k = lane / NR, role = lane % NR;  // segment in the block, stage of the lane
        const int g = g0 + k;
        const int64_t lo = int64_t(g) * S;
        const int rows = g < a.nseg ? int(min(int64_t(S), int64_t(n) - lo)) : 0;
        const unsigned char* bsrc =
            reinterpret_cast<const unsigned char*>(a.item) + a.off[blk] * STEP_BYTES;
        auto refill = [&](unsigned q) {  // group q of this block's steps -> its ring slot
            if (lane == 0 && q < nq) {
                const unsigned slot = q % NG;
                const unsigned bytes = min(G, NS - int(q * G)) * STEP_BYTES;
                bulk_load(&sm.item[slot * G][0][0], bsrc + int64_t(q) * G * STEP_BYTES, bytes, &sm.bar[slot]);
            }
        };
        for (unsigned q = 0; q < NG; ++q) refill(q);

        const char* Yb = reinterpret_cast<const char*>(Ybase + (DM + k) * RYS);
        double* Yo = Ybase + (DM + k) * RYS;
        struct Pre {
            double w[4], rhs, su;
            int o[4];
        };
        auto fetch = [&](int t, Pre& f) {  // static data of step t from the ring
            const uint4* it = &sm.item[t & (PF - 1)][0][lane];
            const uint4 c0 = it[0], c1 = it[32], c2 = it[64];
            f.w[0] = __hiloint2double(int(c0.y), int(c0.x));
            f.w[1] = __hiloint2double(int(c0.w), int(c0.z));
            f.w[2] = __hiloint2double(int(c1.y), int(c1.x));
            f.w[3] = __hiloint2double(int(c1.w), int(c1.z));
            f.o[0] = int(c2.x);
            f.o[1] = int(c2.y);
            f.o[2] = int(c2.z);
            f.o[3] = int(c2.w);
            f.rhs = sm.rhs[t & (PF - 1)][lane];
            if (K == kSkewGS) f.su = sm.su[t & (PF - 1)][lane];
        };
        auto group_wait = [&](unsigned q) {  // items and right-hand sides of group q are in
            if (q < nq) {
                bar_wait(&sm.bar[q % NG], (q / NG) & 1);
                bar_wait(&sm.rfull[q % NG], (q / NG) & 1);
            }
        };
        double res = 0.0, xprev = 0.0;
        int hr = INT_MIN / 2;  // last seen halo_ready
        Pre fa, fb;  // double-buffered step data: even steps of a group read fa, odd steps fb
        group_wait(0);
        fetch(0, fa);
        static_assert(G % 2 == 0, "double-buffered step data needs an even group length");
        for (int tb = 0; tb < NS; tb += G) {
#pragma unroll
            for (int u = 0; u < G; ++u) {
                Pre& f = (u & 1) ? fb : fa;
                Pre& fnext = (u & 1) ? fa : fb;
                const int t = tb + u;
                const int ix = t - P - D * k;  // the segment's stage-0 row at this step
                if (u == G - 1) group_wait(unsigned(tb) / G + 1);  // for fetch(t + 1) below
                const double in0 = __shfl_down_sync(FULL, res, 1);  // partial from the next stage's lane
                if (g0 > 0) {  // all lanes test (uniform branch; lane 0 publishes the ring use)
                    if (lane == 0) *reinterpret_cast<volatile int*>(&sm.cons_ix) = t - P;
                    // hr was loaded one step ago, so the test is off the critical path unless
                    // segment 0 runs right behind the halo; relaxed loads: shared-memory
                    // accesses of a warp are performed in order, the bridge publishes with a
                    // release store
                    if (hr < t - P) {
                        const long long w0 = clock64();
                        do {
                            hr = ld_vol_s(&sm.halo_ready);
                        } while (hr < t - P);
                        if (TR && a.trace && lane == 0) a.trace[blk * 8 + 2] += clock64() - w0;
                    }
                    if (TR && a.trace && lane == 0 && t - P == 200 - 46) a.trace[(blk - 1) * 8 + 7] = gtimer();
                }
                __syncwarp();
                double y[C];
#pragma unroll
                for (int q = 0; q < C; ++q) y[q] = *reinterpret_cast<const double*>(Yb + f.o[q]);
                const double in = role == NR - 1 ? 0.0 : in0;
                if (role == 0) y[0] = f.o[0] ? xprev : 0.0;
                const double r1 = in + f.w[0] * y[0];
                double r = r1;
#pragma unroll
                for (int q = 1; q < C; ++q) r = r + f.w[q] * y[q];
                res = r;
                // stage-0 lanes: finalise (r1 is their complete row sum, w[1] their 1/diagonal)
                const double x = K == kSkewL    ? f.rhs - r1
                                 : K == kSkewU ? (f.rhs - r1) * f.w[1]
                                               : ((f.rhs - r1) - f.su) * f.w[1];  // GS: SPEC order
                {  // predicated stores (no divergent branch on the step's path)
                    const bool put = role == 0 && ix >= 0 && ix < rows;
                    st_shared_if(Yo + (ix & (RY - 1)), x, put);
                    st_relaxed_if(a.out + lo + ix, x, put);
                    if (TR && a.trace && put && k == SPW - 1 && ix == 200) a.trace[blk * 8 + 4] = gtimer();
                }
                xprev = x;
                if (g0 > 0) hr = ld_vol_s(&sm.halo_ready);  // for the next step's test
                fetch(t + 1, fnext);  // static data of the next step
            }
            // group tb/G fully consumed: hand its rhs slots back, refill its item slots
            __syncwarp();
            const unsigned qd = unsigned(tb) / G;
            if (lane == 0) bar_arrive(&sm.rempty[qd % NG]);
            refill(qd + NG);
        }
        if (TR && a.trace && lane == 0) a.trace[blk * 8 + 1] = gtimer();
        __syncwarp();  // every row of the block is stored: publish (blocks far ahead read it)
        if (lane == 0) {
            __threadfence();
            st_release(a.done + blk, 1);
        }
    }
}

// The terms of row v (v-order) of factor S, ascending v-column: count and accessors.
template <int K>
struct RowView {
    const Sell& S;
    int v, n, len;
    int64_t base;
    int li;
    // Gauss-Seidel: only the lower entries (the first nlow[v]) are terms of the sweep
    __device__ RowView(const Sell& s, int v_, const int32_t* nlow)
        : S(s), v(v_), n(s.n), len(K == kSkewGS ? nlow[v_] : s.len[v_]), base(s.off[v_ >> 5]), li(v_ & 31) {}
    __device__ int col(int k) const { return vcol<K>(S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)], n); }
    __device__ double val(int k) const { return S.val[base + (k >> 1) * 64 + li * 2 + (k & 1)]; }
};

// Walk the terms of row v with their stages: f(stage, d, jx) for every term before the v-1
// term; returns false if a term does not fit the layout (more than P stages, own value not
// final by its stage, not ascending, more than MAXD segments back).
template <int K, class F>
__device__ bool for_terms(const Sell& S, const int32_t* nlow, int32_t seg, int v, int NR, int C, int& why, F&& f) {
    RowView<K> r(S, v, nlow);
    const int g = v / seg, ix = v - g * seg, P = NR - 1;
    int q = r.len - 1;
    if (q >= 0 && r.col(q) == v - 1 && ix > 0) --q;  // stage 0: the v-1 term
    int prev = INT_MAX;
    bool ok = true;
    for (int b = 0; q >= 0; --q, ++b) {
        const int c = r.col(q);
        if (c >= prev || c >= v) {  // terms must be strictly ascending and below v
            ok = false;
            why |= 1;
        }
        prev = c;
        const int st = 1 + b / C;
        if (st > P) {
            why |= 2;
            return false;
        }
        const int gc = c / seg, jx = c - gc * seg, d = g - gc;
        if (d == 0 && st > ix - jx - 1) {  // own value not final by the stage's step
            ok = false;
            why |= 4;
        }
        f(st, d, jx, ix, c);  // d > MAXD: a "far" term, read from the block's far table
    }
    return ok;
}

// pass 1a: per block, the lane skew D_b covering every term inside the block; global failure,
// own-segment back reach and segments-back reach.  out[0] fail, out[1] back0, out[2] dmax
template <int K>
__global__ void k_skew_req(Sell S, const int32_t* nlow, int32_t seg, int NR, int C, int32_t* Db, int* out,
                           int* nfar, uint64_t* far, int far_cap) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int SPW = 32 / NR, g = v / seg, k = g % SPW;
    int dreq = 1, back0 = INT_MIN, dmax = 0, why = 0;
    const bool ok = for_terms<K>(S, nlow, seg, v, NR, C, why, [&](int st, int d, int jx, int ix, int c) {
        if (d == 0) {
            back0 = max(back0, ix - jx - st);
        } else if (d > MAXD) {
            const int i = atomicAdd(nfar, 1);  // (block, column) of a far term
            if (far && i < far_cap) far[i] = (uint64_t(uint32_t(g / SPW)) << 32) | uint32_t(c);
        } else {
            dmax = max(dmax, d);
            const int need = st + 1 + jx - ix;  // d * D >= need for a term inside the block
            if (d <= k && need > 0) dreq = max(dreq, (need + d - 1) / d);
        }
    });
    atomicMax(Db + g / SPW, dreq);
    if (!ok) atomicOr(out + 0, why | 16);
    atomicMax(out + 1, back0);
    atomicMax(out + 2, dmax);
}

// pass 1b: per block and halo distance, the lead R and the read-behind window W of segment 0
// (in segment-0 rows); out[0] = ring requirement inside the block
template <int K>
__global__ void k_skew_req2(Sell S, const int32_t* nlow, int32_t seg, int NR, int C,
                            const int32_t* __restrict__ Db, int32_t* R, int32_t* W, int* out) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int SPW = 32 / NR, g = v / seg, k = g % SPW, b = g / SPW;
    const int D = Db[b];
    int ring = INT_MIN;
    int Rl[MAXD], Wl[MAXD];
    for (int d = 0; d < MAXD; ++d) Rl[d] = Wl[d] = INT_MIN;
    int why = 0;
    for_terms<K>(S, nlow, seg, v, NR, C, why, [&](int st, int d, int jx, int ix, int) {
        if (d == 0 || d > MAXD) return;
        if (d <= k) {
            ring = max(ring, ix - jx - st + d * D);  // writer row at the read minus jx
        } else {
            const int hd = d - k - 1;  // halo distance - 1
            Rl[hd] = max(Rl[hd], st + 1 + jx - ix - D * k);
            Wl[hd] = max(Wl[hd], ix + D * k - st - jx);
        }
    });
    for (int d = 0; d < MAXD; ++d)
        if (Rl[d] > INT_MIN) {
            atomicMax(R + b * MAXD + d, Rl[d]);
            atomicMax(W + b * MAXD + d, Wl[d]);
        }
    atomicMax(out, ring);
}

// pass 2: step-major items, one thread per (step, lane)
template <int K>
__global__ void k_skew_fill(Sell S, const int32_t* __restrict__ nlow, const double* __restrict__ dinv, int32_t seg,
                            int32_t nseg, const int32_t* __restrict__ far_off, const int32_t* __restrict__ far_idx,
                            const int32_t* __restrict__ Db, const int64_t* __restrict__ off, int32_t nblk, int NR,
                            int C, int RY, int64_t nsteps, uint4* __restrict__ item) {
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= nsteps * 32) return;
    const int64_t ts = gid >> 5;
    const int lane = int(gid & 31);
    const int SPW = 32 / NR, P = NR - 1;
    const int k = lane / NR, role = lane % NR;
    int lo = 0, hi = nblk;  // the block holding step ts: off[b] <= ts < off[b+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= ts) lo = mid;
        else hi = mid;
    }
    const int b = lo, t = int(ts - off[b]), D = Db[b];
    const int g = b * SPW + k;
    const int ix = t - P - D * k + role;  // the row this lane works on at step t
    const int zero = RY * 8;
    SkewItem it{};
    for (int q = 0; q < 4; ++q) it.o[q] = zero;
    if (g < nseg && ix >= 0 && ix < seg && int64_t(g) * seg + ix < S.n) {
        const int v = g * seg + ix;
        RowView<K> r(S, v, nlow);
        int q = r.len - 1;
        const bool has0 = q >= 0 && r.col(q) == v - 1 && ix > 0;
        if (role == 0) {
            it.w[0] = has0 ? r.val(q) : 0.0;
            it.w[1] = K == kSkewL ? 1.0 : dinv[v];
            it.o[0] = has0 ? 8 : 0;
        } else {
            if (has0) --q;
            const int hi = q - (role - 1) * C;  // the stage's last term
            const int RYS = RY + 1;
            for (int s = 0; s < C; ++s) {
                const int kk = hi - s;
                if (kk < 0) break;
                const int c = r.col(kk);
                const int gc = c / seg, jx = c - gc * seg, d = g - gc;
                it.w[C - 1 - s] = r.val(kk);
                if (d <= MAXD) {
                    it.o[C - 1 - s] = (-d * RYS + (jx & (RY - 1))) * 8;
                } else {  // far table after the block's rings: slot of c in the block's sorted list
                    int lo2 = far_off[b], hi2 = far_off[b + 1];
                    while (lo2 < hi2) {
                        const int mid = (lo2 + hi2) >> 1;
                        if (far_idx[mid] < c) lo2 = mid + 1;
                        else hi2 = mid;
                    }
                    it.o[C - 1 - s] = ((SPW - k) * RYS + (lo2 - far_off[b])) * 8;
                }
            }
        }
    }
    const uint4* src = reinterpret_cast<const uint4*>(&it);
#pragma unroll
    for (int c = 0; c < ICH; ++c) item[(ts * ICH + c) * 32 + lane] = src[c];
}

// Gauss-Seidel pre-pass: su[v] = sum over the upper entries of a_vj * u_old[j], ascending
// from +0 (the oracle's S_U order)
__global__ void k_skew_gs_su(Sell S, const int32_t* __restrict__ nlow, const double* __restrict__ old,
                             double* __restrict__ su) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int64_t base = S.off[v >> 5];
    const int li = v & 31, len = S.len[v];
    double s = 0.0;
    for (int k = nlow[v]; k < len; ++k)
        s = s + S.val[base + (k >> 1) * 64 + li * 2 + (k & 1)] * old[S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)]];
    su[v] = s;
}

__global__ void k_skew_upd(const double* __restrict__ x, double* __restrict__ u, int32_t n) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t i = n - 1 - v;
    u[i] = u[i] + x[v];
}

size_t smem_bytes(int NR, int dm, int ry, int nfar) {
    return sizeof(SkewSmem) + sizeof(double) * ((dm + 32 / NR) * (ry + 1) + nfar);
}

}  // namespace

bool g_skew_trace_on = false;
unsigned long long* g_skew_trace = nullptr;
int g_skew_trace_n = 0;

bool skew_plan(const Sell& S, const double* dinv, int32_t seg, SkewKind kind, int32_t max_terms, SkewPlan& plan,
               cudaStream_t st, const int32_t* nlow) {
    skew_plan_free(plan);
    if (seg <= 0 || S.n == 0) return false;
    // the smallest layout whose stages hold the longest row
    static const int lay[][2] = {{4, 3}, {8, 4}, {16, 4}, {32, 3}, {32, 4}};  // C <= 4: SkewItem
    int NR = 0, C = 0;
    for (auto& l : lay)
        if (1 + (l[0] - 1) * l[1] >= max_terms) {
            NR = l[0];
            C = l[1];
            break;
        }
    if (!NR) return false;
    const int SPW = 32 / NR, P = NR - 1;
    const int nseg = ceil_div(S.n, seg);
    const int nblk = ceil_div(nseg, SPW);
    int32_t *Db = nullptr, *R = nullptr, *W = nullptr;
    int64_t* off = nullptr;
    int* d = nullptr;
    PMG_CUDA(cudaMalloc(&Db, sizeof(int32_t) * nblk));
    PMG_CUDA(cudaMalloc(&R, sizeof(int32_t) * nblk * MAXD));
    PMG_CUDA(cudaMalloc(&W, sizeof(int32_t) * nblk * MAXD));
    PMG_CUDA(cudaMalloc(&off, sizeof(int64_t) * (nblk + 1)));
    PMG_CUDA(cudaMalloc(&d, sizeof(int) * 4));
    auto fail = [&] {
        cudaFree(Db);
        cudaFree(R);
        cudaFree(W);
        cudaFree(off);
        cudaFree(d);
        return false;
    };
    std::vector<int32_t> minus(size_t(nblk) * MAXD, INT_MIN);
    PMG_CUDA(cudaMemsetAsync(Db, 0, sizeof(int32_t) * nblk, st));
    PMG_CUDA(cudaMemcpyAsync(R, minus.data(), sizeof(int32_t) * minus.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(W, minus.data(), sizeof(int32_t) * minus.size(), cudaMemcpyHostToDevice, st));
    const int init[4] = {0, INT_MIN, 0, INT_MIN};
    PMG_CUDA(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int nb = ceil_div(S.n, 256);
    // far terms (> MAXD segments back, e.g. patch interfaces): counted, then collected
    int* nfar = nullptr;
    uint64_t* farp = nullptr;
    PMG_CUDA(cudaMalloc(&nfar, sizeof(int)));
    auto req = [&](uint64_t* fp, int cap) {
        PMG_CUDA(cudaMemsetAsync(nfar, 0, sizeof(int), st));
        PMG_CUDA(cudaMemsetAsync(Db, 0, sizeof(int32_t) * nblk, st));
        if (kind == kSkewL) k_skew_req<kSkewL><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, d, nfar, fp, cap);
        else if (kind == kSkewU) k_skew_req<kSkewU><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, d, nfar, fp, cap);
        else k_skew_req<kSkewGS><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, d, nfar, fp, cap);
        PMG_LAUNCH_CHECK();
        int h = 0;
        PMG_CUDA(cudaMemcpyAsync(&h, nfar, sizeof(int), cudaMemcpyDeviceToHost, st));
        PMG_CUDA(cudaStreamSynchronize(st));
        return h;
    };
    const int nfar_terms = req(nullptr, 0);
    std::vector<uint64_t> hfar;
    if (nfar_terms > 0) {
        PMG_CUDA(cudaMalloc(&farp, sizeof(uint64_t) * nfar_terms));
        req(farp, nfar_terms);
        hfar.resize(nfar_terms);
        PMG_CUDA(cudaMemcpy(hfar.data(), farp, sizeof(uint64_t) * nfar_terms, cudaMemcpyDeviceToHost));
        cudaFree(farp);
    }
    cudaFree(nfar);
    // per block: sorted distinct far rows and the last block they come from
    std::sort(hfar.begin(), hfar.end());
    hfar.erase(std::unique(hfar.begin(), hfar.end()), hfar.end());
    std::vector<int32_t> hfo(nblk + 1, 0), hfi, hfb(nblk, -1);
    int max_far = 0;
    {
        size_t q = 0;
        for (int b = 0; b < nblk; ++b) {
            hfo[b] = int32_t(hfi.size());
            while (q < hfar.size() && int(hfar[q] >> 32) == b) {
                const int32_t c = int32_t(uint32_t(hfar[q]));
                hfi.push_back(c);
                hfb[b] = std::max(hfb[b], (c / seg) / SPW);
                ++q;
            }
            max_far = std::max(max_far, int(hfi.size()) - hfo[b]);
        }
        hfo[nblk] = int32_t(hfi.size());
    }
    if (kind == kSkewL) k_skew_req2<kSkewL><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, R, W, d + 3);
    else if (kind == kSkewU) k_skew_req2<kSkewU><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, R, W, d + 3);
    else k_skew_req2<kSkewGS><<<nb, 256, 0, st>>>(S, nlow, seg, NR, C, Db, R, W, d + 3);
    PMG_LAUNCH_CHECK();
    int h[4];
    std::vector<int32_t> hD(nblk), hR(size_t(nblk) * MAXD), hW(size_t(nblk) * MAXD);
    PMG_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hD.data(), Db, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hR.data(), R, sizeof(int32_t) * hR.size(), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(hW.data(), W, sizeof(int32_t) * hW.size(), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    if (h[0]) {
        if (getenv("PMG_VERBOSE"))
            fprintf(stderr, "[pmg] skew plan rejected (n=%d seg=%d NR=%d): %s%s%s\n", S.n, seg, NR,
                    h[0] & 1 ? "unsorted " : "", h[0] & 2 ? "row too long " : "", h[0] & 4 ? "own value late" : "");
        return fail();
    }
    const int dm = std::max(h[2], 1);
    // rings: the own segment's back reach, what a reader inside the block still needs, and
    // the halo window (lead + read-behind) with room for the bridge to run ahead
    int need = std::max(h[1] + 1, h[3] + 1);
    int64_t Dsum = 0, Dmax = 0;
    for (int b = 0; b < nblk; ++b) {
        Dsum += hD[b];
        Dmax = std::max<int64_t>(Dmax, hD[b]);
        for (int q = 0; q < MAXD; ++q)
            if (hR[size_t(b) * MAXD + q] > INT_MIN) need = std::max(need, hR[size_t(b) * MAXD + q] + hW[size_t(b) * MAXD + q] + 32);
    }
    int ry = 64;
    while (ry <= need) ry *= 2;
    if (ry > 1024 || smem_bytes(NR, dm, ry, max_far) > 227 * 1024) {
        if (getenv("PMG_VERBOSE"))
            fprintf(stderr, "[pmg] skew plan rejected (n=%d seg=%d NR=%d): rings of %d rows or %d far values exceed "
                            "shared memory\n", S.n, seg, NR, ry, max_far);
        return fail();
    }
    int32_t *far_off = nullptr, *far_idx = nullptr, *far_blk = nullptr;
    int* done = nullptr;
    PMG_CUDA(cudaMalloc(&far_off, sizeof(int32_t) * (nblk + 1)));
    PMG_CUDA(cudaMalloc(&far_idx, sizeof(int32_t) * std::max<size_t>(hfi.size(), 1)));
    PMG_CUDA(cudaMalloc(&far_blk, sizeof(int32_t) * nblk));
    PMG_CUDA(cudaMalloc(&done, sizeof(int) * nblk));
    PMG_CUDA(cudaMemcpyAsync(far_off, hfo.data(), sizeof(int32_t) * (nblk + 1), cudaMemcpyHostToDevice, st));
    if (!hfi.empty())
        PMG_CUDA(cudaMemcpyAsync(far_idx, hfi.data(), sizeof(int32_t) * hfi.size(), cudaMemcpyHostToDevice, st));
    PMG_CUDA(cudaMemcpyAsync(far_blk, hfb.data(), sizeof(int32_t) * nblk, cudaMemcpyHostToDevice, st));
    std::vector<int64_t> hoff(nblk + 1, 0);
    for (int b = 0; b < nblk; ++b) {
        const int kl = std::min(SPW - 1, nseg - 1 - b * SPW);
        // whole bulk-copy groups: the padding steps hold rows past the segments (zero items)
        const int64_t ns = seg + int64_t(kl) * hD[b] + P;
        hoff[b + 1] = hoff[b] + (ns + G - 1) / G * G;
    }
    const int64_t nsteps = hoff[nblk];
    PMG_CUDA(cudaMemcpyAsync(off, hoff.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, st));
    uint4* item = nullptr;
    PMG_CUDA(cudaMalloc(&item, size_t(nsteps) * STEP_BYTES));
    const int64_t nthr = nsteps * 32;
    const int nf = ceil_div(nthr, 256);
    if (kind == kSkewL)
        k_skew_fill<kSkewL><<<nf, 256, 0, st>>>(S, nlow, dinv, seg, nseg, far_off, far_idx, Db, off, nblk, NR, C, ry,
                                                nsteps, item);
    else if (kind == kSkewU)
        k_skew_fill<kSkewU><<<nf, 256, 0, st>>>(S, nlow, dinv, seg, nseg, far_off, far_idx, Db, off, nblk, NR, C, ry,
                                                nsteps, item);
    else
        k_skew_fill<kSkewGS><<<nf, 256, 0, st>>>(S, nlow, dinv, seg, nseg, far_off, far_idx, Db, off, nblk, NR, C,
                                                 ry, nsteps, item);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
    plan.n = S.n;
    plan.seg = seg;
    plan.D = int32_t(Dmax);
    int lead = 0;  // the largest interior lead one segment back (reporting)
    for (int b = nblk / 2; b < std::min(nblk, nblk / 2 + 4); ++b) lead = std::max(lead, hR[size_t(b) * MAXD]);
    plan.lead = SPW == 1 ? lead : int32_t(Dsum / nblk);
    plan.dm = dm;
    plan.ry = ry;
    plan.nr = NR;
    plan.c = C;
    plan.nseg = nseg;
    plan.nblk = nblk;
    plan.nsteps = nsteps;
    plan.Db = Db;
    plan.off = off;
    plan.R = R;
    plan.W = W;
    plan.item = item;
    plan.far_off = far_off;
    plan.far_idx = far_idx;
    plan.far_blk = far_blk;
    plan.done = done;
    plan.nfar_max = max_far;
    plan.ok = true;
    return true;
}

void skew_plan_free(SkewPlan& plan) {
    cudaFree(plan.item);
    cudaFree(plan.far_off);
    cudaFree(plan.far_idx);
    cudaFree(plan.far_blk);
    cudaFree(plan.done);
    cudaFree(plan.Db);
    cudaFree(plan.off);
    cudaFree(plan.R);
    cudaFree(plan.W);
    plan = SkewPlan{};
}

namespace {
template <int K, int NR, int C>
void launch(const SkewArgs& a, int grid, int smem, cudaStream_t st) {
    static const bool attr = [] {
        PMG_CUDA(cudaFuncSetAttribute(k_skew<K, NR, C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        PMG_CUDA(cudaFuncSetAttribute(k_skew<K, NR, C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        return true;
    }();
    (void)attr;
    if (a.trace) k_skew<K, NR, C, true><<<grid, NT, smem, st>>>(a);
    else k_skew<K, NR, C, false><<<grid, NT, smem, st>>>(a);
    PMG_LAUNCH_CHECK();
}
template <int K>
void launch_kind(const SkewPlan& p, const SkewArgs& a, int grid, int smem, cudaStream_t st) {
    if (p.nr == 4) launch<K, 4, 3>(a, grid, smem, st);
    else if (p.nr == 8) launch<K, 8, 4>(a, grid, smem, st);
    else if (p.nr == 16) launch<K, 16, 4>(a, grid, smem, st);
    else if (p.c == 3) launch<K, 32, 3>(a, grid, smem, st);
    else launch<K, 32, 4>(a, grid, smem, st);
}
}  // namespace

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st) {
    const SkewPlan& p = *op.plan;
    const int32_t n = p.n;
    if (n == 0) return;
    fill_sentinel(op.out, n, st);
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const int nsm = sm_count();
    const int smem = int(smem_bytes(p.nr, p.dm, p.ry, p.nfar_max));
    // finished-block flags: the caller's scratch after the ticket (the plan's own array only for
    // factors with more blocks than the scratch holds)
    int* done = p.nblk < kSweepScratchInts ? ticket + 1 : p.done;
    PMG_CUDA(cudaMemsetAsync(done, 0, sizeof(int) * p.nblk, st));
    if (op.kind == kSkewGS) {  // upper sums over the old values, before the sweep
        k_skew_gs_su<<<ceil_div(n, 256), 256, 0, st>>>(*op.gsS, op.nlow, op.old, op.su);
        PMG_LAUNCH_CHECK();
    }
    SkewArgs a{p.item,    op.rhs,    op.out,    p.Db,   p.off, p.R,   p.W,   op.su,   p.far_off, p.far_idx,
               p.far_blk, done,      n,         p.seg,  p.nseg, p.dm, p.ry, ticket, nullptr};
    if (g_skew_trace_on) {  // one-shot trace of the next sweep (diagnostics)
        g_skew_trace_on = false;
        cudaFree(g_skew_trace);
        PMG_CUDA(cudaMalloc(&g_skew_trace, sizeof(unsigned long long) * 8 * p.nblk));
        PMG_CUDA(cudaMemsetAsync(g_skew_trace, 0, sizeof(unsigned long long) * 8 * p.nblk, st));
        g_skew_trace_n = p.nblk;
        a.trace = g_skew_trace;
    }
    static const int grid_cap = std::max(0, env_int("PMG_SKEW_GRID", 0));  // tests: fewer CTAs than blocks
    const int per_sm = std::max(1, int((227 * 1024) / (smem + 1024)));
    const int grid = std::min(std::min(p.nblk, nsm * per_sm), grid_cap > 0 ? grid_cap : INT_MAX);
    if (op.kind == kSkewL) launch_kind<kSkewL>(p, a, grid, smem, st);
    else if (op.kind == kSkewU) launch_kind<kSkewU>(p, a, grid, smem, st);
    else launch_kind<kSkewGS>(p, a, grid, smem, st);
    if (op.kind == kSkewU) {
        k_skew_upd<<<ceil_div(n, 256), 256, 0, st>>>(op.out, op.upd, n);
        PMG_LAUNCH_CHECK();
    }
}

}  // namespace pmg
