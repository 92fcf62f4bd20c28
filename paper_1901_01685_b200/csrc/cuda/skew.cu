// Skewed-warp wavefront sweeps for factors with short rows and short reach (the p=1 h-levels).
//
// v-order and segments as in chain.cu (segment = one grid row of S rows; L: ascending rows,
// U: descending rows).  A warp owns a block of SPW = 8 consecutive segments; four lanes
// serve each segment, one per pipeline stage.  At step t the stage-s lane of segment k works
// on row ix + s, ix = t - P - k*D: it adds its stage's (<= 3) terms, in the oracle's
// ascending order, to the partial sum the stage-(s+1) lane handed over (shuffle) at the end
// of step t-1; the stage-0 lane adds the v-1 term (its own previous output, a register) and
// finalises the row.  Every value a term needs is already on chip:
//   * values of the row's own segment: the segment's ring in shared memory;
//   * values one segment back: segment k-1's ring, written >= 1 step earlier because the lane
//     skew D covers the forward reach (chosen per factor at plan time);
//   * segment 0's values one segment back come from the previous block (another CTA) through
//     global memory: a bridge warp polls them (NaN-sentinel protocol), copies them into the
//     halo ring and publishes how many are in.
// The per-step static data (coefficients and shared-memory offsets of every lane's terms) is
// stored step-major per block and moved by bulk copies (cp.async.bulk + mbarrier) into a ring;
// the right-hand side is gathered per step with cp.async.  A sweep costs about
// nseg * D steps; a step is one shuffle + three dependent adds on its critical path.
//
// Compared with chain.cu (one CTA per segment, cross-segment hops through L2 for every
// segment) only every 8th segment boundary crosses the memory system here, which is what the
// p=1 factors (9 entries per row, reach ~8 rows) need: their chained sweeps were bound by the
// per-segment hop latency, not by work.
#include <climits>
#include <cstdlib>

#include "skew.cuh"

namespace pmg {

namespace {

constexpr int SPW = 8;        // segments per warp block
constexpr int NR = kSkewP + 1;  // lanes per segment (one per stage)
constexpr int RY = 64;        // per-segment ring of recent outputs
constexpr int RYS = RY + 1;   // + a zero cell (padding terms point at it)
constexpr int G = 16;         // steps per bulk copy
constexpr int NG = 4;         // bulk-copy groups in the ring
constexpr int PF = G * NG;    // steps staged
constexpr int ICH = 3;        // 16-B chunks per (step, lane) item
constexpr int STEP_BYTES = ICH * 32 * 16;
constexpr int P = kSkewP, C = kSkewC;
constexpr unsigned FULL = 0xffffffffu;
static_assert(SPW * NR == 32, "one warp per block");

// per (step, lane) item: the lane's stage data for the row it works on at that step
//   stage s >= 1: w[0..2], o[0..2] = coefficients / byte offsets of the stage's terms
//   stage 0     : w[0] = coefficient of the v-1 term, flag = has0, dinv
struct __align__(16) SkewItem {
    double w[3];
    int32_t o[3];
    int32_t flag;
    double dinv;
};
static_assert(sizeof(SkewItem) == ICH * 16, "SkewItem layout");

struct SkewSmem {
    uint4 item[PF][ICH][32];  // [step slot][16-B chunk][lane]: conflict-free 128-bit reads
    double rhs[PF][32];
    double Y[SPW + 1][RYS];   // row 0: halo (previous block's last segment); row k+1: segment k
    unsigned long long bar[NG];     // items of a group have landed (bulk copy)
    unsigned long long rfull[NG];   // right-hand sides of a group are in (stager warp)
    unsigned long long rempty[NG];  // a group's slots were consumed (sweep warp)
    int halo_ready;           // halo values [0, halo_ready) are in
    int cons_ix;              // segment 0's current row (halo ring reuse)
    int blk;
};

struct SkewArgs {
    const uint4* item;
    const double* rhs;
    double* out;
    int32_t n, seg, nseg, D, b1, ns_full;
    int* ticket;
    unsigned long long* trace;  // optional: per block [claim, end, halo spins, bridge polls]
    int dbg;                    // timing experiments only (PMG_SKEW_DBG bits)
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
__device__ __forceinline__ void cp_async8_z(void* dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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
__device__ __forceinline__ int ld_acq_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_vol_s(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

template <int K, bool TR>
__global__ void __launch_bounds__(96) k_skew(SkewArgs a) {
    extern __shared__ __align__(128) unsigned char skew_smem[];
    SkewSmem& sm = *reinterpret_cast<SkewSmem*>(skew_smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = a.n, S = a.seg, D = a.D;
    constexpr unsigned gbase = 0;  // barriers are re-initialised per block: group q <-> slot q % NG

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            sm.blk = atomicAdd(a.ticket, 1);
            sm.halo_ready = 0;
            sm.cons_ix = -P;
            // every copy / arrival of the previous block has been waited for or has completed
            for (int q = 0; q < NG; ++q) {
                bar_init(&sm.bar[q]);
                bar_init(&sm.rfull[q]);
                bar_init(&sm.rempty[q]);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int q = threadIdx.x; q < (SPW + 1) * RYS; q += 96) (&sm.Y[0][0])[q] = 0.0;
        __syncthreads();
        const int blk = sm.blk;
        const int g0 = blk * SPW;
        if (g0 >= a.nseg) break;
        if (TR && a.trace && threadIdx.x == 0) a.trace[blk * 8 + 0] = gtimer();
        const int kmax = min(SPW - 1, a.nseg - 1 - g0);
        const int T = S + kmax * D;
        const int NS = T + P;                       // steps of this block (t = tau + P)
        const unsigned nq = (NS + G - 1) / G;       // bulk-copy groups of this block

        if (warp == 2) {
            // ---------------------------------------------------------------- stager
            // right-hand sides of the stage-0 rows, group by group, into the rhs ring
            for (unsigned q = 0; q < nq; ++q) {
                const unsigned Q = gbase + q, slot = Q % NG, use = Q / NG;
                if (use > 0) bar_wait(&sm.rempty[slot], (use - 1) & 1);
#pragma unroll
                for (int e0 = 0; e0 < G * SPW; e0 += 32) {
                    const int e = e0 + lane, st = int(q) * G + e / SPW, kk = e % SPW;
                    const int gg = g0 + kk, ix = st - P - D * kk;
                    const int64_t lo2 = int64_t(gg) * S;
                    const bool in = gg < a.nseg && ix >= 0 && ix < S && lo2 + ix < n;
                    const int64_t v = lo2 + ix;
                    sm.rhs[slot * G + e / SPW][kk * NR] = in ? a.rhs[K == kSkewL ? v : int64_t(n) - 1 - v] : 0.0;
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&sm.rfull[slot]);
            }
            continue;
        }
        if (warp == 1) {
            // ---------------------------------------------------------------- bridge
            // previous block's last segment -> halo ring, in order, as its values appear
            if (g0 > 0) {
                const double* src = a.out + int64_t(g0 - 1) * S;
                int j0 = 0;
                unsigned ns = 16;
                while (j0 < S) {
                    const int cap = ld_vol_s(&sm.cons_ix) - a.b1 + RY - j0;  // ring slots free
                    const int j = j0 + lane;
                    double v = sentinel();
                    if (lane < cap && j < S) v = ld_relaxed_nb(src + j);
                    const unsigned ok = __ballot_sync(FULL, !is_sentinel(v));
                    const int cnt = ok == FULL ? 32 : __ffs(~ok) - 1;
                    if (lane < cnt) sm.Y[0][j & (RY - 1)] = v;
                    if (TR && a.trace && lane < cnt && j == 200) a.trace[(blk - 1) * 8 + 5] = gtimer();
                    __syncwarp();
                    if (cnt > 0) {
                        if (lane == 0) st_rel_cta(&sm.halo_ready, j0 + cnt);
                        j0 += cnt;
                        ns = 16;
                    } else {
                        __nanosleep(ns);
                        ns = min(ns * 2, 256u);
                    }
                    if (TR && a.trace && lane == 0) a.trace[blk * 8 + 3]++;
                }
            }
            continue;
        }

        // -------------------------------------------------------------------- sweep warp
        const int k = lane >> 2, role = lane & 3;   // segment in the block, stage of the lane
        const int g = g0 + k;
        const int64_t lo = int64_t(g) * S;
        const int rows = g < a.nseg ? int(min(int64_t(S), int64_t(n) - lo)) : 0;
        const unsigned char* bsrc = reinterpret_cast<const unsigned char*>(a.item) + int64_t(blk) * a.ns_full * STEP_BYTES;
        auto refill = [&](unsigned q) {  // group q of this block's steps -> its ring slot
            if (lane == 0 && q * G < unsigned(NS)) {
                const unsigned slot = (gbase + q) % NG;
                const unsigned bytes = min(G, NS - int(q * G)) * STEP_BYTES;
                bulk_load(&sm.item[slot * G][0][0], bsrc + int64_t(q) * G * STEP_BYTES, bytes, &sm.bar[slot]);
            }
        };
        for (unsigned q = 0; q < NG; ++q) refill(q);

        const char* Yb = reinterpret_cast<const char*>(&sm.Y[k + 1][0]);
        double* Yo = &sm.Y[k + 1][0];
        struct Pre {
            double w0, w1, w2, dinv, rhs;
            int o0, o1, o2, flag;
        };
        auto fetch = [&](int t, Pre& f) {  // static data of step t from the ring
            const uint4* it = &sm.item[t & (PF - 1)][0][lane];
            const uint4 c0 = it[0], c1 = it[32], c2 = it[64];
            f.w0 = __hiloint2double(int(c0.y), int(c0.x));
            f.w1 = __hiloint2double(int(c0.w), int(c0.z));
            f.w2 = __hiloint2double(int(c1.y), int(c1.x));
            f.o0 = int(c1.z);
            f.o1 = int(c1.w);
            f.o2 = int(c2.x);
            f.flag = int(c2.y);
            f.dinv = __hiloint2double(int(c2.w), int(c2.z));
            f.rhs = sm.rhs[t & (PF - 1)][lane];
        };
        auto group_wait = [&](unsigned q) {  // items and right-hand sides of group q are in
            if (q < nq) {
                const unsigned Q = gbase + q;
                bar_wait(&sm.bar[Q % NG], (Q / NG) & 1);
                bar_wait(&sm.rfull[Q % NG], (Q / NG) & 1);
            }
        };
        long long cyc[4] = {0, 0, 0, 0};
        long long c0 = clock64();
        auto tick = [&](int q) {
            if (TR && (a.dbg & 16)) {
                const long long c1 = clock64();
                cyc[q] += c1 - c0;
                c0 = c1;
            }
        };
        double res = 0.0, xprev = 0.0;
        Pre f;
        group_wait(0);
        fetch(0, f);
        // steps are processed in groups of G (static ring positions)
        for (int tb = 0; tb < NS; tb += G) {
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int t = tb + u;
                if (t >= NS) break;  // slots past the block's last group hold stale data
                const int ix = t - P - D * k;  // the segment's stage-0 row at this step
                tick(3);
                if (u == G - 1) group_wait(unsigned(tb) / G + 1);  // for fetch(t + 1) below
                tick(0);
                const double in0 = __shfl_down_sync(FULL, res, 1);  // partial from the next stage's lane
                if (g0 > 0) {  // all lanes test (uniform branch; lane 0 publishes the ring use)
                    if (lane == 0) *reinterpret_cast<volatile int*>(&sm.cons_ix) = ix;
                    const int need = min(t - P + D, S);
                    // relaxed spin: shared-memory accesses of a warp are performed in order, and
                    // the bridge publishes with a release store
                    if (TR && a.trace && lane == 0 && need == 201) a.trace[(blk - 1) * 8 + 6] = gtimer();
                    if (ld_vol_s(&sm.halo_ready) < need) {
                        const long long w0 = clock64();
                        while (ld_vol_s(&sm.halo_ready) < need) {
                        }
                        if (TR && a.trace && lane == 0) a.trace[blk * 8 + 2] += clock64() - w0;
                    }
                    if (TR && a.trace && lane == 0 && need == 201) a.trace[(blk - 1) * 8 + 7] = gtimer();
                }
                __syncwarp();
                tick(2);
                const double y0s = *reinterpret_cast<const double*>(Yb + f.o0);
                const double y1 = *reinterpret_cast<const double*>(Yb + f.o1);
                const double y2 = *reinterpret_cast<const double*>(Yb + f.o2);
                const double in = role == 3 ? 0.0 : in0;
                const double y0 = role == 0 ? (f.flag ? xprev : 0.0) : y0s;
                const double r1 = in + f.w0 * y0;
                res = (r1 + f.w1 * y1) + f.w2 * y2;
                // stage-0 lanes: finalise (their w1, w2 are zero: r1 is the complete row sum)
                const double x = K == kSkewL ? f.rhs - r1 : (f.rhs - r1) * f.dinv;
                if (role == 0 && ix >= 0 && ix < rows) {
                    Yo[ix & (RY - 1)] = x;
                    st_relaxed(a.out + lo + ix, x);
                    if (TR && a.trace && k == SPW - 1 && ix == 200) a.trace[blk * 8 + 4] = gtimer();
                }
                xprev = x;
                fetch(t + 1, f);  // static data of the next step
            }
            // group tb/G fully consumed: hand its rhs slots back, refill its item slots
            __syncwarp();
            const unsigned qd = unsigned(tb) / G;
            if (lane == 0) bar_arrive(&sm.rempty[(gbase + qd) % NG]);
            refill(qd + NG);
        }
        if (TR && a.trace && lane == 0) a.trace[blk * 8 + 1] = gtimer();
        if (TR && (a.dbg & 16) && a.trace && lane == 0 && blk == (a.dbg >> 8)) {
            a.trace[2] = cyc[0] << 32 | cyc[1];  // (issue + group wait) | rhs wait
            a.trace[3] = cyc[2] << 32 | cyc[3];  // halo + syncwarp | compute + store
        }
    }
}

// The record of row v (v-order) of factor S: stage assignment and shared-memory offsets.
// flags: bit 0 = does not fit.  dreq / back1 / back0 as documented in skew_plan.
template <int K>
__device__ void skew_record(const Sell& S, const double* dinv, int32_t seg, int32_t v, SkewRec& r, int& fail,
                            int& dreq, int& back1, int& back0) {
    const int n = S.n, g = v / seg, ix = v - g * seg;
    const int64_t base = S.off[v >> 5];
    const int li = v & 31;
    const int len = S.len[v];
#pragma unroll
    for (int s = 0; s < kSkewSlots; ++s) {
        r.coef[s] = 0.0;
        if (s < kSkewSlots - 1) r.off[s] = RY * 8;  // the lane's zero cell
    }
    r.has0 = 0;
    r.dinv = K == kSkewU ? dinv[v] : 1.0;
    fail = len > kSkewSlots;
    dreq = 1;
    back1 = back0 = INT_MIN;
    int q = len - 1;
    auto col_at = [&](int k) { return vcol<K>(S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)], n); };
    auto val_at = [&](int k) { return S.val[base + (k >> 1) * 64 + li * 2 + (k & 1)]; };
    if (!fail && q >= 0 && col_at(q) == v - 1 && ix > 0) {
        r.coef[P * C] = val_at(q);
        r.has0 = 1;
        --q;
    }
    int st = 1, used = 0, prev = INT_MAX;
    for (; !fail && q >= 0; --q) {
        const int c = col_at(q);
        if (c >= prev || c >= v) fail = 1;  // terms must be strictly ascending and below v
        prev = c;
        if (used == C) {
            ++st;
            used = 0;
        }
        if (st > P) {
            fail = 1;
            break;
        }
        const int gc = c / seg, jx = c - gc * seg, d = g - gc;
        if (d == 0) {
            if (st > ix - jx - 1) fail = 1;  // own value not final by the stage's step
            back0 = max(back0, ix - jx - st);
        } else if (d == 1) {
            dreq = max(dreq, st + 1 + jx - ix);
            back1 = max(back1, ix - jx - st);
        } else {
            fail = 1;
        }
        const int slot = (P - st) * C + (C - 1 - used);
        r.coef[slot] = val_at(q);
        r.off[slot] = (-d * RYS + (jx & (RY - 1))) * 8;
        ++used;
    }
}

// pass 1: out[0] = required D, out[1] = failure flag, out[2] = max (ix - jx - stage) over
// terms one segment back, out[3] = same over the own segment
template <int K>
__global__ void k_skew_req(Sell S, const double* __restrict__ dinv, int32_t seg, int* out) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    SkewRec r;
    int fail, dreq, back1, back0;
    skew_record<K>(S, dinv, seg, v, r, fail, dreq, back1, back0);
    atomicMax(out + 0, dreq);
    if (fail) atomicMax(out + 1, 1);
    atomicMax(out + 2, back1);
    atomicMax(out + 3, back0);
}

// pass 2: step-major items, one thread per (step, lane)
template <int K>
__global__ void k_skew_fill(Sell S, const double* __restrict__ dinv, int32_t seg, int32_t nseg, int32_t D,
                            int32_t ns_full, int64_t nsteps, uint4* __restrict__ item) {
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= nsteps * 32) return;
    const int64_t ts = gid >> 5;
    const int lane = int(gid & 31);
    const int k = lane >> 2, role = lane & 3;
    const int b = int(ts / ns_full), t = int(ts - int64_t(b) * ns_full);
    const int g = b * SPW + k;
    const int ix = t - P - D * k + role;  // the row this lane works on at step t
    SkewItem it{};
    if (g < nseg && ix >= 0 && ix < seg && int64_t(g) * seg + ix < S.n) {
        SkewRec r;
        int fail, dreq, back1, back0;
        skew_record<K>(S, dinv, seg, g * seg + ix, r, fail, dreq, back1, back0);
        if (role == 0) {
            it.w[0] = r.coef[P * C];
            it.flag = r.has0;
            it.dinv = r.dinv;
            it.o[0] = it.o[1] = it.o[2] = RY * 8;
        } else {
            const int s0 = (P - role) * C;
            for (int q = 0; q < C; ++q) {
                it.w[q] = r.coef[s0 + q];
                it.o[q] = r.off[s0 + q];
            }
        }
    } else {
        it.o[0] = it.o[1] = it.o[2] = RY * 8;
    }
    const uint4* src = reinterpret_cast<const uint4*>(&it);
#pragma unroll
    for (int c = 0; c < ICH; ++c) item[(ts * ICH + c) * 32 + lane] = src[c];
}

__global__ void k_skew_upd(const double* __restrict__ x, double* __restrict__ u, int32_t n) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t i = n - 1 - v;
    u[i] = u[i] + x[v];
}

}  // namespace

bool g_skew_trace_on = false;
unsigned long long* g_skew_trace = nullptr;
int g_skew_trace_n = 0;

bool skew_plan(const Sell& S, const double* dinv, int32_t seg, SkewKind kind, SkewPlan& plan, cudaStream_t st) {
    skew_plan_free(plan);
    if (seg <= 0 || S.n == 0) return false;
    int* d;
    PMG_CUDA(cudaMallocAsync(&d, sizeof(int) * 4, st));
    const int init[4] = {0, 0, INT_MIN, INT_MIN};
    PMG_CUDA(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st));
    if (kind == kSkewL) k_skew_req<kSkewL><<<ceil_div(S.n, 256), 256, 0, st>>>(S, dinv, seg, d);
    else k_skew_req<kSkewU><<<ceil_div(S.n, 256), 256, 0, st>>>(S, dinv, seg, d);
    PMG_LAUNCH_CHECK();
    int h[4];
    PMG_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    PMG_CUDA(cudaFreeAsync(d, st));
    const int D = std::max(h[0], 1);
    // ring reuse: a value read one segment back / in the own segment must not be overwritten
    // before its reading step (RY > D + back1, RY > back0), and D + 2 <= RY for the halo
    const bool ok = !h[1] && D + 2 <= RY && (h[2] == INT_MIN || D + h[2] < RY) && (h[3] == INT_MIN || h[3] < RY);
    if (!ok) return false;
    const int nseg = ceil_div(S.n, seg);
    const int nblk = ceil_div(nseg, SPW);
    const int ns_full = seg + (SPW - 1) * D + P;
    const int kl = nseg - 1 - (nblk - 1) * SPW;
    const int ns_last = seg + kl * D + P;
    const int64_t nsteps = int64_t(nblk - 1) * ns_full + ns_last;
    uint4* item = nullptr;
    PMG_CUDA(cudaMalloc(&item, size_t(nsteps) * STEP_BYTES));
    const int64_t nthr = nsteps * 32;
    if (kind == kSkewL)
        k_skew_fill<kSkewL><<<ceil_div(nthr, 256), 256, 0, st>>>(S, dinv, seg, nseg, D, ns_full, nsteps, item);
    else
        k_skew_fill<kSkewU><<<ceil_div(nthr, 256), 256, 0, st>>>(S, dinv, seg, nseg, D, ns_full, nsteps, item);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaStreamSynchronize(st));
    plan.n = S.n;
    plan.seg = seg;
    plan.D = D;
    plan.b1 = std::max(h[2], 1);
    plan.nseg = nseg;
    plan.nblk = nblk;
    plan.ns_full = ns_full;
    plan.ns_last = ns_last;
    plan.item = item;
    plan.ok = true;
    return true;
}

void skew_plan_free(SkewPlan& plan) {
    cudaFree(plan.item);
    plan = SkewPlan{};
}

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st) {
    const SkewPlan& p = *op.plan;
    const int32_t n = p.n;
    if (n == 0) return;
    fill_sentinel(op.out, n, st);
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const int nseg = ceil_div(n, p.seg);
    const int nblk = ceil_div(nseg, SPW);
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        PMG_CUDA(cudaGetDevice(&dev));
        PMG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const int smem = int(sizeof(SkewSmem));
    static bool attr = false;
    if (!attr) {
        PMG_CUDA(cudaFuncSetAttribute(k_skew<kSkewL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        PMG_CUDA(cudaFuncSetAttribute(k_skew<kSkewU, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        PMG_CUDA(cudaFuncSetAttribute(k_skew<kSkewL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        PMG_CUDA(cudaFuncSetAttribute(k_skew<kSkewU, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    static int dbg = -1;
    if (dbg < 0) {
        const char* e = getenv("PMG_SKEW_DBG");
        dbg = e ? atoi(e) : 0;
    }
    SkewArgs a{p.item, op.rhs, op.out, n, p.seg, nseg, p.D, p.b1, p.ns_full, ticket, nullptr, dbg};
    if (g_skew_trace_on) {  // one-shot trace of the next sweep (diagnostics)
        g_skew_trace_on = false;
        cudaFree(g_skew_trace);
        PMG_CUDA(cudaMalloc(&g_skew_trace, sizeof(unsigned long long) * 8 * nblk));
        PMG_CUDA(cudaMemsetAsync(g_skew_trace, 0, sizeof(unsigned long long) * 8 * nblk, st));
        g_skew_trace_n = nblk;
        a.trace = g_skew_trace;
    }
    static int grid_cap = -1;  // tests: fewer CTAs than blocks (CTAs then loop over blocks)
    if (grid_cap < 0) {
        const char* e = getenv("PMG_SKEW_GRID");
        grid_cap = e ? std::max(1, atoi(e)) : 0;
    }
    const int grid = std::min(std::min(nblk, nsm), grid_cap > 0 ? grid_cap : nsm);
    if (a.trace) {
        if (op.kind == kSkewL) k_skew<kSkewL, true><<<grid, 96, smem, st>>>(a);
        else k_skew<kSkewU, true><<<grid, 96, smem, st>>>(a);
    } else {
        if (op.kind == kSkewL) k_skew<kSkewL, false><<<grid, 96, smem, st>>>(a);
        else k_skew<kSkewU, false><<<grid, 96, smem, st>>>(a);
    }
    PMG_LAUNCH_CHECK();
    if (op.kind == kSkewU) {
        k_skew_upd<<<ceil_div(n, 256), 256, 0, st>>>(op.out, op.upd, n);
        PMG_LAUNCH_CHECK();
    }
}

}  // namespace pmg
