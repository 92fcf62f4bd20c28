// Skewed-warp wavefront sweeps for factors with short rows and short reach (the p=1 h-levels).
//
// v-order and segments as in chain.cu (segment = one grid row).  A warp owns 32 consecutive
// segments, lane k <-> segment g0+k.  At step tau lane k computes the row at position
// ix = tau - k*D of its segment, completely and sequentially in the oracle's order.  D is chosen
// at setup so that every entry of a row that lies d >= 1 segments back satisfies
// jx - ix < d*D: that value was produced by lane k-d at least one step earlier and is read from
// its shared-memory ring; values of the row's own segment come from the lane's own ring; values
// from before the warp's first segment come from global memory (NaN-sentinel protocol).  Warps
// claim 32-segment blocks in order and start once their predecessor is 32*D steps ahead.
#include <climits>
#include <vector>

#include "skew.cuh"

namespace pmg {

namespace {

constexpr int R = 32;       // per-lane ring of recent outputs (rb*D + reach + 2 <= R)
constexpr int WPB = 4;      // warps per CTA
constexpr unsigned FULL = 0xffffffffu;

struct SkewArgs {
    Sell S;
    const double* dinv;
    const int32_t* perm;
    const double* rhs;
    double* out;
    double* upd;
    int32_t n, seg, nseg, D;
    int* ticket;
    int* prog;
};

template <int K>
__device__ __forceinline__ int vcol(int c, int n) {
    return K == kSkewU ? n - 1 - c : c;
}

template <int K>
__global__ void __launch_bounds__(32 * WPB) k_skew(SkewArgs a) {
    __shared__ double ring[WPB][32][R + 1];  // +1: lanes of a warp hit different banks
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double (*my)[R + 1] = ring[warp];
    const int n = a.n, S = a.seg, D = a.D;
    const int nsteps = S + 31 * D;
    for (;;) {
        int wb = 0;
        if (lane == 0) wb = atomicAdd(a.ticket, 1);
        wb = __shfl_sync(FULL, wb, 0);
        const int g0 = wb * 32;
        if (g0 >= a.nseg) break;
        // start once the predecessor block is 32*D steps ahead (or done)
        if (wb > 0 && lane == 0) {
            unsigned ns = 64;
            while (*reinterpret_cast<volatile int*>(a.prog + wb - 1) < min(32 * D, nsteps)) {
                __nanosleep(ns);
                ns = min(ns * 2, 1024u);
            }
        }
        __syncwarp();
        const int g = g0 + lane;
        for (int tau = 0; tau < nsteps; ++tau) {
            const int ix = tau - lane * D;
            const int v = g * S + ix;
            if (g < a.nseg && ix >= 0 && ix < S && v < n) {
                const int64_t base = a.S.off[v >> 5];
                const int li = v & 31;
                const int len = a.S.len[v];
                const int* cb = a.S.col + base + li * 4;
                const double* vb = a.S.val + base + li * 2;
                double acc = 0.0;
                for (int k = 0; k < len; k += 4) {
                    const int4 c4 = __ldg(reinterpret_cast<const int4*>(cb + (k >> 2) * 128));
                    const double2 w0 = __ldg(reinterpret_cast<const double2*>(vb + (k >> 1) * 64));
                    const double2 w1 = __ldg(reinterpret_cast<const double2*>(vb + (k >> 1) * 64 + 64));
                    const int cc[4] = {c4.x, c4.y, c4.z, c4.w};
                    const double ww[4] = {w0.x, w0.y, w1.x, w1.y};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (k + q >= len) break;
                        const int c = vcol<K>(cc[q], n);
                        const int gc = c / S;
                        const int jx = c - gc * S;
                        const int src = lane - (g - gc);  // lane holding segment gc
                        double y;
                        if (src >= 0) y = ring[warp][src][jx & (R - 1)];
                        else y = wait_value(a.out, c);
                        acc = acc + ww[q] * y;
                    }
                }
                double y;
                if (K == kSkewL) y = a.rhs[a.perm ? a.perm[v] : v] - acc;
                else y = (a.rhs[n - 1 - v] - acc) * a.dinv[v];
                my[lane][ix & (R - 1)] = y;
                st_relaxed(a.out + v, y);
                if (K == kSkewU) {
                    const int i = n - 1 - v;
                    const int ui = a.perm ? a.perm[i] : i;
                    a.upd[ui] = a.upd[ui] + y;
                }
            }
            __syncwarp();
            if (lane == 0 && (tau & 15) == 15) *reinterpret_cast<volatile int*>(a.prog + wb) = tau + 1;
        }
        if (lane == 0) *reinterpret_cast<volatile int*>(a.prog + wb) = INT_MAX;
    }
}

// per row: required skew D (> (jx - ix)/d for entries d segments back), rows back, internal reach
__global__ void k_skew_params(Sell S, int32_t seg, int K, int* out /* [3]: D, rb, reach */) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= S.n) return;
    const int n = S.n;
    const int g = v / seg, ix = v - g * seg;
    const int64_t base = S.off[v >> 5];
    const int li = v & 31;
    int Dq = 1, rb = 0, reach = 0;
    for (int k = 0; k < S.len[v]; ++k) {
        int c = S.col[base + (k >> 2) * 128 + li * 4 + (k & 3)];
        if (K == kSkewU) c = n - 1 - c;
        const int gc = c / seg, jx = c - gc * seg, d = g - gc;
        if (d == 0) reach = max(reach, ix - jx);
        else {
            rb = max(rb, d);
            const int diff = jx - ix;  // need diff < d*D
            if (diff >= 0) Dq = max(Dq, diff / d + 1);
        }
    }
    atomicMax(out + 0, Dq);
    atomicMax(out + 1, rb);
    atomicMax(out + 2, reach);
}

}  // namespace

bool skew_plan(const Sell& S, int32_t seg, SkewKind kind, int32_t max_row, SkewPlan& plan, cudaStream_t st) {
    plan = SkewPlan{};
    if (seg <= 0 || S.n == 0 || max_row > 32) return false;
    int* d;
    PMG_CUDA(cudaMallocAsync(&d, sizeof(int) * 3, st));
    PMG_CUDA(cudaMemsetAsync(d, 0, sizeof(int) * 3, st));
    k_skew_params<<<ceil_div(S.n, 256), 256, 0, st>>>(S, seg, int(kind), d);
    PMG_LAUNCH_CHECK();
    int h[3];
    PMG_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    PMG_CUDA(cudaFreeAsync(d, st));
    plan.D = std::max(h[0], 1);
    plan.rb = h[1];
    plan.reach = h[2];
    // ring validity: a value read d segments back lies within rb*D + reach of the writer
    plan.ok = plan.rb <= 2 && plan.rb * plan.D + plan.reach + 2 <= R && plan.reach + 1 < R;
    return plan.ok;
}

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st) {
    const int32_t n = op.S->n;
    if (n == 0) return;
    fill_sentinel(op.out, n, st);
    const int nseg = ceil_div(n, op.seg);
    const int nblk = ceil_div(nseg, 32);
    static int* prog = nullptr;
    static int cap = 0;
    if (nblk > cap) {
        cudaFree(prog);
        PMG_CUDA(cudaMalloc(&prog, sizeof(int) * nblk));
        cap = nblk;
    }
    PMG_CUDA(cudaMemsetAsync(prog, 0, sizeof(int) * nblk, st));
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    SkewArgs a{*op.S, op.dinv, op.perm, op.rhs, op.out, op.upd, n, op.seg, nseg, op.D, ticket, prog};
    const int grid = ceil_div(nblk, WPB);
    if (op.kind == kSkewL) k_skew<kSkewL><<<grid, 32 * WPB, 0, st>>>(a);
    else k_skew<kSkewU><<<grid, 32 * WPB, 0, st>>>(a);
    PMG_LAUNCH_CHECK();
}

}  // namespace pmg
