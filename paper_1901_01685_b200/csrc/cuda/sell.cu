// SELL-32 layout construction and the SpMV-family kernels (residual + norm, restriction,
// prolongation).  One lane per row, sequential ascending accumulation s = s + a*x from +0
// (no FMA: the library is compiled with -fmad=false), 128-bit coalesced loads.
#include <cub/device/device_scan.cuh>

#include "sell.cuh"

namespace pmg {

// ---------------------------------------------------------------- layout build
__global__ void k_sell_rowlen(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ order, SellPick pick, int32_t* __restrict__ len) {
    int32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n) return;
    int32_t r = order ? order[pos] : pos;
    int32_t l = rowptr[r + 1] - rowptr[r];
    if (pick != kPickAll) {
        for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k)
            if (col[k] == r) { --l; break; }
    }
    len[pos] = l;
}

__global__ void k_sell_slicelen(int32_t n, int32_t nslices, const int32_t* __restrict__ len, int64_t* __restrict__ sl) {
    int32_t s = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (s >= nslices) return;
    int32_t pos = s * 32 + lane;
    int32_t l = pos < n ? len[pos] : 0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) l = max(l, __shfl_xor_sync(0xffffffffu, l, off));
    if (lane == 0) sl[s] = int64_t((l + 3) & ~3) * 32;
    if (s == nslices - 1 && lane == 0) sl[nslices] = 0;
}

__global__ void k_sell_fill(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int32_t* __restrict__ order, SellPick pick,
                            const int64_t* __restrict__ off, int32_t* __restrict__ scol, double* __restrict__ sval,
                            double* __restrict__ diag, int32_t* __restrict__ nlow, int32_t* __restrict__ srow) {
    int32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t s = pos / 32, lane = pos & 31;
    int32_t nslices = (n + 31) / 32;
    if (s >= nslices) return;
    const int64_t base = off[s];
    const int32_t slen = int32_t((off[s + 1] - base) / 32);
    int32_t k = 0;
    if (pos < n) {
        int32_t r = order ? order[pos] : pos;
        if (srow) srow[pos] = r;
        int32_t b = rowptr[r], e = rowptr[r + 1];
        double dg = 0.0;
        int32_t nl = 0;
        if (pick == kPickOffDiagDesc) {
            for (int32_t q = e - 1; q >= b; --q) {
                if (col[q] == r) { dg = val[q]; continue; }
                scol[base + (k >> 2) * 128 + lane * 4 + (k & 3)] = col[q];
                sval[base + (k >> 1) * 64 + lane * 2 + (k & 1)] = val[q];
                ++k;
            }
        } else {
            for (int32_t q = b; q < e; ++q) {
                if (pick == kPickOffDiag && col[q] == r) { dg = val[q]; continue; }
                if (col[q] < r) ++nl;
                scol[base + (k >> 2) * 128 + lane * 4 + (k & 3)] = col[q];
                sval[base + (k >> 1) * 64 + lane * 2 + (k & 1)] = val[q];
                ++k;
            }
        }
        if (diag) diag[pos] = dg;
        if (nlow) nlow[pos] = nl;
    }
    for (; k < slen; ++k) {  // padding: never accumulated, but keep gathers in range
        scol[base + (k >> 2) * 128 + lane * 4 + (k & 3)] = 0;
        sval[base + (k >> 1) * 64 + lane * 2 + (k & 1)] = 0.0;
    }
}

void sell_build(Sell& S, int32_t nrows, const int32_t* d_rowptr, const int32_t* d_col, const double* d_val,
                const int32_t* d_order, SellPick pick, double* d_diag, int32_t* d_nlow, cudaStream_t st) {
    S.n = nrows;
    S.nslices = ceil_div(nrows, 32);
    if (nrows == 0) return;
    PMG_CUDA(cudaMallocAsync(&S.len, sizeof(int32_t) * nrows, st));
    PMG_CUDA(cudaMallocAsync(&S.off, sizeof(int64_t) * (S.nslices + 1), st));
    if (d_order) PMG_CUDA(cudaMallocAsync(&S.row, sizeof(int32_t) * nrows, st));
    k_sell_rowlen<<<ceil_div(nrows, 256), 256, 0, st>>>(nrows, d_rowptr, d_col, d_order, pick, S.len);
    PMG_LAUNCH_CHECK();
    int64_t* sl;
    PMG_CUDA(cudaMallocAsync(&sl, sizeof(int64_t) * (S.nslices + 1), st));
    k_sell_slicelen<<<ceil_div(S.nslices, 8), 256, 0, st>>>(nrows, S.nslices, S.len, sl);
    PMG_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sl, S.off, S.nslices + 1, st);
    void* tmp;
    PMG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sl, S.off, S.nslices + 1, st);
    PMG_CUDA(cudaMemcpyAsync(&S.entries, S.off + S.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    PMG_CUDA(cudaFreeAsync(tmp, st));
    PMG_CUDA(cudaFreeAsync(sl, st));
    PMG_CUDA(cudaMallocAsync(&S.col, sizeof(int32_t) * (S.entries + 4), st));
    PMG_CUDA(cudaMallocAsync(&S.val, sizeof(double) * (S.entries + 2), st));
    k_sell_fill<<<S.nslices, 32, 0, st>>>(nrows, d_rowptr, d_col, d_val, d_order, pick, S.off, S.col, S.val, d_diag,
                                          d_nlow, S.row);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaStreamSynchronize(st));
}

void sell_free(Sell& S) {
    cudaFree(S.off);
    cudaFree(S.len);
    cudaFree(S.row);
    cudaFree(S.col);
    cudaFree(S.val);
    S = Sell{};
}

// ---------------------------------------------------------------- row kernels
// last block of the launch folds the per-block partials in the canonical order
__device__ void norm_finalize(const NormCtx& c, int nblocks) {
    __shared__ double wsum[8];
    __shared__ bool last;
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(c.counter, 1u) == unsigned(nblocks - 1);
    __syncthreads();
    if (!last) return;
    double a = 0.0;
    for (int k = threadIdx.x; k < nblocks; k += 256) a = a + ld_relaxed(c.partials + k);
    a = warp_butterfly(a);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = wsum[0];
        for (int w = 1; w < 8; ++w) t = t + wsum[w];
        double nrm = c.raw ? t : sqrt(t);
        if (c.norm_out) c.norm_out[0] = nrm;
        if (c.hist_out) c.hist_out[0] = nrm / c.n0[0];
        *c.counter = 0u;
    }
}

// sum of the block's 256 terms (squares, or products for a dot) in the canonical chunk order
__device__ __forceinline__ void block_partial(double v, const NormCtx& c) {
    __shared__ double ws[8];
    v = warp_butterfly(v);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = ws[0];
        for (int w = 1; w < 8; ++w) t = t + ws[w];
        c.partials[blockIdx.x] = t;
    }
    norm_finalize(c, gridDim.x);
}
__device__ __forceinline__ void block_sq_partial(double v, const NormCtx& c) { block_partial(v * v, c); }

template <int OP, bool NORM>
__global__ void __launch_bounds__(256) k_rowop(Sell S, const double* __restrict__ x, const double* __restrict__ f,
                                               const double* __restrict__ ml, double* __restrict__ y, NormCtx nc) {
    const int32_t pos = blockIdx.x * 256 + threadIdx.x;
    const int32_t s = pos >> 5, lane = threadIdx.x & 31;
    double out = 0.0;
    if (pos < S.n) {
        const int64_t base = S.off[s];
        const int32_t slen = int32_t((S.off[s + 1] - base) >> 5);
        const int32_t len = S.len[pos];
        const int4* cp = reinterpret_cast<const int4*>(S.col + base) + lane;
        const double2* vp = reinterpret_cast<const double2*>(S.val + base) + lane;
        double acc = 0.0;
#pragma unroll 2
        for (int32_t k = 0; k < slen; k += 4) {
            const int4 c = ld_stream_i4(cp + (k >> 2) * 32);
            const double2 v0 = ld_stream_d2(vp + (k >> 1) * 32);
            const double2 v1 = ld_stream_d2(vp + (k >> 1) * 32 + 32);
            if (k < len) acc = acc + v0.x * __ldg(x + c.x);
            if (k + 1 < len) acc = acc + v0.y * __ldg(x + c.y);
            if (k + 2 < len) acc = acc + v1.x * __ldg(x + c.z);
            if (k + 3 < len) acc = acc + v1.y * __ldg(x + c.w);
        }
        if (OP == kOpSpmv) out = acc;
        else if (OP == kOpResidual) out = f[pos] - acc;
        else if (OP == kOpRestrict) out = acc / ml[pos];
        else if (OP == kOpProlongAdd) out = y[pos] + acc / ml[pos];
        else out = y[pos] + acc;
        y[pos] = out;
    }
    if (NORM) block_sq_partial(out, nc);  // rows past n contribute +0
}

void sell_rowop(const Sell& S, RowOp op, const double* x, const double* f, const double* ml, double* y,
                const NormCtx* norm, cudaStream_t st) {
    if (S.n == 0) return;
    const int nb = ceil_div(S.n, 256);
    NormCtx nc = norm ? *norm : NormCtx{};
    switch (op) {
        case kOpSpmv: k_rowop<kOpSpmv, false><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc); break;
        case kOpResidual:
            if (norm) k_rowop<kOpResidual, true><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc);
            else k_rowop<kOpResidual, false><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc);
            break;
        case kOpRestrict: k_rowop<kOpRestrict, false><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc); break;
        case kOpProlongAdd: k_rowop<kOpProlongAdd, false><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc); break;
        case kOpAdd: k_rowop<kOpAdd, false><<<nb, 256, 0, st>>>(S, x, f, ml, y, nc); break;
    }
    PMG_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) k_vec_norm(const double* __restrict__ v, int32_t n, NormCtx nc) {
    int32_t i = blockIdx.x * 256 + threadIdx.x;
    block_sq_partial(i < n ? v[i] : 0.0, nc);
}

void vec_norm(const double* v, int32_t n, const NormCtx& ctx, cudaStream_t st) {
    k_vec_norm<<<ceil_div(n, 256), 256, 0, st>>>(v, n, ctx);
    PMG_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(256) k_vec_dot(const double* __restrict__ x, const double* __restrict__ y, int32_t n,
                                                 NormCtx nc) {
    int32_t i = blockIdx.x * 256 + threadIdx.x;
    block_partial(i < n ? x[i] * y[i] : 0.0, nc);
}

void vec_dot(const double* x, const double* y, int32_t n, NormCtx ctx, cudaStream_t st) {
    ctx.raw = true;
    k_vec_dot<<<ceil_div(n, 256), 256, 0, st>>>(x, y, n, ctx);
    PMG_LAUNCH_CHECK();
}

__global__ void k_fill(double* v, int64_t n, double x) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) v[i] = x;
}
__global__ void k_fill_sentinel(double* v, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        v[i] = sentinel();
}

void fill_value(double* v, int64_t n, double x, cudaStream_t st) {
    if (n <= 0) return;
    k_fill<<<std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(v, n, x);
    PMG_LAUNCH_CHECK();
}
void fill_sentinel(double* v, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_fill_sentinel<<<std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(v, n);
    PMG_LAUNCH_CHECK();
}

}  // namespace pmg
