// Level-scheduled, sync-free triangular / Gauss-Seidel sweeps.
//
// Rows are visited in level order (level sets built once per factor).  One lane owns one
// row and accumulates it sequentially in the oracle's order; before using x_j it spins
// until row j has published its value (a NaN sentinel marks "not yet produced").  Blocks
// take consecutive 256-row windows of the level order through an atomic ticket, so every
// row a block waits on belongs to a block that started earlier -> no deadlock.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

#include "trsv.cuh"

namespace pmg {

// ---------------------------------------------------------------- level sets
__device__ __forceinline__ int wait_level(const int* lev, int j) {
    int v = ld_acquire(lev + j);
    while (v < 0) {
        __nanosleep(32);
        v = ld_acquire(lev + j);
    }
    return v;
}

__global__ void __launch_bounds__(256) k_levels(int32_t n, const int32_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ col, DepKind dep, int* lev, int* ticket) {
    __shared__ int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1);
    __syncthreads();
    int32_t t = blk * 256 + threadIdx.x;
    if (t >= n) return;
    int32_t i = dep == kDepLower ? t : n - 1 - t;
    int m = -1;
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
        int32_t j = col[k];
        if (dep == kDepLower ? j < i : j > i) m = max(m, wait_level(lev, j));
    }
    st_release(lev + i, m + 1);
}

__global__ void k_iota(int32_t* v, int32_t n) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

void level_sets(LevelSets& ls, int32_t n, const int32_t* d_rowptr, const int32_t* d_col, DepKind dep,
                cudaStream_t st) {
    ls.n = n;
    if (n == 0) return;
    int *lev, *ticket, *lev_sorted;
    int32_t* rows;
    PMG_CUDA(cudaMallocAsync(&lev, sizeof(int) * n, st));
    PMG_CUDA(cudaMallocAsync(&lev_sorted, sizeof(int) * n, st));
    PMG_CUDA(cudaMallocAsync(&rows, sizeof(int32_t) * n, st));
    PMG_CUDA(cudaMallocAsync(&ticket, sizeof(int), st));
    PMG_CUDA(cudaMallocAsync(&ls.order, sizeof(int32_t) * n, st));
    PMG_CUDA(cudaMemsetAsync(lev, 0xff, sizeof(int) * n, st));
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    k_levels<<<ceil_div(n, 256), 256, 0, st>>>(n, d_rowptr, d_col, dep, lev, ticket);
    PMG_LAUNCH_CHECK();
    k_iota<<<ceil_div(n, 256), 256, 0, st>>>(rows, n);
    PMG_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, lev, lev_sorted, rows, ls.order, n, 0, 32, st);
    void* tmp;
    PMG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, lev, lev_sorted, rows, ls.order, n, 0, 32, st);
    int last = 0;
    PMG_CUDA(cudaMemcpyAsync(&last, lev_sorted + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    ls.nlevels = last + 1;
    ls.level = lev;
    PMG_CUDA(cudaFreeAsync(tmp, st));
    PMG_CUDA(cudaFreeAsync(lev_sorted, st));
    PMG_CUDA(cudaFreeAsync(rows, st));
    PMG_CUDA(cudaFreeAsync(ticket, st));
}

void level_sets_free(LevelSets& ls) {
    cudaFree(ls.order);
    cudaFree(ls.level);
    ls = LevelSets{};
}

// ---------------------------------------------------------------- sweeps
__device__ __forceinline__ int take_ticket(int* ticket) {
    __shared__ int blk;
    if (threadIdx.x == 0) blk = atomicAdd(ticket, 1);
    __syncthreads();
    return blk;
}

// y_i = r[perm[i]] - sum_j l_ij y_j   (ascending)
__global__ void __launch_bounds__(256) k_lsolve(Sell L, const int32_t* __restrict__ perm, const double* __restrict__ r,
                                                double* y, int* ticket) {
    const int32_t pos = take_ticket(ticket) * 256 + threadIdx.x;
    if (pos >= L.n) return;
    const int32_t s = pos >> 5, lane = threadIdx.x & 31;
    const int64_t base = L.off[s];
    const int32_t len = L.len[pos];
    const int32_t i = L.row[pos];
    const int4* cp = reinterpret_cast<const int4*>(L.col + base) + lane;
    const double2* vp = reinterpret_cast<const double2*>(L.val + base) + lane;
    const double rhs = r[perm ? perm[i] : i];
    double acc = 0.0;
    for (int32_t k = 0; k < len; k += 4) {
        const int4 c = ld_stream_i4(cp + (k >> 2) * 32);
        const double2 v0 = ld_stream_d2(vp + (k >> 1) * 32);
        const double2 v1 = ld_stream_d2(vp + (k >> 1) * 32 + 32);
        acc = acc + v0.x * wait_value(y, c.x);
        if (k + 1 < len) acc = acc + v0.y * wait_value(y, c.y);
        if (k + 2 < len) acc = acc + v1.x * wait_value(y, c.z);
        if (k + 3 < len) acc = acc + v1.y * wait_value(y, c.w);
    }
    st_relaxed(y + i, rhs - acc);
}

// x_i = (y_i - sum_j u_ij x_j) * dinv_i  (descending j; dinv = 1.0/u_ii);  u[perm[i]] += x_i
__global__ void __launch_bounds__(256) k_usolve_add(Sell U, const double* __restrict__ diag,
                                                    const int32_t* __restrict__ perm, const double* __restrict__ y,
                                                    double* x, double* __restrict__ u, int* ticket) {
    const int32_t pos = take_ticket(ticket) * 256 + threadIdx.x;
    if (pos >= U.n) return;
    const int32_t s = pos >> 5, lane = threadIdx.x & 31;
    const int64_t base = U.off[s];
    const int32_t len = U.len[pos];
    const int32_t i = U.row[pos];
    const int4* cp = reinterpret_cast<const int4*>(U.col + base) + lane;
    const double2* vp = reinterpret_cast<const double2*>(U.val + base) + lane;
    double acc = 0.0;
    for (int32_t k = 0; k < len; k += 4) {
        const int4 c = ld_stream_i4(cp + (k >> 2) * 32);
        const double2 v0 = ld_stream_d2(vp + (k >> 1) * 32);
        const double2 v1 = ld_stream_d2(vp + (k >> 1) * 32 + 32);
        acc = acc + v0.x * wait_value(x, c.x);
        if (k + 1 < len) acc = acc + v0.y * wait_value(x, c.y);
        if (k + 2 < len) acc = acc + v1.x * wait_value(x, c.z);
        if (k + 3 < len) acc = acc + v1.y * wait_value(x, c.w);
    }
    const double xi = (y[i] - acc) * diag[pos];
    st_relaxed(x + i, xi);
    const int32_t ui = perm ? perm[i] : i;
    u[ui] = u[ui] + xi;
}

// Gauss-Seidel: lower entries read the new values (published by earlier rows), upper
// entries the old ones; u_new_i = ((f_i - S_L) - S_U) * dinv_i  (dinv = 1.0/a_ii)
__global__ void __launch_bounds__(256) k_gs(Sell A, const double* __restrict__ diag, const int32_t* __restrict__ nlow,
                                            const double* __restrict__ f, const double* __restrict__ u_old,
                                            double* u_new, int* ticket) {
    const int32_t pos = take_ticket(ticket) * 256 + threadIdx.x;
    if (pos >= A.n) return;
    const int32_t s = pos >> 5, lane = threadIdx.x & 31;
    const int64_t base = A.off[s];
    const int32_t len = A.len[pos], nl = nlow[pos];
    const int32_t i = A.row[pos];
    const int4* cp = reinterpret_cast<const int4*>(A.col + base) + lane;
    const double2* vp = reinterpret_cast<const double2*>(A.val + base) + lane;
    double sl = 0.0, su = 0.0;
    for (int32_t k = 0; k < len; k += 4) {
        const int4 c = ld_stream_i4(cp + (k >> 2) * 32);
        const double2 v0 = ld_stream_d2(vp + (k >> 1) * 32);
        const double2 v1 = ld_stream_d2(vp + (k >> 1) * 32 + 32);
        const int cc[4] = {c.x, c.y, c.z, c.w};
        const double vv[4] = {v0.x, v0.y, v1.x, v1.y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (k + q >= len) break;
            if (k + q < nl) sl = sl + vv[q] * wait_value(u_new, cc[q]);
            else su = su + vv[q] * __ldg(u_old + cc[q]);
        }
    }
    st_relaxed(u_new + i, ((f[i] - sl) - su) * diag[pos]);
}

__global__ void k_reciprocal(double* d, int32_t n) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = 1.0 / d[i];
}

void reciprocal_inplace(double* d, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_reciprocal<<<ceil_div(n, 256), 256, 0, st>>>(d, n);
    PMG_LAUNCH_CHECK();
}

void lsolve(const Sell& L, const int32_t* perm, const double* r, double* y, int* ticket, cudaStream_t st) {
    if (L.n == 0) return;
    fill_sentinel(y, L.n, st);
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    k_lsolve<<<ceil_div(L.n, 256), 256, 0, st>>>(L, perm, r, y, ticket);
    PMG_LAUNCH_CHECK();
}

void usolve_add(const Sell& U, const double* diag, const int32_t* perm, const double* y, double* x, double* u,
                int* ticket, cudaStream_t st) {
    if (U.n == 0) return;
    fill_sentinel(x, U.n, st);
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    k_usolve_add<<<ceil_div(U.n, 256), 256, 0, st>>>(U, diag, perm, y, x, u, ticket);
    PMG_LAUNCH_CHECK();
}

void gs_sweep(const Sell& A, const double* diag, const int32_t* nlow, const double* f, const double* u_old,
              double* u_new, int* ticket, cudaStream_t st) {
    if (A.n == 0) return;
    fill_sentinel(u_new, A.n, st);
    PMG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    k_gs<<<ceil_div(A.n, 256), 256, 0, st>>>(A, diag, nlow, f, u_old, u_new, ticket);
    PMG_LAUNCH_CHECK();
}

}  // namespace pmg
