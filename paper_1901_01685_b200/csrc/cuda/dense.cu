// Dense LU (partial pivoting) for the coarsest h-level (h = 2^-2: 25 DOFs single patch,
// 65 for the 3-patch L-shape) -- SPEC.md:390-391, SURVEY K11.  Factorised once at setup
// and applied every cycle on the device; loop orders are the oracle's (first maximal
// pivot; l = a_ik/a_kk; a_ij -= l a_kj; ascending forward/backward sums).
#include "dense.cuh"

namespace pmg {

__global__ void k_dense_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const double* __restrict__ v, double* __restrict__ a) {
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) a[t] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int k = rp[i]; k < rp[i + 1]; ++k) a[i * n + ci[k]] = v[k];
}

__global__ void k_dense_factor(int n, double* a, int* piv, int* err) {
    if (threadIdx.x != 0) return;
    *err = -1;
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (fabs(a[i * n + k]) > fabs(a[p * n + k])) p = i;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) {
                double t = a[k * n + j];
                a[k * n + j] = a[p * n + j];
                a[p * n + j] = t;
            }
        if (a[k * n + k] == 0.0) {
            *err = k;
            return;
        }
        for (int i = k + 1; i < n; ++i) {
            double l = a[i * n + k] / a[k * n + k];
            a[i * n + k] = l;
            for (int j = k + 1; j < n; ++j) a[i * n + j] = a[i * n + j] - l * a[k * n + j];
        }
    }
}

// x = U^{-1} L^{-1} P b.  One warp: lane i owns rows i, i+32, ...; the sums of every row
// are still accumulated one term at a time in ascending column order as soon as the term's
// unknown is final (column-oriented sweep), i.e. exactly the oracle's sequential sums.
__global__ void k_dense_solve(int n, const double* __restrict__ a, const int* __restrict__ piv,
                              const double* __restrict__ b, double* __restrict__ x) {
    extern __shared__ double sy[];
    double* y = sy;
    double* s = sy + n;
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < n; ++i) y[i] = b[i];
        for (int k = 0; k < n; ++k) {
            double t = y[k];
            y[k] = y[piv[k]];
            y[piv[k]] = t;
        }
    }
    for (int i = lane; i < n; i += 32) s[i] = 0.0;
    __syncwarp();
    // forward: y_i = y_i - sum_{j<i} l_ij y_j
    for (int j = 0; j < n; ++j) {
        if (lane == (j & 31)) y[j] = y[j] - s[j];
        __syncwarp();
        const double yj = y[j];
        for (int i = lane; i < n; i += 32)
            if (i > j) s[i] = s[i] + a[i * n + j] * yj;
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) s[i] = 0.0;
    __syncwarp();
    // backward: x_i = (y_i - sum_{j>i} u_ij x_j) / u_ii with the sum ascending in j:
    // row i's sum needs x_{i+1} first, so it is accumulated after all x_j (j > i) are known
    // -- done by the owning lane sequentially once they are final.
    for (int i = n - 1; i >= 0; --i) {
        if (lane == 0) {
            double acc = 0.0;
            for (int j = i + 1; j < n; ++j) acc = acc + a[i * n + j] * x[j];
            x[i] = (y[i] - acc) / a[i * n + i];
        }
        __syncwarp();
    }
}

int dense_setup(DenseLU& D, const DevCsr& A, cudaStream_t st) {
    D.n = A.n;
    PMG_CUDA(cudaMalloc(&D.a, sizeof(double) * size_t(D.n) * D.n));
    PMG_CUDA(cudaMalloc(&D.piv, sizeof(int) * (D.n + 1)));
    k_dense_fill<<<1, 256, 0, st>>>(D.n, A.rowptr, A.col, A.val, D.a);
    PMG_LAUNCH_CHECK();
    k_dense_factor<<<1, 32, 0, st>>>(D.n, D.a, D.piv, D.piv + D.n);
    PMG_LAUNCH_CHECK();
    int err = -1;
    PMG_CUDA(cudaMemcpyAsync(&err, D.piv + D.n, sizeof(int), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    return err;
}

void dense_solve(const DenseLU& D, const double* b, double* x, cudaStream_t st) {
    k_dense_solve<<<1, 32, sizeof(double) * 2 * D.n, st>>>(D.n, D.a, D.piv, b, x);
    PMG_LAUNCH_CHECK();
}

void dense_free(DenseLU& D) {
    cudaFree(D.a);
    cudaFree(D.piv);
    D = DenseLU{};
}

}  // namespace pmg
