// BiCGSTAB vector updates: HBM-bound elementwise kernels, 128-bit loads and stores.
#include <algorithm>

#include "krylov.cuh"

namespace pmg {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int32_t n) { return std::max(1, std::min(ceil_div(n, 2 * kThreads), 148 * 16)); }

// two elements per thread per step; n odd leaves one scalar tail element
__global__ void __launch_bounds__(kThreads) k_update_p(double* __restrict__ p, const double* __restrict__ r,
                                                       const double* __restrict__ v, double beta, double omega,
                                                       int32_t n) {
    const int32_t n2 = n >> 1;
    for (int32_t i = blockIdx.x * kThreads + threadIdx.x; i < n2; i += gridDim.x * kThreads) {
        double2 pp = reinterpret_cast<double2*>(p)[i];
        const double2 rr = reinterpret_cast<const double2*>(r)[i];
        const double2 vv = reinterpret_cast<const double2*>(v)[i];
        pp.x = rr.x + beta * (pp.x - omega * vv.x);
        pp.y = rr.y + beta * (pp.y - omega * vv.y);
        reinterpret_cast<double2*>(p)[i] = pp;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = r[n - 1] + beta * (p[n - 1] - omega * v[n - 1]);
}

__global__ void __launch_bounds__(kThreads) k_update_s(double* __restrict__ s, const double* __restrict__ r,
                                                       const double* __restrict__ v, double alpha, int32_t n) {
    const int32_t n2 = n >> 1;
    for (int32_t i = blockIdx.x * kThreads + threadIdx.x; i < n2; i += gridDim.x * kThreads) {
        const double2 rr = reinterpret_cast<const double2*>(r)[i];
        const double2 vv = reinterpret_cast<const double2*>(v)[i];
        reinterpret_cast<double2*>(s)[i] = make_double2(rr.x - alpha * vv.x, rr.y - alpha * vv.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) s[n - 1] = r[n - 1] - alpha * v[n - 1];
}

__global__ void __launch_bounds__(kThreads) k_update_ur(double* __restrict__ u, double* __restrict__ r,
                                                        const double* __restrict__ s, const double* __restrict__ t,
                                                        const double* __restrict__ ph, const double* __restrict__ sh,
                                                        double alpha, double omega, int32_t n) {
    const int32_t n2 = n >> 1;
    for (int32_t i = blockIdx.x * kThreads + threadIdx.x; i < n2; i += gridDim.x * kThreads) {
        double2 uu = reinterpret_cast<double2*>(u)[i];
        const double2 a = reinterpret_cast<const double2*>(ph)[i];
        const double2 b = reinterpret_cast<const double2*>(sh)[i];
        const double2 ss = reinterpret_cast<const double2*>(s)[i];
        const double2 tt = reinterpret_cast<const double2*>(t)[i];
        uu.x = (uu.x + alpha * a.x) + omega * b.x;
        uu.y = (uu.y + alpha * a.y) + omega * b.y;
        reinterpret_cast<double2*>(u)[i] = uu;
        reinterpret_cast<double2*>(r)[i] = make_double2(ss.x - omega * tt.x, ss.y - omega * tt.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int32_t i = n - 1;
        u[i] = (u[i] + alpha * ph[i]) + omega * sh[i];
        r[i] = s[i] - omega * t[i];
    }
}

__global__ void __launch_bounds__(kThreads) k_vec_add(double* __restrict__ u, const double* __restrict__ e, int32_t n) {
    for (int32_t i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) u[i] = u[i] + e[i];
}

}  // namespace

void vec_add(double* u, const double* e, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_vec_add<<<grid_for(n), kThreads, 0, st>>>(u, e, n);
    PMG_LAUNCH_CHECK();
}

void bicg_update_p(double* p, const double* r, const double* v, double beta, double omega, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_update_p<<<grid_for(n), kThreads, 0, st>>>(p, r, v, beta, omega, n);
    PMG_LAUNCH_CHECK();
}
void bicg_update_s(double* s, const double* r, const double* v, double alpha, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_update_s<<<grid_for(n), kThreads, 0, st>>>(s, r, v, alpha, n);
    PMG_LAUNCH_CHECK();
}
void bicg_update_ur(double* u, double* r, const double* s, const double* t, const double* ph, const double* sh,
                    double alpha, double omega, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_update_ur<<<grid_for(n), kThreads, 0, st>>>(u, r, s, t, ph, sh, alpha, omega, n);
    PMG_LAUNCH_CHECK();
}

}  // namespace pmg
