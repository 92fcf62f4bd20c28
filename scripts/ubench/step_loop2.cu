// Microbenchmark: the chained-segment finisher's step loop as written in chain.cu, with
// optional sleeping "helper" warps polling a shared variable.
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int RS = 64, KIN = 40, RY = 256;
struct P { double* out; const int* gcol; const double* gval; int n; };

__device__ __forceinline__ void st_relaxed(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

template <int HELPERS, int VARIANT>
__global__ void k(P a, long long* cyc, int nsteps) {
    __shared__ double eval_[KIN][RS];
    __shared__ int ecol[KIN][RS];
    __shared__ double yring[RY];
    __shared__ int flag;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) flag = 0;
    for (int q = threadIdx.x; q < KIN * RS; q += blockDim.x) {
        const int r = q % RS, qq = q / RS;
        ecol[qq][r] = (r & 31) + 1 + qq * 2;  // consumed every 2 steps
        eval_[qq][r] = 1e-3;
    }
    __syncthreads();
    if (warp > 0) {
        if (HELPERS) {
            unsigned ns = 32;
            while (ld_vol(&flag) == 0) { __nanosleep(ns); ns = min(ns * 2, 256u); }
        }
        return;
    }
    const int hs = lane;
    double acc = lane * 1e-3, rhs = 1.0 + lane, dinv = 0.5;
    int pos = 0, cnt = 40, f0 = 3;
    const int v = lane;
    auto entry = [&](int q, int& c, double& w) {
        if (q < KIN) { c = ecol[q][hs]; w = eval_[q][hs]; }
        else { c = __ldg(a.gcol + f0 + q + v); w = __ldg(a.gval + f0 + q + v); }
        if (VARIANT == 1) c = a.n - 1 - c;
        if (VARIANT == 1) c = a.n - 1 - c;
    };
    int nc = INT_MAX; double nv = 0.0;
    if (pos < cnt) entry(pos, nc, nv);
    long long t0 = clock64();
    for (int t = 0; t < nsteps; ++t) {
        const int f = t & 31;
        double y = 0.0;
        if (lane == f) {
            y = (rhs - acc) * dinv;
            st_relaxed(a.out + t, y);
            yring[t & (RY - 1)] = y;
        }
        y = __shfl_sync(0xffffffffu, y, f);
        if (nc == t) {
            acc = acc + nv * y;
            ++pos;
            nc = INT_MAX;
            if (pos < cnt) entry(pos, nc, nv);
        }
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; flag = 1; }
    if (acc == 12345.0) a.out[0] = acc;
}

int main() {
    P a; long long* cyc;
    cudaMalloc(&a.out, sizeof(double) * 4096);
    cudaMalloc((void**)&a.gcol, sizeof(int) * 4096);
    cudaMalloc((void**)&a.gval, sizeof(double) * 4096);
    a.n = 1000000;
    cudaMallocManaged(&cyc, sizeof(long long));
    const int steps = 80;
    for (int rep = 0; rep < 2; ++rep) {
        k<0, 0><<<1, 32>>>(a, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("1 warp, L-like          %6.1f cyc/step\n", double(cyc[0]) / steps);
        k<0, 1><<<1, 32>>>(a, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("1 warp, U-like (vcol)   %6.1f cyc/step\n", double(cyc[0]) / steps);
        k<0, 0><<<1, 256>>>(a, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("8 warps, helpers exit   %6.1f cyc/step\n", double(cyc[0]) / steps);
        k<1, 0><<<1, 256>>>(a, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("8 warps, helpers sleep  %6.1f cyc/step\n", double(cyc[0]) / steps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
