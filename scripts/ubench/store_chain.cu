// Microbenchmark: cost of one per-step global store inside a shuffle-chained FP64 recurrence
// (the chained-segment finisher's inner loop).  Build: nvcc -arch=sm_100a -O3 store_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, const double* vals, int steps, long long* cyc) {
    const int lane = threadIdx.x;
    double acc = lane * 1e-3, rhs = 1.0 + lane;
    long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
        const int f = t & 31;
        double y = 0;
        if (lane == f) {
            y = rhs - acc;
            if (MODE == 1) asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(out + t), "d"(y) : "memory");
            if (MODE == 2) out[t] = y;
            if (MODE == 3) asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(out + t), "d"(y));
            if (MODE == 4) asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(out + t), "d"(y));
        }
        y = __shfl_sync(0xffffffffu, y, f);
        acc = acc + vals[(t + lane) & 63] * y;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    double *out, *vals;
    long long* cyc;
    const int steps = 4096;
    cudaMalloc(&out, sizeof(double) * steps);
    cudaMalloc(&vals, sizeof(double) * 64);
    cudaMemset(vals, 0, sizeof(double) * 64);
    cudaMallocManaged(&cyc, sizeof(long long));
    const char* names[] = {"no store", "st.relaxed.gpu", "plain st", "st.cg", "st.volatile"};
    for (int rep = 0; rep < 2; ++rep)
        for (int m = 0; m < 5; ++m) {
            switch (m) {
                case 0: k<0><<<1, 32>>>(out, vals, steps, cyc); break;
                case 1: k<1><<<1, 32>>>(out, vals, steps, cyc); break;
                case 2: k<2><<<1, 32>>>(out, vals, steps, cyc); break;
                case 3: k<3><<<1, 32>>>(out, vals, steps, cyc); break;
                case 4: k<4><<<1, 32>>>(out, vals, steps, cyc); break;
            }
            cudaDeviceSynchronize();
            if (rep) printf("%-16s %7.1f cycles/step\n", names[m], double(cyc[0]) / steps);
        }
    return 0;
}
