// Microbenchmark of the chained-segment finisher step (variants) -- cycles per step.
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>

template <int DIV, int CONSUME_EVERY>
__global__ void k(double* out, long long* cyc, int steps) {
    __shared__ int ecol[32][48];
    __shared__ double eval_[32][48];
    __shared__ double yring[256];
    const int lane = threadIdx.x;
    for (int q = 0; q < 48; ++q) {
        ecol[lane][q] = lane + 1 + q * CONSUME_EVERY;   // entry consumed every CONSUME_EVERY steps
        eval_[lane][q] = 1e-3 * (q + 1);
    }
    __syncwarp();
    double acc = lane * 1e-3, rhs = 1.0 + lane, dg = 2.0 + lane;
    int pos = 0, cnt = 48;
    int nc = ecol[lane][0];
    double nv = eval_[lane][0];
    long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
        const int f = t & 31;
        double y = 0.0;
        if (lane == f) {
            y = DIV ? (rhs - acc) / dg : rhs - acc;
            asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(out + t), "d"(y) : "memory");
            yring[t & 255] = y;
        }
        y = __shfl_sync(0xffffffffu, y, f);
        if (nc == t) {
            acc = acc + nv * y;
            ++pos;
            nc = INT_MAX;
            if (pos < cnt) {
                nc = ecol[lane][pos];
                nv = eval_[lane][pos];
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    double* out;
    long long* cyc;
    const int steps = 4096;
    cudaMalloc(&out, sizeof(double) * steps);
    cudaMallocManaged(&cyc, sizeof(long long));
    for (int rep = 0; rep < 2; ++rep) {
        k<0, 1><<<1, 32>>>(out, cyc, 40); cudaDeviceSynchronize();
        if (rep) printf("no-div consume-every-1   %7.1f cyc/step (40 steps)\n", double(cyc[0]) / 40);
        k<0, 1><<<1, 32>>>(out, cyc, 48); cudaDeviceSynchronize();
        k<0, 8><<<1, 32>>>(out, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("no-div consume-every-8   %7.1f cyc/step\n", double(cyc[0]) / steps);
        k<1, 8><<<1, 32>>>(out, cyc, steps); cudaDeviceSynchronize();
        if (rep) printf("div    consume-every-8   %7.1f cyc/step\n", double(cyc[0]) / steps);
        k<1, 1><<<1, 32>>>(out, cyc, 48); cudaDeviceSynchronize();
        if (rep) printf("div    consume-every-1   %7.1f cyc/step (48 steps)\n", double(cyc[0]) / 48);
    }
    return 0;
}
