// Microbenchmark: the skew sweep's per-step dependency structure in isolation (one warp):
// (a) shfl.down of a double + 4 dependent DADDs (the partial-sum hand-off), (b) the same plus
// __syncwarp, 4 shared loads, 4 DMULs feeding the adds, (c) (b) plus the stage-0 STS that the
// next step's loads read.  Prints cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(double* out, long long* cyc, int steps) {
    __shared__ double Y[32 * 65];
    const int lane = threadIdx.x;
    for (int i = lane; i < 32 * 65; i += 32) Y[i] = 1e-3 * i;
    __syncwarp();
    double res = lane, xprev = 1.0;
    const int o0 = (lane * 7) % 64, o1 = (lane * 11) % 64, o2 = (lane * 13) % 64, o3 = (lane * 17) % 64;
    const double w0 = 1e-3, w1 = 2e-3, w2 = 3e-3, w3 = 4e-3;
    long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
        const double in = __shfl_down_sync(0xffffffffu, res, 1);
        double p0 = w0, p1 = w1, p2 = w2, p3 = w3;
        if (V >= 1) {
            __syncwarp();
            const double* Yb = Y + lane * 65;
            p0 = w0 * Yb[o0]; p1 = w1 * Yb[o1]; p2 = w2 * Yb[o2]; p3 = w3 * Yb[o3];
        }
        const double r1 = in + p0;
        res = ((r1 + p1) + p2) + p3;
        const double x = 1.0 - r1;
        if (V >= 2) Y[lane * 65 + (t & 63)] = x;
        xprev = x;
    }
    long long t1 = clock64();
    out[lane] = res + xprev;
    if (lane == 0) cyc[V] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMallocManaged(&c, 64);
    const int steps = 10000;
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(o, c, steps); k<1><<<1, 32>>>(o, c, steps); k<2><<<1, 32>>>(o, c, steps);
        cudaDeviceSynchronize();
    }
    printf("cycles/step: shfl+4dadd %.1f | +syncwarp+4lds+4dmul %.1f | +sts %.1f\n", c[0] / double(steps),
           c[1] / double(steps), c[2] / double(steps));
    return 0;
}
