// Microbenchmark: dependent-chain latencies on sm_100a (cycles per op): DADD, DMUL, FSEL pair
// (double select), SHFL of a double, LDS.64.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
    __shared__ double S[64];
    const int lane = threadIdx.x;
    S[lane] = lane; S[lane + 32] = 0;
    __syncwarp();
    double x = lane * 1e-3, y = 1.0 + lane;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + a;  // DADD chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) y = y * b;  // DMUL chain
    long long t2 = clock64();
    bool p = lane & 1;
    for (int i = 0; i < n; ++i) { x = p ? x + 0.0 : y; p = !p; }  // (DADD? ) select chain
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    long long t4 = clock64();
    int idx = lane;
    for (int i = 0; i < n; ++i) { double v = S[idx]; idx = (int(v) + 1) & 31; }
    long long t5 = clock64();
    out[lane] = x + y + idx;
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
    const int n = 4096;
    for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, n, 1e-9, 1.0000001); cudaDeviceSynchronize(); }
    printf("cycles/op: DADD %.1f DMUL %.1f sel-loop %.1f SHFL(f64) %.1f LDS.64+cvt+and %.1f\n", c[0] / double(n),
           c[1] / double(n), c[2] / double(n), c[3] / double(n), c[4] / double(n));
    return 0;
}
