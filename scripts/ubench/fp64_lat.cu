// Microbenchmark: dependent FP64 add / mul latency and dependent shared-load latency for one warp
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
    __shared__ int idx[1024];
    __shared__ double vals[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { idx[i] = (i * 7 + 1) & 1023; vals[i] = i; }
    __syncthreads();
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = x + b; x = x + b; x = x + b; x = x + b; }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) { x = x * b; x = x * b; x = x * b; x = x * b; }
    long long t2 = clock64();
    int j = threadIdx.x;
    for (int i = 0; i < iters; ++i) { j = idx[j]; j = idx[j]; j = idx[j]; j = idx[j]; }
    long long t3 = clock64();
    double y = 0;
    for (int i = 0; i < iters; ++i) { y = y + vals[(j + i) & 1023]; j = idx[j]; }  // LDS -> DADD
    long long t4 = clock64();
    out[threadIdx.x] = x + j + y;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 64);
    int it = 4096;
    k<<<1, 32>>>(o, c, 1.0, 1.0000001, it);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 1.0000001, it);
    cudaDeviceSynchronize();
    printf("DADD dep latency %.1f cyc, DMUL %.1f, LDS(int) chain %.1f, LDS->DADD iter %.1f\n", c[0] / (4.0 * it),
           c[1] / (4.0 * it), c[2] / (4.0 * it), c[3] / double(it));
    return 0;
}
