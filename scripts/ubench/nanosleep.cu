// Actual duration of __nanosleep(t) on this GPU (cycles per call), alone and with 8 warps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned t, int reps, long long* out) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) __nanosleep(t);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}
int main() {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    unsigned ts[] = {32, 128, 512, 1024, 4096, 16384, 100000};
    for (unsigned t : ts) {
        for (int thr : {1, 256}) {
            k<<<1, thr>>>(t, 200, d);
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("nanosleep(%6u) threads %3d: %8lld cycles (%.0f ns at 1.965 GHz)\n", t, thr, h, h / 1.965);
        }
    }
    return 0;
}
