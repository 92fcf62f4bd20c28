// Does prefetch.global.L2 (or cp.async.bulk.prefetch.L2) land a line in L2?  Load latency of
// random DRAM lines: cold, after prefetch.global.L2, after a bulk L2 prefetch (cycles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ldnc(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

__global__ void probe(const uint64_t* a, size_t nlines, int mode, int iters, long long* out) {
    long long tot = 0;
    uint64_t sink = 0;
    for (int it = 0; it < iters; ++it) {
        const size_t line = hsh(it * 7919 + mode * 1000003ull + 12345) % nlines;
        const uint64_t* p = a + line * 16;
        if (mode == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
        if (mode == 2) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" ::"l"(p) : "memory");
        if (mode == 3) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p) : "memory");
        long long w = clock64();
        while (clock64() - w < 8000) {}
        long long t0 = clock64();
        sink += ldnc(p + (sink & 1));
        long long t1 = clock64();
        tot += t1 - t0;
    }
    out[0] = tot / iters;
    out[1] = sink;
}

int main() {
    const size_t bytes = size_t(2) << 30;  // 2 GB: far beyond L2
    uint64_t* a;
    long long* o;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    cudaMalloc(&o, 16);
    const char* names[] = {"cold", "prefetch.global.L2", "cp.async.bulk.prefetch.L2", "prefetch.L2::evict_last"};
    for (int m = 0; m < 4; ++m) {
        probe<<<1, 1>>>(a, bytes / 128, m, 2000, o);
        long long h[2];
        cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("%-28s %6lld cycles\n", names[m], h[0]);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
