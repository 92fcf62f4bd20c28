// Dependent-load latency by PTX load flavour (pointer chase through an L2-resident array).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int M>
__device__ __forceinline__ uint64_t ld(const uint64_t* p) {
    uint64_t v;
    if (M == 0) asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (M == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (M == 2) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (M == 3) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (M == 4) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

template <int M>
__global__ void chase(const uint64_t* a, int hops, uint64_t* out, long long* cyc) {
    uint64_t i = 0;
    for (int h = 0; h < 64; ++h) i = ld<M>(a + i);  // warm
    long long t0 = clock64();
    for (int h = 0; h < hops; ++h) i = ld<M>(a + i);
    long long t1 = clock64();
    out[0] = i;
    cyc[0] = t1 - t0;
}

int main() {
    const size_t n = (8u << 20) / 8;  // 8 MB: L2-resident, not L1
    std::vector<uint64_t> h(n);
    std::vector<uint64_t> perm(n / 16);
    for (size_t k = 0; k < perm.size(); ++k) perm[k] = k * 16;  // one element per 128-B line
    std::mt19937_64 rng(1);
    std::shuffle(perm.begin(), perm.end(), rng);
    for (size_t k = 0; k < perm.size(); ++k) h[perm[k]] = perm[(k + 1) % perm.size()];
    uint64_t *d, *o;
    long long* c;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 8);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    // touch everything once so it sits in L2
    const int hops = 20000;
    const char* names[] = {"ld.ca", "ld.cg", "ld.relaxed.gpu", "ld.volatile", "ld.acquire.gpu", "ld.nc.no_alloc"};
    for (int m = 0; m < 6; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (m) {
                case 0: chase<0><<<1, 1>>>(d, hops, o, c); break;
                case 1: chase<1><<<1, 1>>>(d, hops, o, c); break;
                case 2: chase<2><<<1, 1>>>(d, hops, o, c); break;
                case 3: chase<3><<<1, 1>>>(d, hops, o, c); break;
                case 4: chase<4><<<1, 1>>>(d, hops, o, c); break;
                case 5: chase<5><<<1, 1>>>(d, hops, o, c); break;
            }
            long long cy;
            cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-16s %7.1f cycles/hop\n", names[m], double(cy) / hops);
        }
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sm clock attr %d kHz; err=%s\n", clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
