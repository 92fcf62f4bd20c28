// Microbenchmark: one-way latency of handing a double from one SM to another through global memory
// with the sweeps' protocol -- the producer stores the value (plain / st.global.cg / st.relaxed.gpu),
// the consumer polls it with ld.relaxed.gpu against a NaN sentinel -- measured as half a ping-pong
// round trip between two CTAs.  Bounds the cross-CTA hand-over of wave.cu from below.
// Build: nvcc -arch=sm_100a -O3 handover.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
template <int MODE>
__device__ __forceinline__ void st(double* p, double v) {
    if (MODE == 0) *reinterpret_cast<volatile double*>(p) = v;
    if (MODE == 1) asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
    if (MODE == 2) asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// CTA 0 writes a[i], CTA 1 answers in b[i]; one thread each; cells start as NaN
template <int MODE>
__global__ void k(double* a, double* b, int n, long long* cyc, unsigned* smid) {
    if (threadIdx.x != 0) return;
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    smid[blockIdx.x] = id;
    long long t0 = clock64();
    if (blockIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            st<MODE>(a + i, double(i));
            while (ld_relaxed(b + i) != ld_relaxed(b + i)) {
            }
        }
    } else {
        for (int i = 0; i < n; ++i) {
            while (ld_relaxed(a + i) != ld_relaxed(a + i)) {
            }
            st<MODE>(b + i, double(i));
        }
    }
    cyc[blockIdx.x] = clock64() - t0;
}

// The same hand-over when the producer does nothing but shared-memory work after the store (as a
// sweep warp does): the producer stores one value every `gap_ns`, timestamps in shared memory;
// the consumer polls and timestamps the arrival (%globaltimer on both sides).
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int MODE>
__global__ void k_oneway(double* a, int n, unsigned gap_ns, unsigned long long* t_send, unsigned long long* t_recv) {
    __shared__ unsigned long long ts[2048];
    if (threadIdx.x != 0) return;
    if (blockIdx.x == 0) {
        unsigned long long next = gtime() + 20000;
        for (int i = 0; i < n; ++i) {
            while (gtime() < next) {
            }
            ts[i] = gtime();
            st<MODE>(a + i, double(i));
            next += gap_ns;
        }
        for (int i = 0; i < n; ++i) t_send[i] = ts[i];
    } else {
        for (int i = 0; i < n; ++i) {
            while (ld_relaxed(a + i) != ld_relaxed(a + i)) {
            }
            ts[i] = gtime();
        }
        for (int i = 0; i < n; ++i) t_recv[i] = ts[i];
    }
}
template <int MODE>
void run_oneway(const char* name, unsigned gap_ns) {
    const int n = 2000;
    double* a;
    unsigned long long *ts, *tr;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&ts, n * 8);
    cudaMalloc(&tr, n * 8);
    cudaMemset(a, 0xff, n * 8);
    k_oneway<MODE><<<2, 32>>>(a, n, gap_ns, ts, tr);
    static unsigned long long hs[2000], hr[2000];
    cudaMemcpy(hs, ts, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hr, tr, n * 8, cudaMemcpyDeviceToHost);
    double sum = 0, mx = 0;
    for (int i = 100; i < n; ++i) {
        const double d = double(hr[i]) - double(hs[i]);
        sum += d;
        if (d > mx) mx = d;
    }
    printf("%-16s one store per %u ns, producer idle otherwise: store -> seen %.0f ns mean, %.0f ns max\n", name, gap_ns,
           sum / (n - 100), mx);
    cudaFree(a); cudaFree(ts); cudaFree(tr);
}

// ping-pong between block 0 and block `partner` of a grid with one block per SM: the hand-over
// latency as a function of where the two SMs sit (same TPC / GPC / die or not)
__global__ void k_pair(double* a, double* b, int n, int partner, long long* cyc, unsigned* smid) {
    if (threadIdx.x != 0) return;
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (blockIdx.x == 0) {
        smid[0] = id;
        long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            st<0>(a + i, double(i));
            while (ld_relaxed(b + i) != ld_relaxed(b + i)) {
            }
        }
        cyc[0] = clock64() - t0;
    } else if (int(blockIdx.x) == partner) {
        smid[1] = id;
        for (int i = 0; i < n; ++i) {
            while (ld_relaxed(a + i) != ld_relaxed(a + i)) {
            }
            st<0>(b + i, double(i));
        }
    }
}
void run_pairs() {
    const int n = 5000;
    double *a, *b;
    long long* cyc;
    unsigned* smid;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMalloc(&cyc, 16);
    cudaMalloc(&smid, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int partner = 1; partner < nsm; partner += (partner < 8 ? 1 : 9)) {
        cudaMemset(a, 0xff, n * 8);
        cudaMemset(b, 0xff, n * 8);
        k_pair<<<nsm, 32>>>(a, b, n, partner, cyc, smid);
        long long h;
        unsigned s[2];
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(s, smid, 8, cudaMemcpyDeviceToHost);
        printf("pair block 0 / %3d on SMs %3u / %3u: one way %.0f cycles\n", partner, s[0], s[1], double(h) / n / 2);
    }
    cudaFree(a); cudaFree(b); cudaFree(cyc); cudaFree(smid);
}

template <int MODE>
void run(const char* name) {
    const int n = 20000;
    double *a, *b;
    long long* cyc;
    unsigned* smid;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMalloc(&cyc, 16);
    cudaMalloc(&smid, 8);
    cudaMemset(a, 0xff, n * 8);
    cudaMemset(b, 0xff, n * 8);
    k<MODE><<<2, 32>>>(a, b, n, cyc, smid);
    long long h[2];
    unsigned s[2];
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(s, smid, 8, cudaMemcpyDeviceToHost);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-16s SMs %u/%u: round trip %.0f cycles, one way %.0f cycles = %.0f ns at %d MHz\n", name, s[0], s[1],
           double(h[0]) / n, double(h[0]) / n / 2, double(h[0]) / n / 2 / (clk * 1e-6), clk / 1000);
    cudaFree(a); cudaFree(b); cudaFree(cyc); cudaFree(smid);
}

int main() {
    run<0>("volatile store");
    run<1>("st.global.cg");
    run<2>("st.relaxed.gpu");
    run_oneway<0>("volatile store", 2000);
    run_oneway<2>("st.relaxed.gpu", 2000);
    run_pairs();
    return 0;
}
