// Microbenchmark: a triangular-sweep segment split into a FINISHER warp and accumulator warp(s)
// (synthetic data, one segment).  The finisher owns the recurrence: x_v = rh_v - ((((p_v + a x_{v-4})
// + b x_{v-3}) + c x_{v-2}) + d x_{v-1}) with the last four outputs in registers (chain per row:
// DMUL -> DADD -> DADD, ~24 cycles).  The accumulators sum every other term of row v (p_v, the
// oracle's order: they are the row's earlier columns) from a shared-memory ring of finished values
// and hand p_v over through shared memory.  NA accumulator warps split the rows by parity.
// Prints cycles per row.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int RING = 256;
constexpr int NSTEP = 16;  // item ring steps

struct __align__(16) Item {
    double w[4];
    uint32_t o[4];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ double lds(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int ld_acq(unsigned a) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol(unsigned a, int v) {
    asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int wait_ge(unsigned addr, int pv, int need) {
    while (pv < need) pv = ld_acq(addr);
    return pv;
}

template <int NA, int CA>
__global__ void k(const Item* gitems, double* out, long long* cyc, int rows) {
    __shared__ __align__(16) Item items[NSTEP][32];  // shared by the accumulators (timing only)
    __shared__ double xr[RING + 1], pre[RING], rhs[RING];
    __shared__ int progF, progA[NA];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < NSTEP * 32; i += blockDim.x) {
        Item it = gitems[i % (NSTEP * 32)];
        for (int q = 0; q < 4; ++q) it.o[q] = smem_u32(xr) + 8 * (it.o[q] % RING);
        (&items[0][0])[i] = it;
    }
    for (int i = threadIdx.x; i < RING; i += blockDim.x) { xr[i] = 1e-3 * i; pre[i] = 0; rhs[i] = 1.0 + i; }
    if (threadIdx.x == 0) { progF = 0; for (int a = 0; a < NA; ++a) progA[a] = 0; }
    __syncthreads();
    const unsigned sF = smem_u32(&progF);
    long long t0 = clock64();
    if (warp == NA) {
        // ---------------- finisher: one row per iteration, chain DMUL -> DADD -> DADD
        double x1 = 0, x2 = 0, x3 = 0, x4 = 0;
        const double a = 1e-3, b = 2e-3, c = 3e-3, d = 4e-3;
        int pa[NA];
        for (int q = 0; q < NA; ++q) pa[q] = 0;
        for (int v = 0; v < rows; v += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = v + u;
                const int q = r % NA;
                pa[q] = wait_ge(smem_u32(&progA[q]), pa[q], r / NA + 1);  // partial of row r is in
                const double p = pre[r & (RING - 1)];
                const double rh = rhs[r & (RING - 1)];
                const double s = (((p + a * x4) + b * x3) + c * x2) + d * x1;
                const double x = rh - s;
                if (lane == 0) xr[r & (RING - 1)] = x;
                x4 = x3; x3 = x2; x2 = x1; x1 = x;
            }
            st_vol(sF, v + 4);
        }
        if (lane == 0) out[0] = x1;
    } else {
        // ---------------- accumulator warp `warp`: rows r = NA*j + warp, lane = j mod 32 owns
        // the row for 32 steps, CA terms per step (loaded a step ahead from the x ring); the
        // row's values must be older than r-4 (the finisher's own terms)
        const int me = warp;
        double acc = 0.0;
        int pf = 0;
        Item cur = items[0][lane];
        double yc[4];
        for (int q = 0; q < 4; ++q) yc[q] = lds(cur.o[q]);
        Item nxt = items[1][lane];
        for (int j0 = 0; j0 < rows / NA; j0 += 32) {
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const int j = j0 + u;           // step: lane (j mod 32) finishes row NA*j + me
                const int need = NA * (j + 1) + me - 5;  // values up to row NA*(j+1)+me-5 are read next step
                if ((u & 1) == 0) pf = wait_ge(sF, pf, need + NA);
                double yn[4];
#pragma unroll
                for (int q = 4 - CA; q < 4; ++q) yn[q] = lds(nxt.o[q]);
                Item nn = items[(j + 2) % NSTEP][lane];
                double r = acc;
#pragma unroll
                for (int q = 4 - CA; q < 4; ++q) r = r + cur.w[q] * yc[q];
                const bool last = lane == u;  // the lane whose row completes at this step
                if (last) pre[(NA * j + me) & (RING - 1)] = r;
                acc = last ? 0.0 : r;
                if ((u & 1) == 1) st_vol(smem_u32(&progA[me]), j + 1);
#pragma unroll
                for (int q = 0; q < 4; ++q) yc[q] = yn[q];
                cur = nxt;
                nxt = nn;
            }
        }
        out[1 + me * 32 + lane] = acc;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[warp] = t1 - t0;
}

int main(int argc, char** argv) {
    const int na = argc > 1 ? atoi(argv[1]) : 1;
    static Item h[NSTEP * 32];
    for (int s = 0; s < NSTEP; ++s)
        for (int l = 0; l < 32; ++l)
            for (int q = 0; q < 4; ++q) {
                h[s * 32 + l].w[q] = 1e-4 * (q + 1);
                h[s * 32 + l].o[q] = (s * 7 + l * 3 + q * 5) % RING;
            }
    Item* d;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    double* o;
    long long* c;
    cudaMalloc(&o, 8 * 4096);
    cudaMallocManaged(&c, 64);
    const int rows = 32 * 2048 * 6;
    for (int rep = 0; rep < 2; ++rep) {
        if (na == 1) k<1, 4><<<1, 64>>>(d, o, c, rows);
        if (na == 2) k<2, 4><<<1, 96>>>(d, o, c, rows);
        if (na == 3) k<3, 4><<<1, 128>>>(d, o, c, rows);
        cudaDeviceSynchronize();
    }
    printf("NA=%d CA=4: finisher %.1f cycles/row, accumulator 0 %.1f  err=%s\n", na, c[na] / double(rows),
           c[0] / double(rows), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
