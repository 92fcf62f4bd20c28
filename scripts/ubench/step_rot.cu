// Microbenchmark: the step of a "rotating-lane" wavefront sweep (one warp, synthetic data).
// Lane = row (mod NR): a row's partial sum never leaves its lane; the only cross-lane traffic
// per step is one shuffle broadcasting the value finalised at the previous step.  Terms are
// read from a shared-memory ring one step ahead (their values are final two steps before use)
// except a stage's last term when it is the previous step's value (the broadcast).  Items
// (4 coefficients + 4 shared-memory byte addresses) come from a shared-memory ring two steps
// ahead.  Prints cycles per step for the 32x4 (p=5), 8x4 (p=2) and 4x3 (p=1) layouts, with
// (V=1) and without (V=0) the finalised-value stores.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int RY = 128;   // ring rows per segment
constexpr int NS = 16;    // item ring steps
constexpr unsigned FULL = 0xffffffffu;

struct __align__(16) Item {
    double w[4];
    uint32_t o[4];  // shared-memory byte addresses of the terms' values
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ double lds(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int ld_vol(unsigned a) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol(unsigned a, int v) {
    asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int wait_ge(unsigned addr, int pv, int need) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "L:\n\tsetp.ge.s32 p, %0, %2;\n\t@p bra.uni D;\n\t"
        "ld.volatile.shared.b32 %0, [%1];\n\tbra.uni L;\n"
        "D:\n\t}"
        : "+r"(pv)
        : "r"(addr), "r"(need)
        : "memory");
    return pv;
}
__device__ __forceinline__ void sts_if(unsigned a, double v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f64 [%0], %1;\n\t}" ::"r"(a), "d"(v),
                 "r"(int(p)));
}
__device__ __forceinline__ void stg_if(double* a, double v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.relaxed.gpu.global.f64 [%0], %1;\n\t}" ::"l"(a),
                 "d"(v), "r"(int(p)));
}

template <int NR, int C, int U, int V, bool UPPER>
__global__ void k(const Item* gitems, double* out, long long* cyc, int steps) {
    constexpr int SPW = 32 / NR, P = NR - 1;
    __shared__ __align__(16) Item items[NS][32];
    __shared__ double Y[(SPW + 4) * (RY + 1) + 64];
    __shared__ double rhs[NS][SPW];
    const int lane = threadIdx.x;
    const int kseg = lane / NR, rl = lane % NR;
    const unsigned ybase = smem_u32(Y);
    for (int i = lane; i < NS * 32; i += 32) {
        Item it = gitems[i];
        if (V == 9) for (int q = 0; q < 4; ++q) it.o[q] = uint32_t(-(RY + 1) * (q % 3) + ((i % 32) * 16 + q) % RY);
        for (int q = 0; q < 4; ++q) it.o[q] = ybase + 8 * ((4 + (i % 32) / NR) * (RY + 1) + it.o[q]);
        items[i / 32][i % 32] = it;
    }
    for (int i = lane; i < (SPW + 4) * (RY + 1); i += 32) Y[i] = 1e-3 * (i % 97);
    for (int i = lane; i < NS * SPW; i += 32) rhs[i / SPW][i % SPW] = 1.0 + i;
    __syncwarp();
    const int D = 3;
    const unsigned ring = ybase + 8 * (4 + kseg) * (RY + 1);
    const unsigned xbcell = ring + 8 * RY;
    double* Yd = Y;
    const unsigned dummy = ybase + 8 * ((SPW + 4) * (RY + 1) + lane);  // items address the broadcast value through this cell
    const int phase = (rl + P + D * kseg) % NR;   // this lane finalises at step t <=> t % NR == phase
    const int gbase = kseg * NR, c0 = (2 * NR - P - D * kseg % NR) % NR;
    double acc = 0.0, x = 0.0;
    Item cur = items[1][lane], nxt;
    double yc[4], w[4];
    {
        const Item i0 = items[0][lane];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            yc[q] = lds(i0.o[q]);
            w[q] = i0.w[q];
        }
    }
    unsigned o3 = items[0][lane].o[3];
    double rh = rhs[0][kseg];
    double* og = out + 1024 * kseg;
    __shared__ int prog[4];
    const unsigned progaddr = smem_u32(prog);
    if (lane == 0) prog[0] = 0;
    __syncwarp();
    int pv = 0;
    long long t0 = clock64();
    for (int tb = 0; tb < steps; tb += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = tb + u;
            if (V >= 8) {
                pv = wait_ge(progaddr, pv, t - 5);
                pv = ld_vol(progaddr);
            }
            const int fsrc = gbase + ((c0 + u + NR - 1) & (NR - 1));  // finaliser of step t-1
            const double xb = __shfl_sync(FULL, x, fsrc);
            double yn[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) yn[q] = lds(cur.o[q]);
            nxt = items[(t + 2) % NS][lane];
            const double rhn = rhs[(t + 1) % NS][kseg];
            const double y3 = o3 == xbcell ? xb : yc[3];
            double a = acc;
            if (C == 4) a = a + w[0] * yc[0];
            a = a + w[1] * yc[1];
            a = a + w[2] * yc[2];
            a = a + w[3] * y3;
            const bool fin = (u % NR) == phase;
            x = UPPER ? (rh - a) * w[0] : rh - a;  // stage 0: w[0] holds 1/diagonal, its value cell is zero
            if (V == 1) {
                sts_if(ring + 8 * ((t - P) & (RY - 1)), x, fin);
                stg_if(og + ((t - P) & 1023), x, fin);
            } else if (V == 2) {
                sts_if(ring + 8 * ((t - P) & (RY - 1)), x, fin);
            } else if (V == 3) {
                if (fin) og[(t - P) & 1023] = x;
            } else if (V == 4) {
                if (fin) og[(t - P) & 1023] = x;
                if (fin) Yd[(ring - ybase) / 8 + ((t - P) & (RY - 1))] = x;
            } else if (V == 5) {
                const unsigned a = fin ? ring + 8 * ((t - P) & (RY - 1)) : dummy;
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x));
                stg_if(og + ((t - P) & 1023), x, fin);
            } else if (V == 6) {
                const unsigned a = fin ? ring + 8 * ((t - P) & (RY - 1)) : dummy;
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x));
                if (fin) og[(t - P) & 1023] = x;
            } else if (V == 8 || V == 9) {
                if (fin) og[(t - P) & 1023] = x;
                if (fin) Yd[(ring - ybase) / 8 + ((t - P) & (RY - 1))] = x;
            } else if (V == 7) {
                const unsigned a = fin ? ring + 8 * ((t - P) & (RY - 1)) : dummy;
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x));
            }
            acc = fin ? 0.0 : a;
            if (V >= 8) st_vol(progaddr, t + 1);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                yc[q] = yn[q];
                w[q] = cur.w[q];
            }
            o3 = cur.o[3];
            rh = rhn;
            cur = nxt;
        }
    }
    long long t1 = clock64();
    out[4096 + lane] = acc + x;
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    Item h[NS * 32];
    for (int s = 0; s < NS; ++s)
        for (int l = 0; l < 32; ++l) {
            Item& it = h[s * 32 + l];
            for (int q = 0; q < 4; ++q) {
                it.w[q] = 1e-3 * (q + 1);
                // element offsets relative to the lane's ring (negative: earlier segments)
                it.o[q] = uint32_t(-(RY + 1) * (q % 3) + ((s * 7 + l * 3 + q * 5) % RY));
            }
            if ((s + l) % 3 == 0) it.o[3] = RY;  // the broadcast
        }
    Item* d;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    double* o;
    long long* c;
    cudaMalloc(&o, 8 * 8192);
    cudaMallocManaged(&c, 256);
    const int steps = 32 * 4000;
    for (int rep = 0; rep < 2; ++rep) {
        k<32, 4, 32, 1, false><<<1, 32>>>(d, o, c + 0, steps);
        k<32, 4, 32, 1, true><<<1, 32>>>(d, o, c + 1, steps);
        k<32, 4, 32, 0, false><<<1, 32>>>(d, o, c + 2, steps);
        k<8, 4, 32, 1, false><<<1, 32>>>(d, o, c + 3, steps);
        k<4, 3, 32, 1, false><<<1, 32>>>(d, o, c + 4, steps);
        k<4, 3, 32, 1, true><<<1, 32>>>(d, o, c + 5, steps);
        k<32, 4, 32, 2, false><<<1, 32>>>(d, o, c + 6, steps);
        k<32, 4, 32, 3, false><<<1, 32>>>(d, o, c + 7, steps);
        k<32, 4, 32, 4, false><<<1, 32>>>(d, o, c + 8, steps);
        k<32, 4, 32, 5, false><<<1, 32>>>(d, o, c + 9, steps);
        k<32, 4, 32, 6, false><<<1, 32>>>(d, o, c + 10, steps);
        k<32, 4, 32, 7, false><<<1, 32>>>(d, o, c + 11, steps);
        k<32, 4, 32, 8, false><<<1, 32>>>(d, o, c + 12, steps);
        k<32, 4, 32, 9, false><<<1, 32>>>(d, o, c + 13, steps);
        k<32, 4, 32, 8, true><<<1, 32>>>(d, o, c + 14, steps);
        cudaDeviceSynchronize();
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    printf("cycles/step: 32x4 L %.1f | 32x4 U %.1f | 32x4 L no stores %.1f | 8x4 L %.1f | 4x3 L %.1f | 4x3 U %.1f\n",
           c[0] / double(steps), c[1] / double(steps), c[2] / double(steps), c[3] / double(steps),
           c[4] / double(steps), c[5] / double(steps));
    printf("32x4 L: V2 sts_if %.1f | V3 if-stg weak %.1f | V4 if both %.1f | V5 sel-sts+stg_if %.1f | V6 sel-sts+if-stg %.1f | V7 sel-sts only %.1f\n",
           c[6] / double(steps), c[7] / double(steps), c[8] / double(steps), c[9] / double(steps), c[10] / double(steps), c[11] / double(steps));
    printf("32x4: V8 = V4 + progress check/publish %.1f | V9 = V8 + 16-way-ish conflicts %.1f | V8 U %.1f\n",
           c[12] / double(steps), c[13] / double(steps), c[14] / double(steps));
    return 0;
}
