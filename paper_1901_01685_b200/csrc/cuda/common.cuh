// Shared device helpers for libpmg_cuda (sm_100a, FP64, built with -fmad=false).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace pmg {

struct CudaError : std::runtime_error {
    int status;
    CudaError(const std::string& m, int s) : std::runtime_error(m), status(s) {}
};

#define PMG_CUDA(call)                                                                                        \
    do {                                                                                                      \
        cudaError_t e_ = (call);                                                                              \
        if (e_ != cudaSuccess)                                                                                \
            throw ::pmg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_),                        \
                                   e_ == cudaErrorMemoryAllocation ? 5 /*PMG_ERR_OOM*/ : 4 /*PMG_ERR_CUDA*/); \
    } while (0)

#define PMG_LAUNCH_CHECK() PMG_CUDA(cudaGetLastError())

constexpr int kSlice = 32;   // SELL slice height = warp width (one row per lane)
constexpr int kChunk = 256;  // norm / residual block: 8 slices, the canonical norm chunk

// "not yet produced" marker for sync-free solves: a NaN payload no arithmetic produces
constexpr unsigned long long kSentinelBits = 0xFFF4DEAD0BADF00Dull;

__device__ __forceinline__ double sentinel() { return __longlong_as_double((long long)kSentinelBits); }
__device__ __forceinline__ bool is_sentinel(double v) {
    return (unsigned long long)__double_as_longlong(v) == kSentinelBits;
}

// coherent (L2) load / store of a value produced by another thread during this kernel
__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
// same load without a compiler memory barrier: lets independent loads be batched
__device__ __forceinline__ double ld_relaxed_nb(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// predicated relaxed store without a compiler barrier: publishes one lane's value from
// branch-free code (consumers poll each element individually, so no ordering is needed)
__device__ __forceinline__ void st_relaxed_if(double* p, double v, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.relaxed.gpu.global.f64 [%0], %1;\n\t}" ::"l"(p),
        "d"(v), "r"(int(pred)));
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// spin until another thread has published x[j]
__device__ __forceinline__ double wait_value(const double* x, int j) {
    double v = ld_relaxed(x + j);
    while (is_sentinel(v)) {
        __nanosleep(20);
        v = ld_relaxed(x + j);
    }
    return v;
}

// streaming 128-bit loads of matrix data (read once per sweep)
#ifndef PMG_SELL_LD
#define PMG_SELL_LD 0
#endif
#if PMG_SELL_LD == 0
#define PMG_SELL_QUAL "ld.global.nc.L1::no_allocate"
#elif PMG_SELL_LD == 1
#define PMG_SELL_QUAL "ld.global.cg"
#else
#define PMG_SELL_QUAL "ld.global"
#endif
__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
    int4 r;
    asm volatile(PMG_SELL_QUAL ".v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p) {
    double2 r;
    asm volatile(PMG_SELL_QUAL ".v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// canonical xor-butterfly over a warp (offsets 16,8,4,2,1); every lane ends with the sum
__device__ __forceinline__ double warp_butterfly(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

// integer tuning switch from the environment (read by callers into function-local statics,
// whose initialisation is thread-safe)
inline int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// SM count of the current device (cached, thread-safe)
inline int sm_count() {
    static const int n = [] {
        int dev = 0, v = 0;
        PMG_CUDA(cudaGetDevice(&dev));
        PMG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

}  // namespace pmg
