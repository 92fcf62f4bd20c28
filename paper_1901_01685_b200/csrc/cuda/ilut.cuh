// Device CSR and the GPU ILUT factorisation entry point.
#pragma once

#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace pmg {

struct DevCsr {
    int32_t n = 0, m = 0;
    int64_t nnz = 0;
    int32_t* rowptr = nullptr;
    int32_t* col = nullptr;
    double* val = nullptr;
    void free() {
        cudaFree(rowptr);
        cudaFree(col);
        cudaFree(val);
        rowptr = col = nullptr;
        val = nullptr;
    }
};

// ILUT(tau, fillfactor) of the (already permuted) matrix A with bandwidth `band`.
// On success L (strictly lower, unit diagonal implicit) and U (diag first, then ascending
// off-diagonals) are allocated.  Returns 0, or 1 (zero pivot, *err_row = first failing row).
int ilut_factorize_device(const DevCsr& A, int32_t band, double tau, double fillfactor, DevCsr& L, DevCsr& U,
                          int64_t* err_row, double* seconds, cudaStream_t st);

// The same in two steps, so that independent factorisations overlap: ilut_launch enqueues the
// work on `st` (grid capped at max_ctas, 0 = no cap) and returns; ilut_finish waits, compacts the
// rows into L and U and frees the job.
struct IlutJob;
IlutJob* ilut_launch(const DevCsr& A, int32_t band, double tau, double fillfactor, int max_ctas, cudaStream_t st);
// `seconds`: the factorisation kernel; `seconds_since_ref`: from the event `ref` (recorded by the
// caller before the first of several concurrent launches) to the end of this kernel
int ilut_finish(IlutJob* job, DevCsr& L, DevCsr& U, int64_t* err_row, double* seconds, cudaEvent_t ref,
                double* seconds_since_ref);

}  // namespace pmg
