#pragma once

#include "ilut.cuh"

namespace pmg {

struct DenseLU {
    int n = 0;
    double* a = nullptr;  // row-major LU, unit-lower L below the diagonal
    int* piv = nullptr;   // [n] pivot rows (+1 slot for the error flag)
};

int dense_setup(DenseLU& D, const DevCsr& A, cudaStream_t st);  // returns -1 or the zero-pivot step
void dense_solve(const DenseLU& D, const double* b, double* x, cudaStream_t st);
void dense_free(DenseLU& D);

}  // namespace pmg
