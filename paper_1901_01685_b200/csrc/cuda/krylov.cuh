// BiCGSTAB vector updates, each with the oracle's fixed operation order
// (oracle/oracle.cpp bicgstab) and no multiply-add contraction.
#pragma once

#include "common.cuh"

namespace pmg {

// p = r + beta * (p - omega * v)
void bicg_update_p(double* p, const double* r, const double* v, double beta, double omega, int32_t n, cudaStream_t st);
// s = r - alpha * v
void bicg_update_s(double* s, const double* r, const double* v, double alpha, int32_t n, cudaStream_t st);
// u = (u + alpha * ph) + omega * sh;  r = s - omega * t
void bicg_update_ur(double* u, double* r, const double* s, const double* t, const double* ph, const double* sh,
                    double alpha, double omega, int32_t n, cudaStream_t st);

// u = u + e (the p = 1-only hierarchy's h-MG correction)
void vec_add(double* u, const double* e, int32_t n, cudaStream_t st);

}  // namespace pmg
