// Level sets and level-scheduled sync-free sweeps: ILUT forward/backward substitution
// and lexicographic Gauss-Seidel.
#pragma once

#include "sell.cuh"

namespace pmg {

enum DepKind : int { kDepLower = 0, kDepUpper = 1 };

struct LevelSets {
    int32_t n = 0;
    int32_t nlevels = 0;
    int32_t* order = nullptr;  // [n] rows sorted by (level, row)
    int32_t* level = nullptr;  // [n] level of each row
};

// level[i] = 1 + max(level[j]) over the dependencies of row i (j < i for kDepLower,
// j > i for kDepUpper) -- computed on the device, then rows bucketed by level (stable).
void level_sets(LevelSets& ls, int32_t n, const int32_t* d_rowptr, const int32_t* d_col, DepKind dep,
                cudaStream_t st);
void level_sets_free(LevelSets& ls);

// d[i] = 1.0 / d[i] (IEEE): the U / GS sweeps multiply by reciprocal diagonals
void reciprocal_inplace(double* d, int32_t n, cudaStream_t st);

// y = L^{-1} r[perm]   (unit lower, L rows in level order, ascending accumulation)
void lsolve(const Sell& L, const int32_t* perm, const double* r, double* y, int* ticket, cudaStream_t st);
// x = U^{-1} y; u[perm[i]] += x_i   (U off-diagonals descending, diag per position)
void usolve_add(const Sell& U, const double* diag, const int32_t* perm, const double* y, double* x, double* u,
                int* ticket, cudaStream_t st);
// u_new_i = ((f_i - S_L(u_new)) - S_U(u_old)) / a_ii   (rows in level order of tril(A))
void gs_sweep(const Sell& A, const double* diag, const int32_t* nlow, const double* f, const double* u_old,
              double* u_new, int* ticket, cudaStream_t st);

}  // namespace pmg
