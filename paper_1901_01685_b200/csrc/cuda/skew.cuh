// Skewed-warp wavefront sweeps (short rows, short reach: the p=1 h-levels).
#pragma once

#include "sell.cuh"

namespace pmg {

enum SkewKind : int { kSkewL = 0, kSkewU = 1 };

struct SkewPlan {
    int D = 0, rb = 0, reach = 0;
    bool ok = false;
};

// Decide whether the v-ordered factor S (segment length seg) fits the skewed-warp kernel
// (rows of at most 32 entries, at most 2 segments back, rings of 64 suffice) and compute D.
bool skew_plan(const Sell& S, int32_t seg, SkewKind kind, int32_t max_row, SkewPlan& plan, cudaStream_t st);

struct SkewOp {
    SkewKind kind;
    const Sell* S;
    const double* dinv;  // U: reciprocal diagonal per v
    const int32_t* perm;
    const double* rhs;   // L: r (natural, gathered through perm); U: y (natural)
    double* out;         // v-space outputs (sentinel protocol)
    double* upd;         // U: u[perm[i]] += x_i
    int32_t seg, D;
};

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st);

}  // namespace pmg
