// Skewed-warp wavefront sweeps for factors with short rows and short reach (the p=1
// h-levels: <= 9 off-diagonal entries per row, reach one grid row back).
#pragma once

#include "sell.cuh"

namespace pmg {

enum SkewKind : int { kSkewL = 0, kSkewU = 1 };

// Per-row record, staged to shared memory with cp.async (7 x 16 B).  The row's terms are
// pre-assigned to pipeline stages: stage s (s = kSkewP..1) is accumulated s steps before the
// row is finalised, kSkewC terms per stage, in the oracle's ascending order; stage 0 is the
// single v-1 term, taken from a register.  Padding slots have coef 0 and point at a zero cell.
constexpr int kSkewP = 3;
constexpr int kSkewC = 3;
constexpr int kSkewSlots = kSkewP * kSkewC + 1;
struct __align__(16) SkewRec {
    double coef[kSkewSlots];       // slots [0,C): stage P ... [(P-1)C, PC): stage 1; slot PC: stage 0
    int32_t off[kSkewSlots - 1];   // byte offset of the term's value relative to the lane's ring
    int32_t has0;                  // slot PC holds the v-1 term (taken from a register)
    double dinv;                   // U: reciprocal diagonal
};
static_assert(sizeof(SkewRec) == 128, "SkewRec layout");

// The sweep kernel reads per-(step, lane) items (a lane's stage data, 48 B) stored step-major
// per 8-segment warp block, [3 x 16-B chunks][32 lanes] per step, so one bulk copy moves a
// group of steps for the whole warp.  Block b starts at step offset b * ns_full.
struct SkewPlan {
    int32_t n = 0, seg = 0, D = 0, b1 = 1;  // b1: how far behind its row a term one segment back may lie
    int32_t nseg = 0, nblk = 0, ns_full = 0, ns_last = 0;
    uint4* item = nullptr;     // [(nblk-1)*ns_full + ns_last][3][32]
    bool ok = false;
};

// Build the records of the v-ordered factor S (segment length seg) and the lane skew D.
// Returns false (plan.ok = false, nothing allocated) when a row does not fit: more than
// kSkewSlots terms, an entry more than one segment back, or a term whose value would not be
// ready at its stage.
bool skew_plan(const Sell& S, const double* dinv, int32_t seg, SkewKind kind, SkewPlan& plan, cudaStream_t st);
void skew_plan_free(SkewPlan& plan);

struct SkewOp {
    SkewKind kind;
    const SkewPlan* plan;
    const double* rhs;   // L: r (natural order); U: y (natural order)
    double* out;         // v-space outputs (sentinel protocol across warp blocks)
    double* upd;         // U: u[i] += x_i after the sweep
};

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st);

// diagnostics: one-shot trace of the next sweep, 4 u64 per warp block
// [claim globaltimer, end globaltimer, halo spins of lane 0, bridge empty polls]
extern bool g_skew_trace_on;
extern unsigned long long* g_skew_trace;
extern int g_skew_trace_n;

}  // namespace pmg
