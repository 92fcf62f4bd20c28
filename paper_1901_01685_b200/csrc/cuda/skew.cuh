// Skewed-warp wavefront sweeps for sparse triangular solves on tensor-grid orderings
// (rows of up to 125 terms reaching up to 8 grid rows back: every p-level of the configs).
#pragma once

#include "sell.cuh"

namespace pmg {

enum SkewKind : int { kSkewL = 0, kSkewU = 1, kSkewGS = 2 };

// The sweep kernel reads per-(step, lane) items (a lane's stage data, 48 B) stored step-major
// per warp block, [3 x 16-B chunks][32 lanes] per step, so one bulk copy moves a group of
// steps for the whole warp.  Block b's steps start at off[b].
struct SkewPlan {
    int32_t n = 0, seg = 0;
    int32_t D = 0;             // largest lane skew of a block (steps; reporting)
    int32_t lead = 0;          // typical lag between consecutive segments (reporting)
    int32_t dm = 1;            // segments back a term reaches
    int32_t ry = 64;           // ring length (rows) per segment in shared memory
    int32_t nr = 4, c = 3;     // lanes per segment (stages + 1), terms per lane and stage
    int32_t nseg = 0, nblk = 0;
    int64_t nsteps = 0;
    int32_t* Db = nullptr;     // [nblk] lane skew per block (the boundary blocks need more)
    int64_t* off = nullptr;    // [nblk+1] step offsets of the blocks in the item stream
    int32_t* R = nullptr;      // [nblk][8] lead a halo segment needs over the block's segment 0
    int32_t* W = nullptr;      // [nblk][8] read-behind window of the halo rings
    uint4* item = nullptr;     // [nsteps][3][32]
    // terms more than 8 segments back (patch interfaces): per block a table of those values,
    // copied once their last block is done
    int32_t* far_off = nullptr;  // [nblk+1]
    int32_t* far_idx = nullptr;  // sorted v-space rows per block
    int32_t* far_blk = nullptr;  // [nblk] block the last far value comes from (-1: none)
    int* done = nullptr;         // [nblk] finished blocks of the current sweep
    int32_t nfar_max = 0;
    bool ok = false;
};

// Build the step-major items of the v-ordered factor S (segment length seg; longest row
// max_terms off-diagonal terms) and choose the layout and the lane skew D.  Returns false
// (nothing allocated) when a row does not fit: more terms than the widest layout, an entry
// more than 8 segments back, a term whose value would not be final at its stage, or rings
// beyond shared memory.
// Gauss-Seidel (kind kSkewGS): S is the off-diagonal sliced matrix of the sweep (lower entries
// first, nlow[v] of them), dinv the reciprocal diagonal; the terms are the lower entries.
bool skew_plan(const Sell& S, const double* dinv, int32_t seg, SkewKind kind, int32_t max_terms, SkewPlan& plan,
               cudaStream_t st, const int32_t* nlow = nullptr);
void skew_plan_free(SkewPlan& plan);

struct SkewOp {
    SkewKind kind;
    const SkewPlan* plan;
    const double* rhs;   // L: r (natural order); U: y (natural order)
    double* out;         // v-space outputs (sentinel protocol across warp blocks)
    double* upd;         // U: u[i] += x_i after the sweep
    // Gauss-Seidel: u_new = ((f - S_L) - S_U) / a_ii with S_U over the old values, summed by a
    // pre-pass (same ascending order as the oracle) into su
    const Sell* gsS = nullptr;
    const int32_t* nlow = nullptr;
    const double* old = nullptr;
    double* su = nullptr;
};

void skew_sweep(const SkewOp& op, int* ticket, cudaStream_t st);

// diagnostics: one-shot trace of the next sweep, 4 u64 per warp block
// [claim globaltimer, end globaltimer, halo spins of lane 0, bridge empty polls]
extern bool g_skew_trace_on;
extern unsigned long long* g_skew_trace;
extern int g_skew_trace_n;

}  // namespace pmg
