// Chained-segment wavefront sweeps (L solve, U solve + update, Gauss-Seidel).
#pragma once

#include <vector>

#include "sell.cuh"

namespace pmg {

enum ChainKind : int { kChainL = 0, kChainU = 1, kChainGS = 2 };

constexpr int kChainMaxInSeg = 128;  // in-segment entries per row the finisher stages in shared memory
constexpr int kChainRing = 1024;     // rows of finalised outputs kept on chip (in-segment reach bound)

struct ChainOp {
    ChainKind kind;
    const Sell* S;             // v-ordered rows (L: identity; U: reversed, off-diag desc; GS: identity, off-diag)
    const double* diag;        // per v (U, GS)
    const int32_t* nlow;       // GS: # lower entries per row
    const int32_t* split;      // per v: # leading entries in earlier segments (chain_split)
    const int32_t* perm;       // L: rhs = r[perm[v]]; U: u[perm[i]] += x  (null = identity)
    const double* rhs;         // L: r; U: y (natural); GS: f
    const double* old;         // GS: u_old
    double* out;               // v-space outputs with sentinel protocol (L: y, U: x_v, GS: u_new)
    double* upd;               // U: u (updated by a separate pass after the sweep)
    int32_t seg;               // segment length (rows)
    int32_t bs = 32;           // finisher batch: smaller for short-reach factors (lag ~ bs + reach)
    int32_t start_gap = 0;     // rows of the predecessor segment needed before a segment starts (0: default)
};

// per-factor chain plan: start gate (forward reach into the previous segment), and whether
// every row fits the kernel's on-chip buffers (in-segment entries <= kChainMaxInSeg, backward
// in-segment reach <= kChainRing); ok = false -> use the level-scheduled sweeps
struct ChainPlan {
    int32_t gap = 0, max_in = 0, max_back = 0;
    bool ok = false;
};
ChainPlan chain_plan(const Sell& S, const int32_t* nlow, const int32_t* split, int32_t seg, ChainKind kind,
                     cudaStream_t st);

// per-row split point between earlier-segment entries and in-segment entries
void chain_split(const Sell& S, const int32_t* nlow, int32_t seg, ChainKind kind, int32_t* split, cudaStream_t st);

// diagnostics: globaltimer trace of the first sweep after enabling: 6 u64 per segment
// [claim, helpers done, fin start, fin end, helper spins, finisher waits], then for segments
// 7 and 8: 64 batches x [start, hdr ok, catch-up start, steps start, end], then 1024 rows x
// [helper row start, prefix published]
constexpr int kChainTraceExtra = 2 * 64 * 5 + 2 * 2048 + 64;  // + per-chunk stamps of one helper row
extern bool g_chain_trace_on;
extern unsigned long long* g_chain_trace;
extern size_t g_chain_trace_cap;
extern int g_chain_trace_n;

// one sweep; `ticket` is scratch (2 ints).  out[] is filled with sentinels first.
void chain_sweep(const ChainOp& op, int* ticket, cudaStream_t st);

// grid-row length of a tensor-product natural ordering detected from the sparsity pattern of
// the middle row (distance between the starts of consecutive column runs); 0 if none found
int32_t detect_segment(int32_t n, const int32_t* h_rowptr, const int32_t* h_col);
std::vector<int32_t> detect_segment_starts(int32_t n, const int32_t* h_rowptr, const int32_t* h_col);

}  // namespace pmg
