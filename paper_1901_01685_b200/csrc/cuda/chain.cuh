// Chained-segment wavefront sweeps (L solve, U solve + update, Gauss-Seidel).
#pragma once

#include "sell.cuh"

namespace pmg {

enum ChainKind : int { kChainL = 0, kChainU = 1, kChainGS = 2 };

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
    double* upd;               // U: u
    int32_t seg;               // segment length (rows)
    int32_t bs = 32;           // finisher batch: smaller for short-reach factors (lag ~ bs + reach)
    int32_t start_gap = 0;     // rows of the predecessor segment needed before a segment starts (0: default)
};

// data-driven start gate: max over rows of the last previous-segment row they reference, + 1
int32_t chain_start_gap(const Sell& S, const int32_t* split, int32_t seg, ChainKind kind, cudaStream_t st);

// per-row split point between earlier-segment entries and in-segment entries
void chain_split(const Sell& S, const int32_t* nlow, int32_t seg, ChainKind kind, int32_t* split, cudaStream_t st);

// diagnostics: per-segment globaltimer trace of the most recent sweep
extern bool g_chain_trace_on;
extern unsigned long long* g_chain_trace;
extern size_t g_chain_trace_cap;
extern int g_chain_trace_n;

// one sweep; `ticket` is scratch (2 ints).  out[] is filled with sentinels first.
void chain_sweep(const ChainOp& op, int* ticket, cudaStream_t st);

// grid-row length of a tensor-product natural ordering detected from the sparsity pattern of
// the middle row (distance between the starts of consecutive column runs); 0 if none found
int32_t detect_segment(int32_t n, const int32_t* h_rowptr, const int32_t* h_col);

}  // namespace pmg
