// Sliced-ELL (SELL-32) device layout and the SpMV-family kernels.
//
// Layout: rows are grouped in slices of 32 consecutive *positions* (one row per lane);
// every slice stores len_s = roundup4(max row length in the slice) entries per lane,
// interleaved so that a lane fetches its k..k+3 columns with one 128-bit load and its
// values two at a time with 128-bit loads:
//     col(k, lane) at off_s + (k/4)*128 + 4*lane + k%4
//     val(k, lane) at off_s + (k/2)*64  + 2*lane + k%2
// A warp's loads are therefore fully coalesced (512 B per instruction) while each lane
// walks ITS row sequentially in stored order -- which is what keeps every row sum in
// the oracle's ascending order (bit-exact parity).  Padding entries are
// never accumulated (per-row length predicate).
#pragma once

#include "common.cuh"

namespace pmg {

struct Sell {
    int32_t n = 0;            // positions (rows)
    int32_t nslices = 0;
    int64_t* off = nullptr;   // [nslices+1] entry offsets
    int32_t* len = nullptr;   // [n] stored entries of the row at each position
    int32_t* row = nullptr;   // [n] row id at each position (nullptr: identity)
    int32_t* col = nullptr;
    double* val = nullptr;
    int64_t entries = 0;      // allocated (padded) entries
    int64_t nnz = 0;          // real entries
};

// which entries of a CSR row go into the sliced layout
enum SellPick : int {
    kPickAll = 0,         // ascending
    kPickOffDiagDesc = 1, // off-diagonal only, descending column (U solve order)
    kPickOffDiag = 2,     // off-diagonal only, ascending (Gauss-Seidel)
};

// Build a sliced copy of a device CSR.  `order` (device, may be null) maps position ->
// row.  Aux outputs (may be null): diag[pos] = a_ii, nlow[pos] = #entries with j < i.
void sell_build(Sell& S, int32_t nrows, const int32_t* d_rowptr, const int32_t* d_col, const double* d_val,
                const int32_t* d_order, SellPick pick, double* d_diag, int32_t* d_nlow, cudaStream_t st);
void sell_free(Sell& S);

enum RowOp : int {
    kOpSpmv = 0,        // y = A x
    kOpResidual = 1,    // y = f - A x   (+ fused canonical norm when norm_out != null)
    kOpRestrict = 2,    // y = (A x) / ml          (lumped-L2 restriction)
    kOpProlongAdd = 3,  // y = y + (A x) / ml      (lumped-L2 prolongation)
    kOpAdd = 4,         // y = y + A x             (h-MG prolongation)
};

struct NormCtx {
    double* partials = nullptr;   // [nblocks]
    unsigned int* counter = nullptr;
    double* norm_out = nullptr;   // ||y||_2
    const double* n0 = nullptr;   // if set: hist_out = norm / *n0
    double* hist_out = nullptr;
    bool raw = false;             // write the canonical sum itself (a dot product), no sqrt
};

void sell_rowop(const Sell& S, RowOp op, const double* x, const double* f, const double* ml, double* y,
                const NormCtx* norm, cudaStream_t st);

// canonical norm of a plain vector (same reduction tree as the fused residual norm)
void vec_norm(const double* v, int32_t n, const NormCtx& ctx, cudaStream_t st);
// canonical dot product (x, y): the same tree over the products x_i * y_i (ctx.raw forced)
void vec_dot(const double* x, const double* y, int32_t n, NormCtx ctx, cudaStream_t st);

void fill_value(double* v, int64_t n, double value_bits_as_double, cudaStream_t st);

// every sweep receives `ticket`: ticket[0] is the CTA claim counter, ticket[1 .. kSweepScratchInts)
// per-sweep scratch (segment progress / finished blocks) owned by the caller's work object, so
// concurrent solves on one hierarchy never share it
constexpr int kSweepScratchInts = 1 << 17;
void fill_sentinel(double* v, int64_t n, cudaStream_t st);

}  // namespace pmg
