// Rotating-lane wavefront sweeps for the triangular solves and Gauss-Seidel on tensor-grid
// orderings: the default sweep kernel for every factor whose rows
// fit a layout.  See wave.cu for the design; skew.cu / chain.cu / trsv.cu remain as fallbacks.
#pragma once

#include <vector>

#include "skew.cuh"

namespace pmg {

// Per-(block, step, lane) items (4 coefficients + 4 shared-memory byte offsets, 48 B) stored
// step-major per warp block; a CTA runs `w` consecutive blocks (one sweep warp each).
struct WavePlan {
    int32_t n = 0, seg = 0, nseg = 0;  // seg: longest segment
    int32_t* starts = nullptr;   // [nseg+1] first v-row of every segment (device)
    int32_t nr = 4, c = 3;       // lanes per segment, terms per lane and step
    int32_t spw = 8, w = 1;      // segments per warp block, warp blocks per CTA
    int32_t nblk = 0, ntask = 0; // warp blocks, CTA tasks
    int32_t dm = 1;              // segments back a term reaches (halo rings)
    int32_t ry = 256;            // ring rows per segment
    int64_t nsteps = 0;
    int32_t* Db = nullptr;       // [nblk] lane skew between a block's segments
    int32_t* Lb = nullptr;       // [nblk] lead over the previous block: before step t, prog(b-1) >= t + Lb
    int32_t* bp = nullptr;       // [nblk][w] ring back-pressure: before group q, prog(b+j) >= (q+1)G + bp
    int32_t* hoff = nullptr;     // [ntask][8] bridge: halo row counts -> virtual progress of the previous block
    int32_t* hrb = nullptr;      // [ntask][w][8] bridge: halo row j may be written iff j < prog(w) + hrb
    int32_t* hsl = nullptr;      // [ntask][8] bridge: halo row j goes to ring cell (j + hsl) mod ry
    unsigned sbase = 0;          // shared-window address of the kernel's dynamic shared memory
    int64_t* off = nullptr;      // [nblk+1] first step of each block in the item stream
    uint4* item = nullptr;       // [nsteps][3][32]
    int32_t lead = 0;            // median Lb (reporting)
    bool ok = false;
};

// Build the plan of the v-ordered matrix S (kinds and arguments as skew_plan); segments (grid
// rows, any lengths) are given by their first v-rows, starts.back() == n.  Returns false (nothing
// allocated) if a row does not fit the widest layout, reaches more than 8 segments back, or the
// rings do not fit shared memory.
bool wave_plan(const Sell& S, const double* dinv, const std::vector<int32_t>& starts, SkewKind kind,
               int32_t max_terms, WavePlan& plan, cudaStream_t st, const int32_t* nlow = nullptr);
std::vector<int32_t> uniform_starts(int32_t n, int32_t seg);
std::vector<int32_t> reversed_starts(const std::vector<int32_t>& starts);  // natural -> descending v-order
void wave_plan_free(WavePlan& plan);

struct WaveOp {
    SkewKind kind;
    const WavePlan* plan;
    const double* rhs;   // L: r; U: y; GS: f (natural order)
    double* out;         // v-space outputs (sentinel protocol between CTAs)
    double* upd;         // U: u[i] += x_i after the sweep
    const Sell* gsS = nullptr;  // Gauss-Seidel: upper sums over the old values (pre-pass)
    const int32_t* nlow = nullptr;
    const double* old = nullptr;
    double* su = nullptr;
    bool prepared = false;  // the caller filled `out` with sentinels and zeroed the ticket (wave_prepare2)
};

void wave_sweep(const WaveOp& op, int* ticket, cudaStream_t st);
// one launch in place of two sentinel fills and two ticket resets: prepares the outputs of the L
// and the U sweep of one ILUT application (their claim counters are ticket[0] and ticket[1])
void wave_prepare2(double* y, double* x, int32_t n, int* ticket, cudaStream_t st);

// diagnostics: one-shot trace of the next sweep, 4 u64 per warp block
// [globaltimer at step 0, at step 192, at the end, CTA task]
extern bool g_wave_trace_on;
extern bool g_wave_dump;              // keep a copy of each sweep's output (per kind)
extern double* g_wave_dump_buf[3];
extern int g_wave_dump_n[3];
extern unsigned long long* g_wave_trace;
extern int g_wave_trace_n;

}  // namespace pmg
