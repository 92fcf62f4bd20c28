// GPU ILUT(tau, m) factorisation -- row-parallel IKJ elimination, bit-identical to the
// oracle.
//
// Persistent CTAs claim rows in ascending order through an atomic ticket.  A CTA keeps the
// working row dense over the band window [i-b, i+b] (b = bandwidth of the permuted matrix;
// LU fill never leaves the band) in shared memory, with two bitmaps: `pres` (structurally
// present entries) and `piv` (pending L-part pivots).  Pivots are taken in ascending
// column order; before using U row k the CTA waits for row k's `done` flag (release /
// acquire), so the elimination follows the dynamic dependency DAG of the factorisation
// ("row-parallel elimination over the L-dependency levels").  Row i publishes U first
// (it gates later rows) and selects its L part afterwards.
//
// Per-row arithmetic and dropping are exactly the oracle's:
//   w_k = w_k / u_kk ; |w_k| < tau_i -> drop ; else w_j = w_j - w_k * u_kj   (ascending k)
//   U entries |w_j| < tau_i dropped; rule 2 keeps the M largest (|v| desc, col asc) in L and U.
// Top-M selection is a block-wide MSD radix select on the |v| bit patterns (exact: the
// kept set under a strict total order is unique, so any exact selection matches).
#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <vector>

#include "ilut.cuh"

namespace pmg {

namespace {

constexpr int kThreads = 256;
constexpr unsigned FULL = 0xffffffffu;
// candidates of a selection are also kept in shared memory when they fit (the selection after the
// last pivot is on the row-to-row critical path: no L2 round trips there)
constexpr int kCandSh = 1024;
// up to this many candidates the selection is by ranks (one barrier round: the p = 1 factors);
// larger sets use the block-wide radix select (ranks cost C^2 comparisons: ~1000 candidates per row
// of the p = 5 factor took 58 us against 4.7 us)
constexpr int kCandRank = 128;

struct IlutDev {
    int32_t n, M, b, W, nwords;
    const int32_t* rp;
    const int32_t* ci;
    const double* v;
    const double* tau;
    int32_t* Ucol;
    double* Uval;
    int32_t* Ulen;
    int32_t* Lcol;
    double* Lval;
    int32_t* Llen;
    int* done;
    int* ticket;
    int* err_row;
    double* gw;          // [slots * W] work rows when they do not fit in shared memory
    int32_t* gcand_col;  // [slots * W]
    double* gcand_val;
    int smem_w;
    unsigned long long* trace;  // PMG_ILUT_TRACE: 6 timestamps for kTraceRows rows from trace_row0 on
    int32_t trace_row0;
};
constexpr int kTraceRows = 4096;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define ILUT_STAMP(slot)                                                                   \
    do {                                                                                   \
        if (d.trace && threadIdx.x == 0 && i >= d.trace_row0 && i < d.trace_row0 + kTraceRows) \
            d.trace[size_t(i - d.trace_row0) * 6 + (slot)] = gtime();                      \
    } while (0)

__device__ __forceinline__ uint64_t absbits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7FFFFFFFFFFFFFFFull;
}

__device__ __forceinline__ int block_scan_excl(int v, int* sh, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const int c = sh[w];
        if (w < wid) base += c;
        tot += c;
    }
    __syncthreads();  // sh is reused by the next scan
    total = tot;
    return base + x - v;
}

// gather the band entries [lo, hi) that are present (and, if filter, |w| >= tau) into the
// candidate arrays in ascending order; returns the count.  Lane = entry of a 32-entry word:
// the kept mask of every word by ballot (words interleaved over the warps), an exclusive scan of the
// word counts, then every kept entry is written at its rank -- no per-thread serial bit loops.
__device__ int gather(const double* w, const uint32_t* pres, uint32_t* kmask, int32_t* woff, int32_t* wlist, int lo, int hi,
                      bool filter, double tau, int col0, int32_t* ccol, double* cval, int32_t* scol, double* sval, int* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int w0 = lo >> 5, w1 = (hi + 31) >> 5;
    auto word = [&](int wi) {
        uint32_t bits = pres[wi];
        if (wi == (lo >> 5)) bits &= FULL << (lo & 31);
        if (wi == ((hi - 1) >> 5) && (hi & 31)) bits &= FULL >> (32 - (hi & 31));
        return bits;
    };
    // the non-empty words, ascending (the band window is mostly empty)
    int nlist = 0;
    for (int wb = w0; wb < w1; wb += kThreads) {
        const int wi = wb + threadIdx.x;
        const bool nz = wi < w1 && word(wi) != 0u;
        int tot;
        const int o = block_scan_excl(nz ? 1 : 0, sh, tot) + nlist;
        if (nz) wlist[o] = wi;
        nlist += tot;
    }
    __syncthreads();
    for (int e = wid; e < nlist; e += kThreads / 32) {
        const int wi = wlist[e];
        uint32_t bits = word(wi);
        if (filter) {
            const bool keep = ((bits >> lane) & 1u) && !(fabs(w[wi * 32 + lane]) < tau);
            bits = __ballot_sync(FULL, keep);
        }
        if (lane == 0) kmask[e] = bits;
    }
    __syncthreads();
    int base = 0;
    for (int eb = 0; eb < nlist; eb += kThreads) {
        const int e = eb + threadIdx.x;
        int tot;
        const int o = block_scan_excl(e < nlist ? __popc(kmask[e]) : 0, sh, tot) + base;
        if (e < nlist) woff[e] = o;
        base += tot;
    }
    __syncthreads();
    for (int e = wid; e < nlist; e += kThreads / 32) {
        const uint32_t km = kmask[e];
        if ((km >> lane) & 1u) {
            const int wi = wlist[e];
            const int o = woff[e] + __popc(km & ((1u << lane) - 1u));
            const int32_t c = col0 + wi * 32 + lane;
            const double v = w[wi * 32 + lane];
            ccol[o] = c;
            cval[o] = v;
            if (o < kCandSh) {
                scol[o] = c;
                sval[o] = v;
            }
        }
    }
    __syncthreads();
    return base;
}

// rule 2 by ranks, for candidates held in shared memory: every thread counts, for each of its
// candidates, the candidates that precede it in the selection order (|v| descending, column
// ascending) -- broadcast reads, no barrier, no histogram -- and keeps it iff fewer than M do; the
// kept entries are written in column order through one scan per 256 candidates.  Exact: the order
// is total, so the kept set is the one any exact selection finds.
__device__ int select_write_rank(const int32_t* scol, const double* sval, int C, int M, int32_t* ocol, double* oval,
                                 int* sh) {
    if (C <= M) {
        for (int t = threadIdx.x; t < C; t += kThreads) {
            ocol[t] = scol[t];
            oval[t] = sval[t];
        }
        __syncthreads();
        return C;
    }
    int base = 0;
    for (int c0 = 0; c0 < C; c0 += kThreads) {
        const int t = c0 + threadIdx.x;
        bool keep = false;
        if (t < C) {
            const uint64_t kt = absbits(sval[t]);
            int rank = 0;
            for (int j = 0; j < C; ++j) {
                const uint64_t kj = absbits(sval[j]);
                rank += (kj > kt || (kj == kt && j < t)) ? 1 : 0;
            }
            keep = rank < M;
        }
        int tot;
        const int o = block_scan_excl(keep ? 1 : 0, sh, tot) + base;
        if (keep) {
            ocol[o] = scol[t];
            oval[o] = sval[t];
        }
        base += tot;
    }
    __syncthreads();
    return base;
}

// rule 2: keep the M largest |v| (ties by ascending column = candidate order); write the
// kept entries in ascending column order to (ocol, oval); returns the kept count
__device__ int select_write(const int32_t* ccol, const double* cval, int C, int M, int32_t* ocol, double* oval,
                            int* sh, int* hist, uint64_t* s64) {
    const bool keep_all = C <= M;
    uint64_t T = 0;
    int need = 0;
    bool eq_all = true;
    if (!keep_all) {
        if (threadIdx.x == 0) {
            s64[0] = 0;  // prefix
            s64[1] = 0;  // mask
            s64[2] = uint64_t(M);
        }
        __syncthreads();
        // magnitudes of one row share the top byte of their keys nearly always: then that pass is
        // a single vote
        int shift0 = 56;
        {
            const uint64_t top = absbits(cval[0]) >> 56;
            bool same = true;
            for (int t = threadIdx.x; t < C; t += kThreads) same = same && (absbits(cval[t]) >> 56) == top;
            if (__syncthreads_and(same)) {
                if (threadIdx.x == 0) {
                    s64[0] = top << 56;
                    s64[1] = uint64_t(255) << 56;
                }
                shift0 = 48;
                __syncthreads();
            }
        }
        for (int shift = shift0; shift >= 0; shift -= 8) {
            hist[threadIdx.x] = 0;  // kThreads == 256 bins
            __syncthreads();
            const uint64_t pre = s64[0], msk = s64[1];
            for (int t = threadIdx.x; t < C; t += kThreads) {
                uint64_t k = absbits(cval[t]);
                if ((k & msk) == pre) atomicAdd(&hist[(k >> shift) & 255], 1);
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                // bins from the top: lane l covers bins 255-8l .. 248-8l; the bin where the running
                // count reaches the number still needed holds the threshold
                const int lane = threadIdx.x;
                const int nd = int(s64[2]);
                int loc[8], sum = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    loc[j] = hist[255 - 8 * lane - j];
                    sum += loc[j];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                const unsigned bal = __ballot_sync(FULL, incl >= nd);
                if (lane == __ffs(bal) - 1) {
                    int cum = incl - sum, j = 0;
                    for (; j < 7; ++j) {
                        if (cum + loc[j] >= nd) break;
                        cum += loc[j];
                    }
                    s64[0] = pre | (uint64_t(255 - 8 * lane - j) << shift);
                    s64[1] = msk | (uint64_t(255) << shift);
                    s64[2] = uint64_t(nd - cum);
                    s64[3] = uint64_t(loc[j]);  // size of the threshold bin
                }
            }
            __syncthreads();
            if (s64[3] == 1 && shift > 0) {
                // one element left in the threshold bin: it is the threshold, take its whole key
                const uint64_t pre2 = s64[0], msk2 = s64[1];
                for (int t = threadIdx.x; t < C; t += kThreads) {
                    const uint64_t k = absbits(cval[t]);
                    if ((k & msk2) == pre2) s64[4] = k;
                }
                __syncthreads();
                if (threadIdx.x == 0) s64[0] = s64[4];
                __syncthreads();
                break;
            }
        }
        T = s64[0];
        need = int(s64[2]);
        // the threshold bin of the last pass holds exactly the elements equal to T
        eq_all = uint64_t(need) == s64[3];
    }
    int base = 0, eqbase = 0;
    for (int c0 = 0; c0 < C; c0 += kThreads) {
        const int t = c0 + threadIdx.x;
        const bool in = t < C;
        const uint64_t k = in ? absbits(cval[t]) : 0;
        const bool eq = in && !keep_all && k == T;
        int eqtot = 0, ktot;
        // rank among the elements equal to the threshold: only when some of them are dropped
        const int eqr = eq_all ? 0 : block_scan_excl(eq ? 1 : 0, sh, eqtot) + eqbase;
        const bool keep = in && (keep_all || k > T || (eq && (eq_all || eqr < need)));
        const int kr = block_scan_excl(keep ? 1 : 0, sh, ktot);
        if (keep) {
            ocol[base + kr] = ccol[t];
            oval[base + kr] = cval[t];
        }
        base += ktot;
        eqbase += eqtot;
    }
    __syncthreads();
    return base;
}

__global__ void __launch_bounds__(kThreads) k_ilut(IlutDev d) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int sh[kThreads / 32 + 1];
    __shared__ int hist[256];
    __shared__ uint64_t s64[5];
    __shared__ int s_row, s_k;
    uint32_t* pres = reinterpret_cast<uint32_t*>(smem);
    uint32_t* piv = pres + d.nwords;
    uint32_t* kmask = piv + d.nwords;                              // gather: kept mask per word
    int32_t* woff = reinterpret_cast<int32_t*>(kmask + d.nwords);  // gather: output offset per word
    int32_t* wlist = woff + d.nwords;                              // gather: the non-empty words
    double* w = d.smem_w ? reinterpret_cast<double*>(smem + ((size_t(5 * d.nwords) * 4 + 15) & ~size_t(15)))
                         : d.gw + size_t(blockIdx.x) * d.W;
    int32_t* ccol = d.gcand_col + size_t(blockIdx.x) * d.W;
    double* cval = d.gcand_val + size_t(blockIdx.x) * d.W;
    __shared__ int32_t scol[kCandSh];
    __shared__ double sval[kCandSh];
    const int b = d.b, M = d.M;
    double t_pre = 0.0;  // pre-threshold of the U-part selection (see below)

    for (int q = threadIdx.x; q < d.W; q += kThreads) w[q] = 0.0;
    for (int q = threadIdx.x; q < 2 * d.nwords; q += kThreads) pres[q] = 0;
    __syncthreads();

    for (;;) {
        if (threadIdx.x == 0) s_row = atomicAdd(d.ticket, 1);
        __syncthreads();
        const int i = s_row;
        if (i >= d.n) break;
        // scatter row i of the permuted matrix into the band window
        for (int q = d.rp[i] + threadIdx.x; q < d.rp[i + 1]; q += kThreads) {
            const int jb = d.ci[q] - i + b;
            w[jb] = d.v[q];
            atomicOr(&pres[jb >> 5], 1u << (jb & 31));
            if (jb < b) atomicOr(&piv[jb >> 5], 1u << (jb & 31));
        }
        const double tau_i = d.tau[i];
        __syncthreads();
        ILUT_STAMP(0);
        int kb = 0;
        const int nwl = (b + 31) >> 5;
        for (;;) {
            if (threadIdx.x < 32) {  // next pending pivot >= kb
                int found = -1;
                for (int wb = kb >> 5; wb < nwl && found < 0; wb += 32) {
                    const int wi = wb + threadIdx.x;
                    uint32_t bits = wi < nwl ? piv[wi] : 0u;
                    if (wi == (kb >> 5)) bits &= FULL << (kb & 31);
                    const uint32_t bal = __ballot_sync(FULL, bits != 0u);
                    if (bal) {
                        const int fl = __ffs(bal) - 1;
                        const uint32_t wbits = __shfl_sync(FULL, bits, fl);
                        found = (wb + fl) * 32 + __ffs(wbits) - 1;
                    }
                }
                if (threadIdx.x == 0) s_k = found;
            }
            __syncthreads();
            const int k = s_k;
            if (k < 0) break;
            // every thread waits for U row jk and loads its own entry together with the diagonal and
            // the length: one L2 round trip per pivot.  All threads form the same multiplier.
            const int jk = i - b + k;
            if ((threadIdx.x & 31) == 0)  // one poller per warp; the warp's loads below follow it
                while (ld_acquire(d.done + jk) == 0) __nanosleep(20);
            __syncwarp();
            ILUT_STAMP(1);
            const size_t ub = size_t(jk) * (M + 1);
            const double udiag = __ldcg(d.Uval + ub);
            const int ulen = __ldcg(d.Ulen + jk);
            int jb0 = 0;
            double uv0 = 0.0;
            if (threadIdx.x + 1 < ulen) {
                jb0 = __ldcg(d.Ucol + ub + 1 + threadIdx.x) - i + b;
                uv0 = __ldcg(d.Uval + ub + 1 + threadIdx.x);
            }
            const double wk = w[k] / udiag;  // w[k] is not written before the barrier below
            const bool go = !(fabs(wk) < tau_i);
            if (go) {
                if (threadIdx.x + 1 < ulen) {
                    const uint32_t bit = 1u << (jb0 & 31);
                    const uint32_t old = atomicOr(&pres[jb0 >> 5], bit);
                    if (!(old & bit) && jb0 < b) atomicOr(&piv[jb0 >> 5], bit);
                    w[jb0] = w[jb0] - wk * uv0;
                }
                for (int q = threadIdx.x + kThreads; q < ulen - 1; q += kThreads) {
                    const int jb = __ldcg(d.Ucol + ub + 1 + q) - i + b;
                    const double uv = __ldcg(d.Uval + ub + 1 + q);
                    const uint32_t bit = 1u << (jb & 31);
                    const uint32_t old = atomicOr(&pres[jb >> 5], bit);
                    if (!(old & bit) && jb < b) atomicOr(&piv[jb >> 5], bit);
                    w[jb] = w[jb] - wk * uv;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {  // U row jk has no column <= jk: nobody touched w[k] or its bits
                piv[k >> 5] &= ~(1u << (k & 31));
                if (go) {
                    w[k] = wk;
                } else {
                    w[k] = 0.0;
                    pres[k >> 5] &= ~(1u << (k & 31));
                }
            }
            __syncwarp();  // warp 0 searches the pivot bitmap next
            kb = k + 1;
        }
        // ---- U part: diagonal + selected off-diagonals, published first
        ILUT_STAMP(2);
        double diag = w[b];
        const bool has_diag = (pres[b >> 5] >> (b & 31)) & 1u;
        if (!has_diag || diag == 0.0) {
            if (threadIdx.x == 0) atomicMin(d.err_row, i);
            diag = 1.0;  // keep going so that no other CTA deadlocks; the host reports err_row
        }
        // Rule 2 keeps the M largest of the entries >= tau_i.  A row of the p = 5 factor has ~1,000
        // of them and keeps 121; a lower bound of the kept magnitudes, guessed from the last row
        // this CTA selected (t_pre = half its M-th largest), drops most of the rest in the gather.
        // Exact: if at least M entries pass the bound, the M largest pass it; otherwise gather again.
        int C = gather(w, pres, kmask, woff, wlist, b + 1, d.W, true, fmax(tau_i, t_pre), i - b, ccol, cval, scol, sval, sh);
        if (t_pre > tau_i && C < M)
            C = gather(w, pres, kmask, woff, wlist, b + 1, d.W, true, tau_i, i - b, ccol, cval, scol, sval, sh);
        const size_t ub = size_t(i) * (M + 1);
        ILUT_STAMP(3);
        int nu;
        if (C <= kCandRank) {
            nu = select_write_rank(scol, sval, C, M, d.Ucol + ub + 1, d.Uval + ub + 1, sh);
        } else {
            nu = select_write(C <= kCandSh ? scol : ccol, C <= kCandSh ? sval : cval, C, M, d.Ucol + ub + 1,
                              d.Uval + ub + 1, sh, hist, s64);
            // s64[0] holds the bits of the M-th largest magnitude (C > M here); all threads read it
            // before the next selection's first barrier-separated write
            if (C > M) t_pre = __longlong_as_double((long long)s64[0]) * 0.5;
        }
        ILUT_STAMP(4);
        __threadfence();  // every writer orders its U entries before the release below
        __syncthreads();
        if (threadIdx.x == 0) {
            d.Ucol[ub] = i;
            d.Uval[ub] = diag;
            d.Ulen[i] = nu + 1;
            st_release(d.done + i, 1);  // orders this thread's three stores; the others fenced above
        }
        ILUT_STAMP(5);
        // ---- L part: the kept multipliers
        C = gather(w, pres, kmask, woff, wlist, 0, b, false, 0.0, i - b, ccol, cval, scol, sval, sh);
        const size_t lb = size_t(i) * M;
        int nl = C <= kCandRank ? select_write_rank(scol, sval, C, M, d.Lcol + lb, d.Lval + lb, sh)
                                : select_write(C <= kCandSh ? scol : ccol, C <= kCandSh ? sval : cval, C, M, d.Lcol + lb,
                                               d.Lval + lb, sh, hist, s64);
        if (threadIdx.x == 0) d.Llen[i] = nl;
        // ---- reset the window
        for (int wi = threadIdx.x; wi < d.nwords; wi += kThreads) {
            uint32_t bits = pres[wi];
            while (bits) {
                int q = __ffs(bits) - 1;
                bits &= bits - 1;
                w[wi * 32 + q] = 0.0;
            }
            pres[wi] = 0;
        }
        __syncthreads();
    }
}

// tau_i = tau * (sum_j |a_ij| / nnz_i), ascending column (oracle order)
__global__ void k_row_tau(int32_t n, const int32_t* __restrict__ rp, const double* __restrict__ v, double tau,
                          double* __restrict__ out) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) s = s + fabs(v[k]);
    out[i] = tau * (s / double(rp[i + 1] - rp[i]));
}

__global__ void k_compact(int32_t n, int stride, const int32_t* __restrict__ len, const int32_t* __restrict__ pcol,
                          const double* __restrict__ pval, const int32_t* __restrict__ rowptr, int32_t* __restrict__ col,
                          double* __restrict__ val) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t src = size_t(i) * stride;
    const int32_t dst = rowptr[i];
    for (int q = 0; q < len[i]; ++q) {
        col[dst + q] = pcol[src + q];
        val[dst + q] = pval[src + q];
    }
}

void compact_rows(int32_t n, int stride, const int32_t* len, const int32_t* pcol, const double* pval, DevCsr& out,
                  cudaStream_t st) {
    out.n = out.m = n;
    PMG_CUDA(cudaMallocAsync(&out.rowptr, sizeof(int32_t) * (n + 1), st));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, len, out.rowptr, n + 1, st);
    void* tmp;
    PMG_CUDA(cudaMallocAsync(&tmp, tb, st));
    // len has n entries; scan n+1 with a zero tail: copy into a padded buffer first
    int32_t* lp;
    PMG_CUDA(cudaMallocAsync(&lp, sizeof(int32_t) * (n + 1), st));
    PMG_CUDA(cudaMemcpyAsync(lp, len, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    PMG_CUDA(cudaMemsetAsync(lp + n, 0, sizeof(int32_t), st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, lp, out.rowptr, n + 1, st);
    int32_t nnz = 0;
    PMG_CUDA(cudaMemcpyAsync(&nnz, out.rowptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    out.nnz = nnz;
    PMG_CUDA(cudaMallocAsync(&out.col, sizeof(int32_t) * std::max(nnz, 1), st));
    PMG_CUDA(cudaMallocAsync(&out.val, sizeof(double) * std::max(nnz, 1), st));
    k_compact<<<ceil_div(n, 256), 256, 0, st>>>(n, stride, len, pcol, pval, out.rowptr, out.col, out.val);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaFreeAsync(tmp, st));
    PMG_CUDA(cudaFreeAsync(lp, st));
}

}  // namespace

struct IlutJob {
    IlutDev d{};
    int32_t n = 0, M = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaStream_t st = nullptr;
    int* h_err = nullptr;  // pinned: first failing row
};

// Launch the factorisation of A on `st` and return without waiting: factorisations of independent
// matrices (the levels of a hierarchy) run concurrently, each a row-to-row chain that needs only a
// few dozen CTAs.  `max_ctas` caps the grid (0 = as many as fit).
IlutJob* ilut_launch(const DevCsr& A, int32_t band, double tau, double fillfactor, int max_ctas, cudaStream_t st) {
    auto* job = new IlutJob;
    const int32_t n = A.n;
    const int32_t M = int32_t(std::ceil(fillfactor * double(A.nnz) / double(n)));
    const int32_t b = std::max(band, 1);
    const int32_t W = 2 * b + 1;
    const int32_t nwords = (W + 31) / 32;
    job->n = n;
    job->M = M;
    job->st = st;
    PMG_CUDA(cudaEventCreate(&job->e0));
    PMG_CUDA(cudaEventCreate(&job->e1));
    PMG_CUDA(cudaMallocHost(&job->h_err, sizeof(int)));
    PMG_CUDA(cudaEventRecord(job->e0, st));

    int dev = 0, nsm = 0;
    PMG_CUDA(cudaGetDevice(&dev));
    PMG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int max_smem = 0;
    PMG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t bits_bytes = (size_t(5 * nwords) * 4 + 15) & ~size_t(15);
    const size_t static_bytes = 4096 + size_t(kCandSh) * 12;
    size_t dyn = bits_bytes + size_t(W) * 8;
    int smem_w = 1;
    if (dyn + static_bytes > size_t(max_smem)) {
        smem_w = 0;
        dyn = bits_bytes;
    }
    if (dyn + static_bytes > size_t(max_smem)) throw CudaError("ilut: band too wide for the bitmaps", 6);
    {
        // the attribute is per function, not per launch: only ever raise it (concurrent launches)
        static std::mutex mu;
        static size_t cur = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (dyn > cur) {
            PMG_CUDA(cudaFuncSetAttribute(k_ilut, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)));
            cur = dyn;
        }
    }
    int occ = 0;
    PMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ilut, kThreads, dyn));
    occ = std::max(1, std::min(occ, 2));  // waiting CTAs only poll: two per SM keep the chain fed
    int grid = int(std::min<int64_t>(int64_t(nsm) * occ, std::max<int32_t>(n, 1)));
    if (max_ctas > 0) grid = std::min(grid, max_ctas);

    IlutDev& d = job->d;
    d.n = n; d.M = M; d.b = b; d.W = W; d.nwords = nwords;
    d.rp = A.rowptr; d.ci = A.col; d.v = A.val;
    d.smem_w = smem_w;
    PMG_CUDA(cudaMallocAsync(&d.tau, sizeof(double) * n, st));
    k_row_tau<<<ceil_div(n, 256), 256, 0, st>>>(n, A.rowptr, A.val, tau, const_cast<double*>(d.tau));
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaMallocAsync(&d.Ucol, sizeof(int32_t) * size_t(n) * (M + 1), st));
    PMG_CUDA(cudaMallocAsync(&d.Uval, sizeof(double) * size_t(n) * (M + 1), st));
    PMG_CUDA(cudaMallocAsync(&d.Ulen, sizeof(int32_t) * n, st));
    PMG_CUDA(cudaMallocAsync(&d.Lcol, sizeof(int32_t) * size_t(n) * std::max(M, 1), st));
    PMG_CUDA(cudaMallocAsync(&d.Lval, sizeof(double) * size_t(n) * std::max(M, 1), st));
    PMG_CUDA(cudaMallocAsync(&d.Llen, sizeof(int32_t) * n, st));
    PMG_CUDA(cudaMallocAsync(&d.done, sizeof(int) * n, st));
    PMG_CUDA(cudaMallocAsync(&d.ticket, sizeof(int) * 2, st));
    d.err_row = d.ticket + 1;
    PMG_CUDA(cudaMallocAsync(&d.gcand_col, sizeof(int32_t) * size_t(grid) * W, st));
    PMG_CUDA(cudaMallocAsync(&d.gcand_val, sizeof(double) * size_t(grid) * W, st));
    d.trace = nullptr;
    if (getenv("PMG_ILUT_TRACE") && n > 4 * kTraceRows) {
        PMG_CUDA(cudaMallocAsync(&d.trace, sizeof(unsigned long long) * kTraceRows * 6, st));
        PMG_CUDA(cudaMemsetAsync(d.trace, 0, sizeof(unsigned long long) * kTraceRows * 6, st));
        d.trace_row0 = n / 2;
    }
    d.gw = nullptr;
    if (!smem_w) PMG_CUDA(cudaMallocAsync(&d.gw, sizeof(double) * size_t(grid) * W, st));
    PMG_CUDA(cudaMemsetAsync(d.done, 0, sizeof(int) * n, st));
    PMG_CUDA(cudaMemsetAsync(d.ticket, 0, sizeof(int), st));
    PMG_CUDA(cudaMemsetAsync(d.err_row, 0x7f, sizeof(int), st));  // 0x7f7f7f7f: no failing row yet
    k_ilut<<<grid, kThreads, dyn, st>>>(d);
    PMG_LAUNCH_CHECK();
    PMG_CUDA(cudaEventRecord(job->e1, st));
    PMG_CUDA(cudaMemcpyAsync(job->h_err, d.err_row, sizeof(int), cudaMemcpyDeviceToHost, st));
    return job;
}

// Wait for a launched factorisation, compact its rows into L and U and release the job.
int ilut_finish(IlutJob* job, DevCsr& L, DevCsr& U, int64_t* err_row, double* seconds, cudaEvent_t ref,
                double* seconds_since_ref) {
    std::unique_ptr<IlutJob> own(job);
    IlutDev& d = job->d;
    cudaStream_t st = job->st;
    const int32_t n = job->n, M = job->M;
    PMG_CUDA(cudaStreamSynchronize(st));
    if (d.trace) {  // diagnostics: where the row-to-row chain spends its time (ns, means over the window)
        std::vector<unsigned long long> t(size_t(kTraceRows) * 6);
        PMG_CUDA(cudaMemcpy(t.data(), d.trace, t.size() * 8, cudaMemcpyDeviceToHost));
        double s[6] = {0, 0, 0, 0, 0, 0};
        int cnt = 0;
        for (int r = 1; r < kTraceRows; ++r) {
            const unsigned long long *a = &t[size_t(r) * 6], *p = &t[size_t(r - 1) * 6];
            if (!a[5] || !p[5] || !a[1]) continue;
            s[0] += double(a[5]) - double(p[5]);                         // chain period
            s[1] += double(a[1]) - double(p[5]);                         // release -> observed by the next row
            s[2] += double(a[2]) - double(a[1]);                         // last pivot
            s[3] += double(a[3]) - double(a[2]);                         // gather U
            s[4] += double(a[4]) - double(a[3]);                         // select + write
            s[5] += double(a[5]) - double(a[4]);                         // fence + release
            ++cnt;
        }
        if (cnt)
            fprintf(stderr, "[pmg] ilut trace n=%d M=%d (%d rows): period %.0f ns = hand-over %.0f + last pivot %.0f + gather %.0f + "
                    "select %.0f + publish %.0f\n", job->n, job->M, cnt, s[0] / cnt, s[1] / cnt, s[2] / cnt, s[3] / cnt, s[4] / cnt,
                    s[5] / cnt);
        PMG_CUDA(cudaFreeAsync(d.trace, st));
        d.trace = nullptr;
    }
    const int er = *job->h_err;
    int status = 0;
    if (er != 0x7f7f7f7f) {
        if (err_row) *err_row = er;
        status = 1;  // PMG_ZERO_PIVOT
    } else {
        compact_rows(n, M, d.Llen, d.Lcol, d.Lval, L, st);
        compact_rows(n, M + 1, d.Ulen, d.Ucol, d.Uval, U, st);
    }
    float ms = 0;
    PMG_CUDA(cudaEventElapsedTime(&ms, job->e0, job->e1));  // the factorisation kernel (compaction excluded)
    if (seconds) *seconds = ms * 1e-3;
    if (ref && seconds_since_ref) {
        PMG_CUDA(cudaEventElapsedTime(&ms, ref, job->e1));
        *seconds_since_ref = ms * 1e-3;
    }
    cudaEventDestroy(job->e0);
    cudaEventDestroy(job->e1);
    cudaFreeHost(job->h_err);
    for (void* p : {(void*)d.tau, (void*)d.Ucol, (void*)d.Uval, (void*)d.Ulen, (void*)d.Lcol, (void*)d.Lval,
                    (void*)d.Llen, (void*)d.done, (void*)d.ticket, (void*)d.gcand_col, (void*)d.gcand_val, (void*)d.gw})
        if (p) PMG_CUDA(cudaFreeAsync(p, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    return status;
}

int ilut_factorize_device(const DevCsr& A, int32_t band, double tau, double fillfactor, DevCsr& L, DevCsr& U,
                          int64_t* err_row, double* seconds, cudaStream_t st) {
    return ilut_finish(ilut_launch(A, band, tau, fillfactor, 0, st), L, U, err_row, seconds, nullptr, nullptr);
}

}  // namespace pmg
