// C ABI of libpmg_cuda.so (include/pmg_cuda.h): device handles, the p-multigrid
// hierarchy and the V-cycle / solve drivers.  Every floating-point operation of the
// solve runs in the kernels of sell.cu / trsv.cu / dense.cu; the host only sequences
// launches on the work stream.
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/pmg_cuda.h"
#include "chain.cuh"
#include "dense.cuh"
#include "ilut.cuh"
#include "krylov.cuh"
#include "rcm.hpp"
#include "skew.cuh"
#include "sell.cuh"
#include "trsv.cuh"
#include "wave.cuh"

using namespace pmg;

namespace {
thread_local std::string g_err;
}
namespace pmg {
void set_last_error(const std::string& m) { g_err = m; }  // for the other translation units (assemble.cu)
}
namespace {

struct ArgError : std::runtime_error {
    int status;
    ArgError(const std::string& m, int s) : std::runtime_error(m), status(s) {}
};

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const CudaError& e) {
        g_err = e.what();
        return e.status;
    } catch (const ArgError& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_err = "host allocation failed";
        return PMG_ERR_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PMG_ERR_CUDA;
    }
}

void check_view(const pmg_csr_view* v) {
    if (!v || v->nrows < 0 || v->ncols < 0 || !v->rowptr) throw ArgError("null/invalid CSR view", PMG_ERR_ARG);
    if (v->rowptr[0] != 0) throw ArgError("CSR rowptr[0] != 0", PMG_ERR_ARG);
    for (int32_t i = 0; i < v->nrows; ++i) {
        if (v->rowptr[i + 1] < v->rowptr[i]) throw ArgError("CSR rowptr decreasing", PMG_ERR_ARG);
        for (int32_t k = v->rowptr[i]; k < v->rowptr[i + 1]; ++k) {
            if (v->col[k] < 0 || v->col[k] >= v->ncols) throw ArgError("CSR column out of range", PMG_ERR_ARG);
            if (k > v->rowptr[i] && v->col[k] <= v->col[k - 1])
                throw ArgError("CSR columns not strictly increasing", PMG_ERR_ARG);
        }
    }
}

template <class T>
T* dalloc(size_t n) {
    T* p = nullptr;
    PMG_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
    return p;
}

DevCsr upload(const pmg_csr_view& v, cudaStream_t st) {
    DevCsr d;
    d.n = v.nrows;
    d.m = v.ncols;
    d.nnz = v.rowptr[v.nrows];
    d.rowptr = dalloc<int32_t>(v.nrows + 1);
    d.col = dalloc<int32_t>(d.nnz);
    d.val = dalloc<double>(d.nnz);
    PMG_CUDA(cudaMemcpyAsync(d.rowptr, v.rowptr, sizeof(int32_t) * (v.nrows + 1), cudaMemcpyHostToDevice, st));
    if (d.nnz) {
        PMG_CUDA(cudaMemcpyAsync(d.col, v.col, sizeof(int32_t) * d.nnz, cudaMemcpyHostToDevice, st));
        PMG_CUDA(cudaMemcpyAsync(d.val, v.val, sizeof(double) * d.nnz, cudaMemcpyHostToDevice, st));
    }
    return d;
}

bool env_flag(const char* name) {
    const char* e = getenv(name);
    return e && e[0] == '1';
}
bool force_levelsched() { return env_flag("PMG_FORCE_LEVELSCHED"); }

// PMG_VERBOSE: wall time of setup phases on stderr
struct Lap {
    bool on = getenv("PMG_VERBOSE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void operator()(const char* what, long long n = 0) {
        if (!on) return;
        cudaDeviceSynchronize();
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[pmg] setup %-28s n=%lld: %.3f s\n", what, n, std::chrono::duration<double>(now - t).count());
        t = now;
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { PMG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
};

}  // namespace

// =================================================================== handles
struct pmg_csr_s {
    DevCsr A;
    Sell S;                       // identity-order sliced layout (SpMV family)
    std::vector<int32_t> h_rowptr, h_col;
    std::vector<double> h_val;    // host copy, fetched from the device when RCM needs it
    std::once_flag h_once;
    void ensure_host() {
        std::call_once(h_once, [&] {
            h_rowptr.resize(size_t(A.n) + 1);
            h_col.resize(size_t(A.nnz));
            h_val.resize(size_t(A.nnz));
            PMG_CUDA(cudaMemcpy(h_rowptr.data(), A.rowptr, sizeof(int32_t) * h_rowptr.size(), cudaMemcpyDeviceToHost));
            PMG_CUDA(cudaMemcpy(h_col.data(), A.col, sizeof(int32_t) * h_col.size(), cudaMemcpyDeviceToHost));
            PMG_CUDA(cudaMemcpy(h_val.data(), A.val, sizeof(double) * h_val.size(), cudaMemcpyDeviceToHost));
        });
    }
    int32_t band = 0;
    // Gauss-Seidel structures (built on first use)
    bool gs_ready = false;
    int64_t gs_zero_row = -1;
    LevelSets gs_lv;
    Sell gs;
    double* gs_diag = nullptr;
    int32_t* gs_nlow = nullptr;
    int32_t seg = 0;              // chained-segment length (0: level-scheduled sweeps)
    std::vector<int32_t> starts;  // grid-row segments of the natural order (empty: no structure)
    int32_t* gs_split = nullptr;
    int32_t gs_gap = 0;
    bool gs_chain = false;        // chained GS sweep (else level-scheduled)
    bool gs_skew = false;         // skewed-warp GS sweep
    SkewPlan gs_plan;
    bool gs_wave = false;         // rotating-lane GS sweep (default for tensor-grid orderings)
    WavePlan gs_wplan;
    ~pmg_csr_s() {
        A.free();
        sell_free(S);
        if (gs_ready) {
            level_sets_free(gs_lv);
            sell_free(gs);
            cudaFree(gs_diag);
            cudaFree(gs_nlow);
            cudaFree(gs_split);
            skew_plan_free(gs_plan);
            wave_plan_free(gs_wplan);
        }
    }
};

struct pmg_factor_s {
    int32_t n = 0;
    DevCsr L, U;
    int32_t* perm = nullptr;          // device, null for the identity ordering
    std::vector<int32_t> h_perm;
    LevelSets lvL, lvU;               // built on first use: reporting, level-scheduled fallback
    std::once_flag lv_once;
    void ensure_levels(cudaStream_t st) {
        std::call_once(lv_once, [&] {
            level_sets(lvL, n, L.rowptr, L.col, kDepLower, st);
            level_sets(lvU, n, U.rowptr, U.col, kDepUpper, st);
            PMG_CUDA(cudaStreamSynchronize(st));
        });
    }
    Sell Ls, Us;
    double* Udiag = nullptr;          // 1.0 / diagonal of U per sweep position
    int32_t max_row_L = 0, max_row_U = 0;
    double seconds = 0;
    int32_t seg = 0;                  // chained-segment length (0: level-scheduled sweeps)
    std::vector<int32_t> starts;      // grid-row segments (rotating-lane sweeps)
    int32_t* rev = nullptr;           // v -> row for the U sweep (descending rows)
    int32_t *splitL = nullptr, *splitU = nullptr;
    bool skew = false;                // skewed-warp sweeps (short rows, short reach)
    bool wave = false;                // rotating-lane sweeps (default for tensor-grid orderings)
    WavePlan waveL, waveU;
    int32_t bs = 32;                  // chain finisher batch
    int32_t gapL = 0, gapU = 0;       // chain start gates
    SkewPlan planL, planU;
    ~pmg_factor_s() {
        L.free();
        U.free();
        cudaFree(perm);
        level_sets_free(lvL);
        level_sets_free(lvU);
        sell_free(Ls);
        sell_free(Us);
        cudaFree(Udiag);
        cudaFree(rev);
        cudaFree(splitL);
        cudaFree(splitU);
        skew_plan_free(planL);
        skew_plan_free(planU);
        wave_plan_free(waveL);
        wave_plan_free(waveU);
    }
};

namespace {

// e = U^{-1} L^{-1} r[perm] added into u[perm]  (y, x: scratch)
void apply_factor(pmg_factor_s* F, const double* r, double* y, double* x, double* u, int* ticket, cudaStream_t st) {
    if (F->wave) {
        wave_prepare2(y, x, F->n, ticket, st);  // sentinels in both outputs, both claim counters
        WaveOp l{kSkewL, &F->waveL, r, y, nullptr};
        l.prepared = true;
        wave_sweep(l, ticket, st);
        WaveOp up{kSkewU, &F->waveU, y, x, u};
        up.prepared = true;
        wave_sweep(up, ticket + 1, st);
    } else if (F->skew) {
        SkewOp l{kSkewL, &F->planL, r, y, nullptr};
        skew_sweep(l, ticket, st);
        SkewOp up{kSkewU, &F->planU, y, x, u};
        skew_sweep(up, ticket, st);
    } else if (F->seg > 0) {
        ChainOp l{kChainL, &F->Ls, nullptr, nullptr, F->splitL, F->perm, r, nullptr, y, nullptr, F->seg, F->bs, F->gapL};
        chain_sweep(l, ticket, st);
        ChainOp up{kChainU, &F->Us, F->Udiag, nullptr, F->splitU, F->perm, y, nullptr, x, u, F->seg, F->bs, F->gapU};
        chain_sweep(up, ticket, st);
    } else {
        lsolve(F->Ls, F->perm, r, y, ticket, st);
        usolve_add(F->Us, F->Udiag, F->perm, y, x, u, ticket, st);
    }
}

// su: n doubles of caller scratch (the skew pre-pass writes the upper sums there)
void gs_apply(pmg_csr_s* A, const double* f, const double* uo, double* un, double* su, int* ticket,
              cudaStream_t st) {
    if (A->gs_wave) {
        WaveOp g{kSkewGS, &A->gs_wplan, f, un, nullptr, &A->gs, A->gs_nlow, uo, su};
        wave_sweep(g, ticket, st);
    } else if (A->gs_skew) {
        SkewOp g{kSkewGS, &A->gs_plan, f, un, nullptr, &A->gs, A->gs_nlow, uo, su};
        skew_sweep(g, ticket, st);
    } else if (A->gs_chain) {
        ChainOp g{kChainGS, &A->gs, A->gs_diag, A->gs_nlow, A->gs_split, nullptr, f, uo, un, nullptr, A->seg, 8, A->gs_gap};
        chain_sweep(g, ticket, st);
    } else {
        gs_sweep(A->gs, A->gs_diag, A->gs_nlow, f, uo, un, ticket, st);
    }
}

pmg_csr_s* make_csr(const pmg_csr_view& v, cudaStream_t st) {
    auto h = std::make_unique<pmg_csr_s>();
    Lap lap;
    h->A = upload(v, st);
    lap("csr upload", v.nrows);
    h->band = pmg_host::bandwidth(v.nrows, v.rowptr, v.col);
    h->seg = force_levelsched() ? 0 : detect_segment(v.nrows, v.rowptr, v.col);
    if (!force_levelsched() && v.nrows == v.ncols) h->starts = detect_segment_starts(v.nrows, v.rowptr, v.col);
    lap("csr band/segments", v.nrows);
    sell_build(h->S, v.nrows, h->A.rowptr, h->A.col, h->A.val, nullptr, kPickAll, nullptr, nullptr, st);
    PMG_CUDA(cudaStreamSynchronize(st));
    lap("csr sell", v.nrows);
    return h.release();
}

void ensure_gs(pmg_csr_s* h, cudaStream_t st) {
    if (h->gs_ready) return;
    const int32_t n = h->A.n;
    level_sets(h->gs_lv, n, h->A.rowptr, h->A.col, kDepLower, st);
    h->gs_diag = dalloc<double>(n);
    h->gs_nlow = dalloc<int32_t>(n);
    // sliced layout in row order for the wavefront kernels (grid-row segments), level order for
    // the level-scheduled fallback
    bool natural = h->seg > 0 || !h->starts.empty();
    auto build = [&](bool nat) {
        sell_free(h->gs);
        sell_build(h->gs, n, h->A.rowptr, h->A.col, h->A.val, nat ? nullptr : h->gs_lv.order, kPickOffDiag,
                   h->gs_diag, h->gs_nlow, st);
    };
    build(natural);
    // first row (in row order) with a zero or missing diagonal -> SPEC.md:237 smoother error
    std::vector<double> dg(n);
    std::vector<int32_t> ord(n);
    PMG_CUDA(cudaMemcpyAsync(dg.data(), h->gs_diag, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(ord.data(), h->gs_lv.order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    int64_t zr = -1;
    for (int32_t p = 0; p < n; ++p) {
        const int32_t row = natural ? p : ord[p];
        if (dg[p] == 0.0 && (zr < 0 || row < zr)) zr = row;
    }
    h->gs_zero_row = zr;
    reciprocal_inplace(h->gs_diag, n, st);
    int32_t mx = 0;  // longest lower part
    if (natural) {
        std::vector<int32_t> nl(n);
        PMG_CUDA(cudaMemcpyAsync(nl.data(), h->gs_nlow, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        PMG_CUDA(cudaStreamSynchronize(st));
        for (int32_t v : nl) mx = std::max(mx, v);
    }
    // 1. rotating-lane GS sweep over the lower entries (any grid-row segments)
    const char* wv = getenv("PMG_WAVE");
    if (!h->starts.empty() && !(wv && wv[0] == '0'))
        h->gs_wave = wave_plan(h->gs, h->gs_diag, h->starts, kSkewGS, mx, h->gs_wplan, st, h->gs_nlow);
    // 2. uniform segments: chained GS, skewed warps where they fit
    h->gs_chain = !h->gs_wave && h->seg > 0;
    if (h->gs_chain) {
        h->gs_split = dalloc<int32_t>(n);
        chain_split(h->gs, h->gs_nlow, h->seg, kChainGS, h->gs_split, st);
        const ChainPlan pl = chain_plan(h->gs, h->gs_nlow, h->gs_split, h->seg, kChainGS, st);
        h->gs_gap = pl.gap;
        if (!pl.ok) {  // rows exceed the chain kernel's on-chip buffers
            h->gs_chain = false;
            cudaFree(h->gs_split);
            h->gs_split = nullptr;
        }
    }
    const char* sk = getenv("PMG_SKEW");
    if (h->gs_chain && !(sk && sk[0] == '0'))
        h->gs_skew = skew_plan(h->gs, h->gs_diag, h->seg, kSkewGS, mx, h->gs_plan, st, h->gs_nlow);
    // 3. level-scheduled sweep (level-order layout; the diagonal follows the layout)
    if (!h->gs_wave && !h->gs_chain && natural) {
        build(false);
        reciprocal_inplace(h->gs_diag, n, st);
    }
    h->gs_ready = true;
}

// ILUT of csr under `ordering` in two steps, so that the factorisations of a hierarchy's levels run
// concurrently: factor_begin permutes (RCM) and launches the factorisation on `sj`; factor_end waits
// for it and builds level sets, sweep layouts and plans on `st`.  On zero pivot factor_end returns
// PMG_ZERO_PIVOT with *err_row.
struct PendingFactor {
    std::unique_ptr<pmg_factor_s> F;
    pmg_csr_s* A = nullptr;
    DevCsr owned;
    IlutJob* job = nullptr;
};

PendingFactor factor_begin(pmg_csr_s* A, double tau, double fillfactor, int ordering, int max_ctas, cudaStream_t sj) {
    if (A->A.n != A->A.m) throw ArgError("ilut: matrix not square", PMG_ERR_DIM);
    if (!(tau >= 0) || !(fillfactor >= 1)) throw ArgError("ilut: tau >= 0 and fillfactor >= 1 required", PMG_ERR_ARG);
    PendingFactor pf;
    pf.A = A;
    pf.F = std::make_unique<pmg_factor_s>();
    auto& F = pf.F;
    const int32_t n = A->A.n;
    F->n = n;
    DevCsr Ap = A->A;
    int32_t band = A->band;
    F->seg = A->seg;
    F->starts = A->starts;
    if (ordering == PMG_ORDER_RCM) {
        A->ensure_host();
        F->h_perm = pmg_host::rcm_ordering(n, A->h_rowptr.data(), A->h_col.data());
        std::vector<int32_t> brp, bci;
        std::vector<double> bv;
        band = pmg_host::permute_symmetric(n, A->h_rowptr.data(), A->h_col.data(), A->h_val.data(), F->h_perm, brp,
                                           bci, bv);
        pmg_csr_view v{n, n, brp.data(), bci.data(), bv.data()};
        F->seg = force_levelsched() ? 0 : detect_segment(n, brp.data(), bci.data());
        pf.owned = upload(v, sj);
        Ap = pf.owned;
        F->perm = dalloc<int32_t>(n);
        PMG_CUDA(cudaMemcpyAsync(F->perm, F->h_perm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, sj));
        PMG_CUDA(cudaStreamSynchronize(sj));
    } else if (ordering != PMG_ORDER_NONE) {
        throw ArgError("unknown ordering", PMG_ERR_ARG);
    }
    pf.job = ilut_launch(Ap, band, tau, fillfactor, max_ctas, sj);
    return pf;
}

int factor_end(PendingFactor& pf, pmg_factor_s** out, int64_t* err_row, cudaStream_t st, cudaEvent_t ref = nullptr,
               double* since_ref = nullptr) {
    auto& F = pf.F;
    pmg_csr_s* A = pf.A;
    const int32_t n = F->n;
    IlutJob* job = pf.job;
    pf.job = nullptr;
    int rc = ilut_finish(job, F->L, F->U, err_row, &F->seconds, ref, since_ref);
    pf.owned.free();
    if (getenv("PMG_VERBOSE"))
        fprintf(stderr, "[pmg] ilut n=%d band=%d nnz(A)=%lld: %.3f s (%.2f us/row)\n", n, A->band, (long long)A->A.nnz,
                F->seconds, 1e6 * F->seconds / std::max(n, 1));
    if (rc != 0) return PMG_ZERO_PIVOT;
    Lap lap;
    F->Udiag = dalloc<double>(n);
    // sliced layouts: natural order (L ascending, U descending rows) for the wavefront kernels,
    // level order for the level-scheduled fallback
    auto build_sells = [&](bool natural) {
        if (!natural) F->ensure_levels(st);
        sell_free(F->Ls);
        sell_free(F->Us);
        if (natural && !F->rev) {
            F->rev = dalloc<int32_t>(n);
            std::vector<int32_t> rv(n);
            for (int32_t v = 0; v < n; ++v) rv[v] = n - 1 - v;
            PMG_CUDA(cudaMemcpyAsync(F->rev, rv.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        }
        sell_build(F->Ls, n, F->L.rowptr, F->L.col, F->L.val, natural ? nullptr : F->lvL.order, kPickAll, nullptr,
                   nullptr, st);
        sell_build(F->Us, n, F->U.rowptr, F->U.col, F->U.val, natural ? F->rev : F->lvU.order, kPickOffDiagDesc,
                   F->Udiag, nullptr, st);
        reciprocal_inplace(F->Udiag, n, st);  // nonzero: a zero pivot was reported above
    };
    // wavefront kernels need the natural (unpermuted) order and grid-row segments
    if (F->perm || force_levelsched()) F->starts.clear();
    const bool natural = F->seg > 0 || !F->starts.empty();
    build_sells(natural);
    lap("factor sells", n);
    // longest rows (reporting, layouts)
    std::vector<int32_t> lr(n + 1), ur(n + 1);
    PMG_CUDA(cudaMemcpyAsync(lr.data(), F->L.rowptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaMemcpyAsync(ur.data(), F->U.rowptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
    PMG_CUDA(cudaStreamSynchronize(st));
    for (int32_t i = 0; i < n; ++i) {
        F->max_row_L = std::max(F->max_row_L, lr[i + 1] - lr[i]);
        F->max_row_U = std::max(F->max_row_U, ur[i + 1] - ur[i]);
    }
    // short rows (p=1 factors): the per-segment lag is dominated by the finisher batch
    F->bs = std::max(F->max_row_L, F->max_row_U) <= 16 ? 8 : 32;
    if (const char* e = getenv("PMG_CHAIN_BS")) F->bs = atoi(e);
    // 1. rotating-lane sweeps (wave.cu) for every grid-row ordering, any segment lengths
    const char* sk = getenv("PMG_SKEW");
    const char* wv = getenv("PMG_WAVE");
    if (!F->starts.empty() && !(wv && wv[0] == '0')) {
        const bool okL = wave_plan(F->Ls, nullptr, F->starts, kSkewL, F->max_row_L, F->waveL, st);
        const bool okU =
            okL && wave_plan(F->Us, F->Udiag, reversed_starts(F->starts), kSkewU, F->max_row_U - 1, F->waveU, st);
        F->wave = okL && okU;
        if (!F->wave) {
            wave_plan_free(F->waveL);
            wave_plan_free(F->waveU);
        }
    }
    // 2. uniform segments: chained-segment sweeps, skewed warps where they fit
    bool chain = !F->wave && F->seg > 0;
    if (chain) {
        F->splitL = dalloc<int32_t>(n);
        F->splitU = dalloc<int32_t>(n);
        chain_split(F->Ls, nullptr, F->seg, kChainL, F->splitL, st);
        chain_split(F->Us, nullptr, F->seg, kChainU, F->splitU, st);
        const ChainPlan pl = chain_plan(F->Ls, nullptr, F->splitL, F->seg, kChainL, st);
        const ChainPlan pu = chain_plan(F->Us, nullptr, F->splitU, F->seg, kChainU, st);
        F->gapL = pl.gap;
        F->gapU = pu.gap;
        if (getenv("PMG_VERBOSE"))
            fprintf(stderr, "[pmg] factor n=%d seg=%d gap %d/%d in-seg %d/%d back %d/%d\n", F->n, F->seg, pl.gap,
                    pu.gap, pl.max_in, pu.max_in, pl.max_back, pu.max_back);
        if (!(pl.ok && pu.ok)) {  // rows exceed the chain kernel's on-chip buffers
            chain = false;
            cudaFree(F->splitL);
            cudaFree(F->splitU);
            F->splitL = F->splitU = nullptr;
        }
    }
    if (chain && !F->perm && !(sk && sk[0] == '0')) {
        const bool okL = skew_plan(F->Ls, nullptr, F->seg, kSkewL, F->max_row_L, F->planL, st);
        const bool okU = okL && skew_plan(F->Us, F->Udiag, F->seg, kSkewU, F->max_row_U - 1, F->planU, st);
        F->skew = okL && okU;
        if (!F->skew) {
            skew_plan_free(F->planL);
            skew_plan_free(F->planU);
        }
        if (getenv("PMG_VERBOSE"))
            fprintf(stderr, "[pmg] factor n=%d skew %d NRxC %dx%d D %d/%d dm %d/%d ring %d/%d\n", F->n, int(F->skew),
                    F->planL.nr, F->planL.c, F->planL.D, F->planU.D, F->planL.dm, F->planU.dm, F->planL.ry,
                    F->planU.ry);
    }
    // 3. level-scheduled sweeps (level-order layouts)
    if (!F->wave && !chain) {
        F->seg = 0;
        if (natural) build_sells(false);
    }
    lap("factor layouts + plans", n);
    *out = F.release();
    return PMG_OK;
}

int make_factor(pmg_csr_s* A, double tau, double fillfactor, int ordering, pmg_factor_s** out, int64_t* err_row,
                cudaStream_t st) {
    PendingFactor pf = factor_begin(A, tau, fillfactor, ordering, 0, st);
    return factor_end(pf, out, err_row, st);
}

}  // namespace

// =================================================================== hierarchy
namespace {

struct PLev {
    int degree = 1;
    pmg_csr_s* A = nullptr;
    pmg_csr_s* P = nullptr;   // level l+1 -> l (rows of this level)
    pmg_csr_s* PT = nullptr;
    double* ML = nullptr;
    pmg_factor_s* F = nullptr;
};
struct HLev {
    pmg_csr_s* A = nullptr;   // for j = 0: alias of the last p-level's A
    bool own_A = false;
    pmg_csr_s* P = nullptr;
    pmg_csr_s* PT = nullptr;
    pmg_factor_s* F = nullptr;
};

}  // namespace

struct pmg_hier_s {
    std::vector<PLev> pl;
    std::vector<HLev> hl;
    DenseLU coarse;
    int smoother = PMG_SMOOTHER_ILUT, nu1 = 1, nu2 = 1;
    pmg_hier_stats stats{};
    ~pmg_hier_s() {
        for (auto& l : pl) {
            delete l.A;
            delete l.P;
            delete l.PT;
            cudaFree(l.ML);
            delete l.F;
        }
        for (auto& h : hl) {
            if (h.own_A) delete h.A;
            delete h.P;
            delete h.PT;
            delete h.F;
        }
        dense_free(coarse);
    }
};

// -------------------------------------------------------------------- work / cycle
namespace {

enum Cls { kClsResid0 = 0, kClsL0, kClsU0, kClsGS0, kClsTransfer, kClsCoarse, kClsMisc, kNumCls };

struct PWork {
    double* u[2] = {nullptr, nullptr};
    int cur = 0;
    double *f = nullptr, *r = nullptr, *y = nullptr, *x = nullptr;
};
struct HWork {
    double *e = nullptr, *r = nullptr, *res = nullptr, *y = nullptr, *x = nullptr;
};

}  // namespace

struct pmg_work_s {
    pmg_hier_s* H = nullptr;
    cudaStream_t st = nullptr;
    std::vector<PWork> pw;
    std::vector<HWork> hw;
    int* ticket = nullptr;
    NormCtx nc{};
    double* norm0 = nullptr;
    double* dhist = nullptr;
    int hist_cap = 0;
    double* h_pinned = nullptr;
    // BiCGSTAB vectors (allocated on first use): u, r, rh, p, v, s, t, ph, sh; dots
    double* kv[9] = {};
    double* kdot = nullptr;   // device: [rho, rv, tt, ts, ||r||]
    double* kdot_h = nullptr; // pinned host copy
    // optional per-class event timing
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
    std::vector<int> ev_cls;
    size_t ev_used = 0;
    double cls_ms[kNumCls] = {};
    int64_t launches = 0;
    int64_t cls_launches[kNumCls] = {};
    // one solve cycle (V-cycle + stop-test residual) captured as a CUDA graph:
    // replayed per cycle, re-captured when the right-hand side buffer changes
    cudaGraphExec_t gx = nullptr;
    const double* gx_f = nullptr;
    int gx_cur = -1;
    int64_t gx_launches = 0;
    int64_t gx_cls[kNumCls] = {};
    double* rho_dev = nullptr;    // the cycle's rho (device), copied to rho_host by the graph
    double* rho_host = nullptr;   // pinned

    ~pmg_work_s() {
        for (auto& p : pw) {
            cudaFree(p.u[0]);
            cudaFree(p.u[1]);
            cudaFree(p.f);
            cudaFree(p.r);
            cudaFree(p.y);
            cudaFree(p.x);
        }
        for (auto& h : hw) {
            cudaFree(h.e);
            cudaFree(h.r);
            cudaFree(h.res);
            cudaFree(h.y);
            cudaFree(h.x);
        }
        cudaFree(ticket);
        cudaFree(nc.partials);
        cudaFree(nc.counter);
        cudaFree(norm0);
        cudaFree(dhist);
        cudaFreeHost(h_pinned);
        for (double* v : kv) cudaFree(v);
        cudaFree(kdot);
        cudaFreeHost(kdot_h);
        for (auto& e : ev_pool) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        if (gx) cudaGraphExecDestroy(gx);
        cudaFree(rho_dev);
        cudaFreeHost(rho_host);
        if (st) cudaStreamDestroy(st);
    }

    template <class F>
    void run(int cls, int nlaunch, F&& f) {
        launches += nlaunch;
        cls_launches[cls] += nlaunch;
        if (!prof) {
            f();
            return;
        }
        if (ev_used == ev_pool.size()) {
            cudaEvent_t a, b;
            PMG_CUDA(cudaEventCreate(&a));
            PMG_CUDA(cudaEventCreate(&b));
            ev_pool.push_back({a, b});
            ev_cls.push_back(0);
        }
        auto& e = ev_pool[ev_used];
        ev_cls[ev_used] = cls;
        ++ev_used;
        PMG_CUDA(cudaEventRecord(e.first, st));
        f();
        PMG_CUDA(cudaEventRecord(e.second, st));
    }
    void collect() {
        if (!prof || ev_used == 0) return;
        PMG_CUDA(cudaStreamSynchronize(st));
        for (size_t k = 0; k < ev_used; ++k) {
            float ms = 0;
            PMG_CUDA(cudaEventElapsedTime(&ms, ev_pool[k].first, ev_pool[k].second));
            cls_ms[ev_cls[k]] += ms;
        }
        ev_used = 0;
    }
};

namespace {

void smooth_ilut(pmg_work_s& W, pmg_csr_s* A, pmg_factor_s* F, double* u, const double* f, const double* r_known,
                 double* r, double* y, double* x, bool fine) {
    const double* rr = r_known;
    if (!rr) {
        W.run(fine ? kClsResid0 : kClsCoarse, 1, [&] { sell_rowop(A->S, kOpResidual, u, f, nullptr, r, nullptr, W.st); });
        rr = r;
    }
    // launch counts: our kernels per sweep (sentinel fill, sweep, and the U update pass)
    if (F->wave) {  // one preparation launch for both sweeps, then L, U, and the U update pass
        W.run(fine ? kClsL0 : kClsCoarse, 2, [&] {
            wave_prepare2(y, x, F->n, W.ticket, W.st);
            WaveOp l{kSkewL, &F->waveL, rr, y, nullptr};
            l.prepared = true;
            wave_sweep(l, W.ticket, W.st);
        });
        W.run(fine ? kClsU0 : kClsCoarse, 2, [&] {
            WaveOp up{kSkewU, &F->waveU, y, x, u};
            up.prepared = true;
            wave_sweep(up, W.ticket + 1, W.st);
        });
    } else if (F->skew) {
        W.run(fine ? kClsL0 : kClsCoarse, 2, [&] {
            SkewOp l{kSkewL, &F->planL, rr, y, nullptr};
            skew_sweep(l, W.ticket, W.st);
        });
        W.run(fine ? kClsU0 : kClsCoarse, 3, [&] {
            SkewOp up{kSkewU, &F->planU, y, x, u};
            skew_sweep(up, W.ticket, W.st);
        });
    } else if (F->seg > 0) {
        W.run(fine ? kClsL0 : kClsCoarse, 2, [&] {
            ChainOp l{kChainL, &F->Ls, nullptr, nullptr, F->splitL, F->perm, rr, nullptr, y, nullptr, F->seg, F->bs, F->gapL};
            chain_sweep(l, W.ticket, W.st);
        });
        W.run(fine ? kClsU0 : kClsCoarse, 3, [&] {
            ChainOp up{kChainU, &F->Us, F->Udiag, nullptr, F->splitU, F->perm, y, nullptr, x, u, F->seg, F->bs, F->gapU};
            chain_sweep(up, W.ticket, W.st);
        });
    } else {
        W.run(fine ? kClsL0 : kClsCoarse, 3, [&] { lsolve(F->Ls, F->perm, rr, y, W.ticket, W.st); });
        W.run(fine ? kClsU0 : kClsCoarse, 3, [&] { usolve_add(F->Us, F->Udiag, F->perm, y, x, u, W.ticket, W.st); });
    }
}

// one h-MG V(1,1) cycle on h-level j from e = 0
void hmg(pmg_work_s& W, int j, double* e, const double* r) {
    pmg_hier_s& H = *W.H;
    HLev& L = H.hl[j];
    HWork& w = W.hw[j];
    const int32_t n = L.A->A.n;
    if (j == int(H.hl.size()) - 1) {
        W.run(kClsCoarse, 1, [&] { dense_solve(H.coarse, r, e, W.st); });
        return;
    }
    W.run(kClsCoarse, 0, [&] { PMG_CUDA(cudaMemsetAsync(e, 0, sizeof(double) * n, W.st)); });
    smooth_ilut(W, L.A, L.F, e, r, r, nullptr, w.y, w.x, false);
    W.run(kClsCoarse, 1, [&] { sell_rowop(L.A->S, kOpResidual, e, r, nullptr, w.res, nullptr, W.st); });
    HWork& c = W.hw[j + 1];
    W.run(kClsCoarse, 1, [&] { sell_rowop(L.PT->S, kOpSpmv, w.res, nullptr, nullptr, c.r, nullptr, W.st); });
    hmg(W, j + 1, c.e, c.r);
    W.run(kClsCoarse, 1, [&] { sell_rowop(L.P->S, kOpAdd, c.e, nullptr, nullptr, e, nullptr, W.st); });
    smooth_ilut(W, L.A, L.F, e, r, nullptr, w.res, w.y, w.x, false);
}

int smooth(pmg_work_s& W, int l, const double* f, const double* r_known) {
    pmg_hier_s& H = *W.H;
    PLev& L = H.pl[l];
    PWork& w = W.pw[l];
    const bool fine = l == 0;
    if (H.smoother == PMG_SMOOTHER_GS) {
        if (L.A->gs_zero_row >= 0) return PMG_ZERO_DIAG;
        double* uo = w.u[w.cur];
        double* un = w.u[1 - w.cur];
        W.run(fine ? kClsGS0 : kClsCoarse, L.A->gs_wave ? 2 : L.A->gs_skew ? 3 : 2,
              [&] { gs_apply(L.A, f, uo, un, w.y, W.ticket, W.st); });  // w.y: idle in GS mode
        w.cur = 1 - w.cur;
        return PMG_OK;
    }
    smooth_ilut(W, L.A, L.F, w.u[w.cur], f, r_known, w.r, w.y, w.x, fine);
    return PMG_OK;
}

// V-cycle at p-level l; `zero`: u == 0 on entry (its residual is f)
int vcycle(pmg_work_s& W, int l, const double* f, const double* r_known, bool zero) {
    pmg_hier_s& H = *W.H;
    PWork& w = W.pw[l];
    if (l == int(H.pl.size()) - 1) {
        if (zero) {  // u == 0: the h-MG correction is the new iterate
            hmg(W, 0, w.u[w.cur], f);
            return PMG_OK;
        }
        // a hierarchy of p = 1 alone: e = hmg(f - A u), u += e
        PLev& L = H.pl[l];
        const int32_t n = L.A->A.n;
        const int cls = l == 0 ? kClsResid0 : kClsCoarse;
        const double* r = r_known;
        if (!r) {
            W.run(cls, 1, [&] { sell_rowop(L.A->S, kOpResidual, w.u[w.cur], f, nullptr, w.r, nullptr, W.st); });
            r = w.r;
        }
        hmg(W, 0, w.y, r);
        W.run(kClsCoarse, 1, [&] { vec_add(w.u[w.cur], w.y, n, W.st); });
        return PMG_OK;
    }
    PLev& L = H.pl[l];
    const bool fine = l == 0;
    for (int s = 0; s < H.nu1; ++s) {
        int rc = smooth(W, l, f, s == 0 ? (zero ? f : r_known) : nullptr);
        if (rc) return rc;
    }
    W.run(fine ? kClsResid0 : kClsCoarse, 1,
          [&] { sell_rowop(L.A->S, kOpResidual, w.u[w.cur], f, nullptr, w.r, nullptr, W.st); });
    PLev& C = H.pl[l + 1];
    PWork& c = W.pw[l + 1];
    W.run(fine ? kClsTransfer : kClsCoarse, 1,
          [&] { sell_rowop(L.PT->S, kOpRestrict, w.r, nullptr, C.ML, c.f, nullptr, W.st); });
    W.run(kClsCoarse, 0, [&] { PMG_CUDA(cudaMemsetAsync(c.u[c.cur], 0, sizeof(double) * C.A->A.n, W.st)); });
    int rc = vcycle(W, l + 1, c.f, nullptr, true);
    if (rc) return rc;
    W.run(fine ? kClsTransfer : kClsCoarse, 1,
          [&] { sell_rowop(L.P->S, kOpProlongAdd, c.u[c.cur], nullptr, L.ML, w.u[w.cur], nullptr, W.st); });
    for (int s = 0; s < H.nu2; ++s) {
        rc = smooth(W, l, f, nullptr);
        if (rc) return rc;
    }
    return PMG_OK;
}

void ensure_hist(pmg_work_s& W, int max_cycles) {
    if (W.hist_cap >= max_cycles + 1) return;
    cudaFree(W.dhist);
    cudaFreeHost(W.h_pinned);
    W.dhist = dalloc<double>(max_cycles + 1);
    PMG_CUDA(cudaMallocHost(&W.h_pinned, sizeof(double) * (max_cycles + 1)));
    W.hist_cap = max_cycles + 1;
}

// the solve loop on device-resident f / u (u = pw[0].u[cur] on entry and exit)
int solve_loop(pmg_work_s& W, const double* d_f, double tol, int max_cycles, double* rho_hist, int* cycles, int* flags,
               double* seconds) {
    pmg_hier_s& H = *W.H;
    PLev& L0 = H.pl[0];
    PWork& w0 = W.pw[0];
    const int32_t n = L0.A->A.n;
    ensure_hist(W, max_cycles);
    cudaEvent_t e0, e1;
    PMG_CUDA(cudaEventCreate(&e0));
    PMG_CUDA(cudaEventCreate(&e1));
    PMG_CUDA(cudaEventRecord(e0, W.st));
    NormCtx nc = W.nc;
    nc.norm_out = W.norm0;
    nc.n0 = nullptr;
    nc.hist_out = nullptr;
    W.run(kClsResid0, 1, [&] { sell_rowop(L0.A->S, kOpResidual, w0.u[w0.cur], d_f, nullptr, w0.r, &nc, W.st); });
    PMG_CUDA(cudaMemcpyAsync(W.h_pinned, W.norm0, sizeof(double), cudaMemcpyDeviceToHost, W.st));
    PMG_CUDA(cudaStreamSynchronize(W.st));
    const double n0 = W.h_pinned[0];
    rho_hist[0] = 1.0;
    *cycles = 0;
    *flags = 0;
    int rc = PMG_OK;
    if (n0 == 0.0) {
        *flags = PMG_FLAG_CONVERGED;
    } else {
        // one cycle: V-cycle, then the stop-test residual (reused by the next cycle's first
        // pre-smoothing) with rho = ||r|| / ||r0|| formed on the device
        auto body = [&]() -> int {
            int r = vcycle(W, 0, d_f, w0.r, false);
            if (r) return r;
            NormCtx ncc = W.nc;
            ncc.norm_out = nullptr;
            ncc.n0 = W.norm0;
            ncc.hist_out = W.rho_dev;
            W.run(kClsResid0, 1,
                  [&] { sell_rowop(L0.A->S, kOpResidual, w0.u[w0.cur], d_f, nullptr, w0.r, &ncc, W.st); });
            PMG_CUDA(cudaMemcpyAsync(W.rho_host, W.rho_dev, sizeof(double), cudaMemcpyDeviceToHost, W.st));
            return PMG_OK;
        };
        const bool graphs = !W.prof && !env_flag("PMG_NO_GRAPH");
        auto cur_mask = [&] {  // which of the two iterate buffers each p-level uses
            int m = 0;
            for (size_t l = 0; l < W.pw.size(); ++l) m |= W.pw[l].cur << l;
            return m;
        };
        for (int c = 1; c <= max_cycles; ++c) {
            // the first cycle of a solve runs eagerly (lazy one-time setup happens there)
            const bool replay = graphs && W.gx && W.gx_f == d_f && W.gx_cur == cur_mask();
            if (graphs && !replay && c >= 2) {
                if (W.gx) cudaGraphExecDestroy(W.gx);
                W.gx = nullptr;
                std::vector<int> curs;
                for (auto& pw : W.pw) curs.push_back(pw.cur);
                const int64_t l0 = W.launches;
                int64_t c0[kNumCls], c1[kNumCls];
                std::copy(W.cls_launches, W.cls_launches + kNumCls, c0);
                cudaGraph_t g = nullptr;
                PMG_CUDA(cudaStreamBeginCapture(W.st, cudaStreamCaptureModeThreadLocal));
                int r = PMG_OK;
                try {
                    r = body();
                } catch (...) {
                    cudaStreamEndCapture(W.st, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                const int64_t l1 = W.launches;
                std::copy(W.cls_launches, W.cls_launches + kNumCls, c1);
                PMG_CUDA(cudaStreamEndCapture(W.st, &g));
                if (r) {
                    cudaGraphDestroy(g);
                    rc = r;
                    break;
                }
                // a cycle must leave every level's buffer selection as it found it (Gauss-Seidel
                // flips it per sweep), else the replay would read stale buffers
                bool same = true;
                for (size_t l = 0; l < W.pw.size(); ++l) {
                    same = same && W.pw[l].cur == curs[l];
                    W.pw[l].cur = curs[l];
                }
                W.launches = l0;  // counted per execution below
                std::copy(c0, c0 + kNumCls, W.cls_launches);
                if (same) {
                    PMG_CUDA(cudaGraphInstantiate(&W.gx, g, 0));
                    W.gx_f = d_f;
                    W.gx_cur = cur_mask();
                    W.gx_launches = l1 - l0;
                    for (int k = 0; k < kNumCls; ++k) W.gx_cls[k] = c1[k] - c0[k];
                }
                cudaGraphDestroy(g);
            }
            if (graphs && W.gx && W.gx_f == d_f && W.gx_cur == cur_mask()) {
                PMG_CUDA(cudaGraphLaunch(W.gx, W.st));
                W.launches += W.gx_launches;
                for (int k = 0; k < kNumCls; ++k) W.cls_launches[k] += W.gx_cls[k];
            } else {
                rc = body();
                if (rc) break;
            }
            PMG_CUDA(cudaStreamSynchronize(W.st));
            const double rho = *W.rho_host;
            rho_hist[c] = rho;
            *cycles = c;
            if (rho <= tol) {
                *flags = PMG_FLAG_CONVERGED;
                break;
            }
            if (!(rho <= 1e10)) {
                *flags = PMG_FLAG_DIVERGED;
                break;
            }
        }
    }
    PMG_CUDA(cudaEventRecord(e1, W.st));
    PMG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    PMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (seconds) *seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    W.collect();
    (void)n;
    return rc;
}

// Right-preconditioned BiCGSTAB, the preconditioner one
// V-cycle from zero.  Same algorithm, breakdown rules and operation order as the oracle
// (oracle/oracle.cpp bicgstab): canonical dots on the device, scalars formed on the host from
// the (bit-identical) dot values, fused vector updates.  u = kv[0] on entry and exit.
int bicgstab_loop(pmg_work_s& W, const double* d_f, double tol, int max_iter, double* hist, int* iters, int* flags,
                  double* seconds) {
    pmg_hier_s& H = *W.H;
    pmg_csr_s* A = H.pl[0].A;
    PWork& w0 = W.pw[0];
    const int32_t n = A->A.n;
    double *u = W.kv[0], *r = W.kv[1], *rh = W.kv[2], *p = W.kv[3], *v = W.kv[4], *s = W.kv[5], *t = W.kv[6],
           *ph = W.kv[7], *sh = W.kv[8];
    cudaEvent_t e0, e1;
    PMG_CUDA(cudaEventCreate(&e0));
    PMG_CUDA(cudaEventCreate(&e1));
    PMG_CUDA(cudaEventRecord(e0, W.st));
    auto fetch = [&](int k) {  // dot slots [0, k) to the host
        PMG_CUDA(cudaMemcpyAsync(W.kdot_h, W.kdot, sizeof(double) * k, cudaMemcpyDeviceToHost, W.st));
        PMG_CUDA(cudaStreamSynchronize(W.st));
    };
    auto dot = [&](const double* x, const double* y, int slot) {
        NormCtx c = W.nc;
        c.norm_out = W.kdot + slot;
        c.n0 = nullptr;
        c.hist_out = nullptr;
        W.run(kClsMisc, 1, [&] { vec_dot(x, y, n, c, W.st); });
    };
    auto prec = [&](const double* x, double* z) {  // z = one V-cycle from zero with right-hand side x
        w0.cur = 0;
        W.run(kClsMisc, 0, [&] { PMG_CUDA(cudaMemsetAsync(w0.u[0], 0, sizeof(double) * n, W.st)); });
        int rc = vcycle(W, 0, x, x, true);
        W.run(kClsMisc, 0, [&] {
            PMG_CUDA(cudaMemcpyAsync(z, w0.u[w0.cur], sizeof(double) * n, cudaMemcpyDeviceToDevice, W.st));
        });
        return rc;
    };
    auto spmv = [&](const double* x, double* y) {
        W.run(kClsResid0, 1, [&] { sell_rowop(A->S, kOpSpmv, x, nullptr, nullptr, y, nullptr, W.st); });
    };
    NormCtx nc = W.nc;
    nc.norm_out = W.kdot + 4;
    nc.n0 = nullptr;
    nc.hist_out = nullptr;
    W.run(kClsResid0, 1, [&] { sell_rowop(A->S, kOpResidual, u, d_f, nullptr, r, &nc, W.st); });
    PMG_CUDA(cudaMemcpyAsync(W.kdot_h + 4, W.kdot + 4, sizeof(double), cudaMemcpyDeviceToHost, W.st));
    PMG_CUDA(cudaStreamSynchronize(W.st));
    const double n0 = W.kdot_h[4];
    hist[0] = 1.0;
    *iters = 0;
    *flags = 0;
    int rc = PMG_OK;
    if (n0 == 0.0) {
        *flags = PMG_FLAG_CONVERGED;
    } else {
        PMG_CUDA(cudaMemcpyAsync(rh, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, W.st));
        double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
        for (int it = 1; it <= max_iter; ++it) {
            dot(rh, r, 0);
            fetch(1);
            const double rho = W.kdot_h[0];
            if (rho == 0.0 || !std::isfinite(rho)) {
                *flags |= PMG_FLAG_BREAKDOWN;
                break;
            }
            if (it == 1) {
                PMG_CUDA(cudaMemcpyAsync(p, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, W.st));
            } else {
                const double beta = (rho / rho_prev) * (alpha / omega);
                W.run(kClsMisc, 1, [&] { bicg_update_p(p, r, v, beta, omega, n, W.st); });
            }
            if ((rc = prec(p, ph))) break;
            spmv(ph, v);
            dot(rh, v, 1);
            fetch(2);
            const double rv = W.kdot_h[1];
            if (rv == 0.0 || !std::isfinite(rv)) {
                *flags |= PMG_FLAG_BREAKDOWN;
                break;
            }
            alpha = rho / rv;
            W.run(kClsMisc, 1, [&] { bicg_update_s(s, r, v, alpha, n, W.st); });
            if ((rc = prec(s, sh))) break;
            spmv(sh, t);
            dot(t, t, 2);
            dot(t, s, 3);
            fetch(4);
            const double tt = W.kdot_h[2], ts = W.kdot_h[3];
            omega = tt == 0.0 ? 0.0 : ts / tt;
            W.run(kClsMisc, 1, [&] { bicg_update_ur(u, r, s, t, ph, sh, alpha, omega, n, W.st); });
            NormCtx nr = W.nc;
            nr.norm_out = W.kdot + 4;
            nr.n0 = nullptr;
            nr.hist_out = nullptr;
            W.run(kClsMisc, 1, [&] { vec_norm(r, n, nr, W.st); });
            PMG_CUDA(cudaMemcpyAsync(W.kdot_h + 4, W.kdot + 4, sizeof(double), cudaMemcpyDeviceToHost, W.st));
            PMG_CUDA(cudaStreamSynchronize(W.st));
            const double res = W.kdot_h[4] / n0;
            hist[it] = res;
            *iters = it;
            if (res <= tol) {
                *flags |= PMG_FLAG_CONVERGED;
                break;
            }
            if (!(res <= 1e10)) {
                *flags |= PMG_FLAG_DIVERGED;
                break;
            }
            if (omega == 0.0) {
                *flags |= PMG_FLAG_BREAKDOWN;
                break;
            }
            rho_prev = rho;
        }
    }
    PMG_CUDA(cudaEventRecord(e1, W.st));
    PMG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    PMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (seconds) *seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    W.collect();
    return rc;
}

void ensure_krylov(pmg_work_s& W) {
    if (W.kdot) return;
    const int32_t n = W.H->pl[0].A->A.n;
    for (double*& v : W.kv) v = dalloc<double>(n);
    W.kdot = dalloc<double>(8);
    PMG_CUDA(cudaMallocHost(&W.kdot_h, sizeof(double) * 8));
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* pmg_status_string(int s) {
    switch (s) {
        case PMG_OK: return "ok";
        case PMG_ZERO_PIVOT: return "zero pivot";
        case PMG_ZERO_DIAG: return "zero diagonal";
        case PMG_ERR_DIM: return "dimension mismatch";
        case PMG_ERR_CUDA: return "cuda error";
        case PMG_ERR_OOM: return "out of memory";
        case PMG_ERR_ARG: return "invalid argument";
    }
    return "unknown";
}

const char* pmg_last_error(void) { return g_err.c_str(); }

int pmg_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    return guarded([&] {
        int dev = 0;
        PMG_CUDA(cudaGetDevice(&dev));
        cudaDeviceProp p;
        PMG_CUDA(cudaGetDeviceProperties(&p, dev));
        if (sm_count) *sm_count = p.multiProcessorCount;
        if (cc_major) *cc_major = p.major;
        if (cc_minor) *cc_minor = p.minor;
        return PMG_OK;
    });
}

int pmg_csr_create(const pmg_csr_view* A, pmg_csr* out) {
    return guarded([&] {
        check_view(A);
        Stream s;
        *out = make_csr(*A, s.s);
        return PMG_OK;
    });
}

int pmg_csr_destroy(pmg_csr A) {
    delete A;
    return PMG_OK;
}

namespace {
struct HostVecs {
    std::vector<double*> ptrs;
    ~HostVecs() {
        for (auto p : ptrs) cudaFree(p);
    }
    double* make(size_t n) {
        ptrs.push_back(dalloc<double>(n));
        return ptrs.back();
    }
};
}  // namespace

int pmg_spmv(pmg_csr A, const double* x, double* y) {
    return guarded([&] {
        Stream s;
        HostVecs hv;
        double* dx = hv.make(A->A.m);
        double* dy = hv.make(A->A.n);
        PMG_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * A->A.m, cudaMemcpyHostToDevice, s.s));
        sell_rowop(A->S, kOpSpmv, dx, nullptr, nullptr, dy, nullptr, s.s);
        PMG_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * A->A.n, cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return PMG_OK;
    });
}

int pmg_residual(pmg_csr A, const double* x, const double* f, double* r, double* norm2) {
    return guarded([&] {
        Stream s;
        HostVecs hv;
        const int32_t n = A->A.n;
        double* dx = hv.make(A->A.m);
        double* df = hv.make(n);
        double* dr = hv.make(n);
        double* parts = hv.make(ceil_div(n, 256) + 1);
        double* nrm = hv.make(1);
        unsigned* cnt = reinterpret_cast<unsigned*>(hv.make(1));
        PMG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(double), s.s));
        PMG_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * A->A.m, cudaMemcpyHostToDevice, s.s));
        PMG_CUDA(cudaMemcpyAsync(df, f, sizeof(double) * n, cudaMemcpyHostToDevice, s.s));
        NormCtx nc{parts, cnt, nrm, nullptr, nullptr};
        sell_rowop(A->S, kOpResidual, dx, df, nullptr, dr, &nc, s.s);
        PMG_CUDA(cudaMemcpyAsync(r, dr, sizeof(double) * n, cudaMemcpyDeviceToHost, s.s));
        if (norm2) PMG_CUDA(cudaMemcpyAsync(norm2, nrm, sizeof(double), cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return PMG_OK;
    });
}

int pmg_gs_sweep(pmg_csr A, double* u, const double* f, int64_t* err_row) {
    return guarded([&] {
        if (A->A.n != A->A.m) throw ArgError("gs: matrix not square", PMG_ERR_DIM);
        Stream s;
        ensure_gs(A, s.s);
        if (A->gs_zero_row >= 0) {
            if (err_row) *err_row = A->gs_zero_row;
            return int(PMG_ZERO_DIAG);
        }
        HostVecs hv;
        const int32_t n = A->A.n;
        double* du = hv.make(n);
        double* dn = hv.make(n);
        double* df = hv.make(n);
        double* dsu = hv.make(n);
        int* tk = reinterpret_cast<int*>(hv.make(kSweepScratchInts / 2));  // ticket + per-sweep scratch
        PMG_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * n, cudaMemcpyHostToDevice, s.s));
        PMG_CUDA(cudaMemcpyAsync(df, f, sizeof(double) * n, cudaMemcpyHostToDevice, s.s));
        gs_apply(A, df, du, dn, dsu, tk, s.s);
        PMG_CUDA(cudaMemcpyAsync(u, dn, sizeof(double) * n, cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return int(PMG_OK);
    });
}

int pmg_rcm_ordering(const pmg_csr_view* A, int32_t* perm) {
    return guarded([&] {
        check_view(A);
        auto p = pmg_host::rcm_ordering(A->nrows, A->rowptr, A->col);
        std::copy(p.begin(), p.end(), perm);
        return PMG_OK;
    });
}

int pmg_ilut_factorize(pmg_csr A, double tau, double fillfactor, int ordering, pmg_factor* out, int64_t* err_row) {
    return guarded([&] {
        Stream s;
        return make_factor(A, tau, fillfactor, ordering, out, err_row, s.s);
    });
}

int pmg_factor_destroy(pmg_factor F) {
    delete F;
    return PMG_OK;
}

int pmg_ilut_apply(pmg_factor F, const double* r, double* e) {
    return guarded([&] {
        Stream s;
        HostVecs hv;
        const int32_t n = F->n;
        double* dr = hv.make(n);
        double* dy = hv.make(n);
        double* dx = hv.make(n);
        double* de = hv.make(n);
        int* tk = reinterpret_cast<int*>(hv.make(kSweepScratchInts / 2));  // ticket + per-sweep scratch
        PMG_CUDA(cudaMemcpyAsync(dr, r, sizeof(double) * n, cudaMemcpyHostToDevice, s.s));
        PMG_CUDA(cudaMemsetAsync(de, 0, sizeof(double) * n, s.s));
        apply_factor(F, dr, dy, dx, de, tk, s.s);
        PMG_CUDA(cudaMemcpyAsync(e, de, sizeof(double) * n, cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return PMG_OK;
    });
}

int pmg_factor_stats(pmg_factor F, int64_t* nnz_L, int64_t* nnz_U, int32_t* levels_L, int32_t* levels_U,
                     int32_t* max_row_L, int32_t* max_row_U) {
    if (nnz_L) *nnz_L = F->L.nnz;
    if (nnz_U) *nnz_U = F->U.nnz;
    if (levels_L || levels_U) {
        const int rc = guarded([&] {
            Stream s;
            F->ensure_levels(s.s);
            return int(PMG_OK);
        });
        if (rc != PMG_OK) return rc;
    }
    if (levels_L) *levels_L = F->lvL.nlevels;
    if (levels_U) *levels_U = F->lvU.nlevels;
    if (max_row_L) *max_row_L = F->max_row_L;
    if (max_row_U) *max_row_U = F->max_row_U;
    return PMG_OK;
}

int pmg_factor_sweep_info(pmg_factor F, int32_t* kind, int32_t* seg, int32_t* skew_D_L, int32_t* skew_D_U) {
    if (kind) *kind = F->wave ? PMG_SWEEP_WAVE : F->skew ? PMG_SWEEP_SKEW : F->seg > 0 ? PMG_SWEEP_CHAIN : PMG_SWEEP_LEVELS;
    if (seg) *seg = F->seg;
    if (skew_D_L) *skew_D_L = F->wave ? F->waveL.lead : F->skew ? F->planL.lead : 0;
    if (skew_D_U) *skew_D_U = F->wave ? F->waveU.lead : F->skew ? F->planU.lead : 0;
    return PMG_OK;
}

int pmg_factor_export(pmg_factor F, int32_t* Lrp, int32_t* Lc, double* Lv, int32_t* Urp, int32_t* Uc, double* Uv,
                      int32_t* perm) {
    return guarded([&] {
        const int32_t n = F->n;
        auto cp = [](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) PMG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        };
        cp(Lrp, F->L.rowptr, sizeof(int32_t) * (n + 1));
        cp(Lc, F->L.col, sizeof(int32_t) * F->L.nnz);
        cp(Lv, F->L.val, sizeof(double) * F->L.nnz);
        cp(Urp, F->U.rowptr, sizeof(int32_t) * (n + 1));
        cp(Uc, F->U.col, sizeof(int32_t) * F->U.nnz);
        cp(Uv, F->U.val, sizeof(double) * F->U.nnz);
        if (perm) {
            if (F->h_perm.empty())
                for (int32_t i = 0; i < n; ++i) perm[i] = i;
            else
                std::copy(F->h_perm.begin(), F->h_perm.end(), perm);
        }
        return PMG_OK;
    });
}

int pmg_hier_create(const pmg_hier_desc* d, pmg_hier* out, int* err_level, int64_t* err_row) {
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        if (!d || d->n_plevels < 1 || d->n_hlevels < 1) throw ArgError("hierarchy: need >= 1 p- and h-level", PMG_ERR_ARG);
        if (d->degrees[d->n_plevels - 1] != 1) throw ArgError("hierarchy: last p-level must have degree 1", PMG_ERR_ARG);
        if (d->nu1 < 0 || d->nu2 < 0) throw ArgError("hierarchy: nu1, nu2 >= 0", PMG_ERR_ARG);
        Stream s;
        auto H = std::make_unique<pmg_hier_s>();
        H->smoother = d->smoother;
        H->nu1 = d->nu1;
        H->nu2 = d->nu2;
        const int np = d->n_plevels, nh = d->n_hlevels;
        H->pl.resize(np);
        for (int l = 0; l < np; ++l) {
            check_view(&d->A[l]);
            PLev& L = H->pl[l];
            L.degree = d->degrees[l];
            L.A = make_csr(d->A[l], s.s);
            L.ML = dalloc<double>(L.A->A.n);
            PMG_CUDA(cudaMemcpyAsync(L.ML, d->ML[l], sizeof(double) * L.A->A.n, cudaMemcpyHostToDevice, s.s));
            if (l + 1 < np) {
                check_view(&d->P[l]);
                check_view(&d->PT[l]);
                if (d->P[l].nrows != d->A[l].nrows || d->P[l].ncols != d->A[l + 1].nrows ||
                    d->PT[l].nrows != d->P[l].ncols || d->PT[l].ncols != d->P[l].nrows)
                    throw ArgError("hierarchy: transfer dimensions", PMG_ERR_DIM);
                L.P = make_csr(d->P[l], s.s);
                L.PT = make_csr(d->PT[l], s.s);
            }
        }
        for (int l = 0; l + 1 < np; ++l) {
            if (H->smoother != PMG_SMOOTHER_ILUT) {
                ensure_gs(H->pl[l].A, s.s);
                if (H->pl[l].A->gs_zero_row >= 0) {
                    if (err_level) *err_level = l;
                    if (err_row) *err_row = H->pl[l].A->gs_zero_row;
                    return int(PMG_ZERO_DIAG);
                }
            }
        }
        H->hl.resize(nh);
        for (int j = 0; j < nh; ++j) {
            HLev& L = H->hl[j];
            if (j == 0) {
                L.A = H->pl.back().A;
            } else {
                check_view(&d->HA[j]);
                L.A = make_csr(d->HA[j], s.s);
                L.own_A = true;
            }
            if (j + 1 < nh) {
                check_view(&d->HP[j]);
                check_view(&d->HPT[j]);
                L.P = make_csr(d->HP[j], s.s);
                L.PT = make_csr(d->HPT[j], s.s);
            }
        }
        PMG_CUDA(cudaStreamSynchronize(s.s));
        // ILUT of every level at once: each factorisation is a row-to-row chain that keeps only a
        // few dozen CTAs busy, so the levels' chains run side by side on their own streams (the
        // largest first; grids capped so that all of them are resident together)
        struct Slot {
            pmg_csr_s* A;
            pmg_factor_s** F;
            int level;
            PendingFactor pf;
            std::unique_ptr<Stream> st;
        };
        std::vector<Slot> slots;
        if (H->smoother == PMG_SMOOTHER_ILUT)
            for (int l = 0; l + 1 < np; ++l) slots.push_back({H->pl[l].A, &H->pl[l].F, l, {}, nullptr});
        for (int j = 0; j + 1 < nh; ++j) slots.push_back({H->hl[j].A, &H->hl[j].F, np - 1 + j, {}, nullptr});
        cudaEvent_t ref = nullptr;
        PMG_CUDA(cudaEventCreate(&ref));
        struct Cleanup {  // on an error path: wait for and drop the factorisations still in flight
            std::vector<Slot>& sl;
            cudaEvent_t ev;
            ~Cleanup() {
                for (auto& x : sl)
                    if (x.pf.job) {
                        DevCsr l, u;
                        try {
                            ilut_finish(x.pf.job, l, u, nullptr, nullptr, nullptr, nullptr);
                        } catch (...) {
                        }
                        x.pf.job = nullptr;
                        l.free();
                        u.free();
                        x.pf.owned.free();
                    }
                cudaEventDestroy(ev);
            }
        } cleanup{slots, ref};
        static const bool serial = env_int("PMG_ILUT_SERIAL", 0) != 0;
        const int nsm = sm_count();
        double ilut_s = 0;
        if (serial || slots.size() < 2) {
            for (auto& x : slots) {
                int rc = make_factor(x.A, d->tau, d->fillfactor, d->ordering, x.F, err_row, s.s);
                if (rc) {
                    if (err_level) *err_level = x.level;
                    return rc;
                }
                ilut_s += (*x.F)->seconds;
            }
        } else {
            for (size_t q = 0; q < slots.size(); ++q) {
                Slot& x = slots[q];
                x.st = std::make_unique<Stream>();
                if (q == 0) PMG_CUDA(cudaEventRecord(ref, x.st->s));
                const bool heavy = x.A->A.nnz >= int64_t(32) * std::max(x.A->A.n, 1);
                x.pf = factor_begin(x.A, d->tau, d->fillfactor, d->ordering, heavy ? nsm + nsm / 2 : 32, x.st->s);
            }
            for (auto& x : slots) {
                double since = 0;
                int rc = factor_end(x.pf, x.F, err_row, s.s, ref, &since);
                if (rc) {
                    if (err_level) *err_level = x.level;
                    return rc;
                }
                ilut_s = std::max(ilut_s, since);
            }
        }
        {
            const int k = dense_setup(H->coarse, H->hl[nh - 1].A->A, s.s);
            if (k >= 0) {
                if (err_level) *err_level = np - 1 + nh - 1;
                if (err_row) *err_row = k;
                return int(PMG_ZERO_PIVOT);
            }
        }
        PMG_CUDA(cudaStreamSynchronize(s.s));
        size_t fr = 0, tot = 0;
        PMG_CUDA(cudaMemGetInfo(&fr, &tot));
        H->stats.device_bytes = int64_t(tot - fr);
        H->stats.ilut_seconds = ilut_s;
        H->stats.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = H.release();
        return int(PMG_OK);
    });
}

int pmg_hier_destroy(pmg_hier H) {
    delete H;
    return PMG_OK;
}

int pmg_hier_get_stats(pmg_hier H, pmg_hier_stats* s) {
    *s = H->stats;
    return PMG_OK;
}

int pmg_hier_factor(pmg_hier H, int which, pmg_factor* out) {
    const int np = int(H->pl.size());
    if (which < np - 1) {
        *out = H->pl[which].F;
    } else {
        int j = which - (np - 1);
        if (j < 0 || j >= int(H->hl.size()) - 1) return PMG_ERR_ARG;
        *out = H->hl[j].F;
    }
    return *out ? PMG_OK : PMG_ERR_ARG;
}

int pmg_work_create(pmg_hier H, pmg_work* out) {
    return guarded([&] {
        auto W = std::make_unique<pmg_work_s>();
        W->H = H;
        PMG_CUDA(cudaStreamCreateWithFlags(&W->st, cudaStreamNonBlocking));
        W->pw.resize(H->pl.size());
        for (size_t l = 0; l < H->pl.size(); ++l) {
            const size_t n = H->pl[l].A->A.n;
            PWork& w = W->pw[l];
            w.u[0] = dalloc<double>(n);
            w.u[1] = dalloc<double>(n);
            w.f = dalloc<double>(n);
            w.r = dalloc<double>(n);
            w.y = dalloc<double>(n);
            w.x = dalloc<double>(n);
        }
        W->hw.resize(H->hl.size());
        for (size_t j = 0; j < H->hl.size(); ++j) {
            const size_t n = H->hl[j].A->A.n;
            HWork& w = W->hw[j];
            w.e = dalloc<double>(n);
            w.r = dalloc<double>(n);
            w.res = dalloc<double>(n);
            w.y = dalloc<double>(n);
            w.x = dalloc<double>(n);
        }
        W->ticket = reinterpret_cast<int*>(dalloc<double>(kSweepScratchInts / 2));  // ticket + per-sweep scratch
        const int32_t n0 = H->pl[0].A->A.n;
        W->nc.partials = dalloc<double>(ceil_div(n0, 256) + 1);
        W->nc.counter = reinterpret_cast<unsigned*>(dalloc<double>(1));
        // the norm's last-block counter must be zero before the first fused residual on W->st
        // (a non-blocking stream: order the reset on that stream and wait for it)
        PMG_CUDA(cudaMemsetAsync(W->nc.counter, 0, sizeof(double), W->st));
        W->norm0 = dalloc<double>(1);
        W->rho_dev = dalloc<double>(1);
        PMG_CUDA(cudaMallocHost(&W->rho_host, sizeof(double)));
        ensure_hist(*W, 200);
        PMG_CUDA(cudaStreamSynchronize(W->st));
        *out = W.release();
        return PMG_OK;
    });
}

int pmg_work_destroy(pmg_work W) {
    delete W;
    return PMG_OK;
}

int pmg_solve_device(pmg_work W, const double* d_f, double* d_u, double tol, int max_cycles, double* rho_hist,
                     int* cycles, int* flags, double* solve_seconds) {
    return guarded([&] {
        if (max_cycles < 0) throw ArgError("max_cycles < 0", PMG_ERR_ARG);
        const int32_t n = W->H->pl[0].A->A.n;
        PWork& w0 = W->pw[0];
        w0.cur = 0;
        PMG_CUDA(cudaMemcpyAsync(w0.u[0], d_u, sizeof(double) * n, cudaMemcpyDeviceToDevice, W->st));
        int rc = solve_loop(*W, d_f, tol, max_cycles, rho_hist, cycles, flags, solve_seconds);
        PMG_CUDA(cudaMemcpyAsync(d_u, w0.u[w0.cur], sizeof(double) * n, cudaMemcpyDeviceToDevice, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

int pmg_solve(pmg_work W, const double* f, double* u_inout, double tol, int max_cycles, double* rho_hist, int* cycles,
              int* flags, double* solve_seconds) {
    return guarded([&] {
        if (max_cycles < 0) throw ArgError("max_cycles < 0", PMG_ERR_ARG);
        const int32_t n = W->H->pl[0].A->A.n;
        PWork& w0 = W->pw[0];
        w0.cur = 0;
        PMG_CUDA(cudaMemcpyAsync(w0.f, f, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        PMG_CUDA(cudaMemcpyAsync(w0.u[0], u_inout, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        int rc = solve_loop(*W, w0.f, tol, max_cycles, rho_hist, cycles, flags, solve_seconds);
        PMG_CUDA(cudaMemcpyAsync(u_inout, w0.u[w0.cur], sizeof(double) * n, cudaMemcpyDeviceToHost, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

int pmg_bicgstab_device(pmg_work W, const double* d_f, double* d_u, double tol, int max_iter, double* res_hist,
                        int* iters, int* flags, double* solve_seconds) {
    return guarded([&] {
        if (max_iter < 0) throw ArgError("max_iter < 0", PMG_ERR_ARG);
        ensure_krylov(*W);
        const int32_t n = W->H->pl[0].A->A.n;
        PMG_CUDA(cudaMemcpyAsync(W->kv[0], d_u, sizeof(double) * n, cudaMemcpyDeviceToDevice, W->st));
        int rc = bicgstab_loop(*W, d_f, tol, max_iter, res_hist, iters, flags, solve_seconds);
        PMG_CUDA(cudaMemcpyAsync(d_u, W->kv[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

int pmg_bicgstab(pmg_work W, const double* f, double* u_inout, double tol, int max_iter, double* res_hist, int* iters,
                 int* flags, double* solve_seconds) {
    return guarded([&] {
        if (max_iter < 0) throw ArgError("max_iter < 0", PMG_ERR_ARG);
        ensure_krylov(*W);
        const int32_t n = W->H->pl[0].A->A.n;
        PWork& w0 = W->pw[0];
        PMG_CUDA(cudaMemcpyAsync(w0.f, f, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        PMG_CUDA(cudaMemcpyAsync(W->kv[0], u_inout, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        int rc = bicgstab_loop(*W, w0.f, tol, max_iter, res_hist, iters, flags, solve_seconds);
        PMG_CUDA(cudaMemcpyAsync(u_inout, W->kv[0], sizeof(double) * n, cudaMemcpyDeviceToHost, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

int pmg_cycle(pmg_work W, int level, double* u, const double* f) {
    return guarded([&] {
        pmg_hier_s& H = *W->H;
        if (level < 0 || level >= int(H.pl.size())) throw ArgError("cycle: bad level", PMG_ERR_ARG);
        const int32_t n = H.pl[level].A->A.n;
        PWork& w = W->pw[level];
        w.cur = 0;
        // f must live in a buffer the cycle does not overwrite: use the level's y buffer
        // only as a staging area for the coarse levels; level f buffers are overwritten by
        // restriction, so stage into a dedicated allocation.
        HostVecs hv;
        double* df = hv.make(n);
        PMG_CUDA(cudaMemcpyAsync(df, f, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        PMG_CUDA(cudaMemcpyAsync(w.u[0], u, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        int rc = vcycle(*W, level, df, nullptr, false);
        PMG_CUDA(cudaMemcpyAsync(u, w.u[w.cur], sizeof(double) * n, cudaMemcpyDeviceToHost, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

// One smoothing step (GS: SPEC.md:233-241) or one coarse-grid correction
// (steps 2-4 of the cycle, PAPER §4 "referred to as 'coarse grid correction'": restrict the
// residual, one cycle at level+1 from zero, prolongate and add) at p-level `level`, on host
// vectors; the building blocks of reduction_factors.
static int part_step(pmg_work W, int level, double* u, const double* f, bool cgc) {
    return guarded([&] {
        pmg_hier_s& H = *W->H;
        const int top = int(H.pl.size()) - 1 - (cgc ? 1 : 0);
        if (level < 0 || level > top) throw ArgError(cgc ? "coarse_correction: bad level" : "smooth: bad level", PMG_ERR_ARG);
        PLev& L = H.pl[level];
        const int32_t n = L.A->A.n;
        PWork& w = W->pw[level];
        w.cur = 0;
        HostVecs hv;
        double* df = hv.make(n);
        PMG_CUDA(cudaMemcpyAsync(df, f, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        PMG_CUDA(cudaMemcpyAsync(w.u[0], u, sizeof(double) * n, cudaMemcpyHostToDevice, W->st));
        int rc = PMG_OK;
        if (!cgc) {
            if (level == int(H.pl.size()) - 1) {  // p = 1: the ILUT smoother of the finest h-level
                HLev& hl = H.hl[0];
                if (!hl.F) throw ArgError("smooth: the p = 1 level is the dense coarsest level", PMG_ERR_ARG);
                smooth_ilut(*W, hl.A, hl.F, w.u[0], df, nullptr, w.r, w.y, w.x, false);
            } else {
                rc = smooth(*W, level, df, nullptr);
            }
        } else {
            PLev& C = H.pl[level + 1];
            PWork& c = W->pw[level + 1];
            W->run(kClsResid0, 1, [&] { sell_rowop(L.A->S, kOpResidual, w.u[0], df, nullptr, w.r, nullptr, W->st); });
            W->run(kClsTransfer, 1, [&] { sell_rowop(L.PT->S, kOpRestrict, w.r, nullptr, C.ML, c.f, nullptr, W->st); });
            PMG_CUDA(cudaMemsetAsync(c.u[c.cur], 0, sizeof(double) * C.A->A.n, W->st));
            rc = vcycle(*W, level + 1, c.f, nullptr, true);
            if (!rc)
                W->run(kClsTransfer, 1,
                       [&] { sell_rowop(L.P->S, kOpProlongAdd, c.u[c.cur], nullptr, L.ML, w.u[0], nullptr, W->st); });
        }
        PMG_CUDA(cudaMemcpyAsync(u, w.u[w.cur], sizeof(double) * n, cudaMemcpyDeviceToHost, W->st));
        PMG_CUDA(cudaStreamSynchronize(W->st));
        return rc;
    });
}

int pmg_smooth(pmg_work W, int level, double* u, const double* f) { return part_step(W, level, u, f, false); }

int pmg_coarse_correction(pmg_work W, int level, double* u, const double* f) {
    return part_step(W, level, u, f, true);
}

int pmg_prolongate(pmg_hier H, int level, const double* vc, double* vf) {
    return guarded([&] {
        if (level < 0 || level + 1 >= int(H->pl.size())) throw ArgError("prolongate: bad level", PMG_ERR_ARG);
        PLev& L = H->pl[level];
        Stream s;
        HostVecs hv;
        double* dc = hv.make(L.P->A.m);
        double* df = hv.make(L.P->A.n);
        PMG_CUDA(cudaMemcpyAsync(dc, vc, sizeof(double) * L.P->A.m, cudaMemcpyHostToDevice, s.s));
        sell_rowop(L.P->S, kOpRestrict, dc, nullptr, L.ML, df, nullptr, s.s);  // (P v) / ML
        PMG_CUDA(cudaMemcpyAsync(vf, df, sizeof(double) * L.P->A.n, cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return PMG_OK;
    });
}

int pmg_restrict(pmg_hier H, int level, const double* rf, double* rc) {
    return guarded([&] {
        if (level < 0 || level + 1 >= int(H->pl.size())) throw ArgError("restrict: bad level", PMG_ERR_ARG);
        PLev& L = H->pl[level];
        PLev& C = H->pl[level + 1];
        Stream s;
        HostVecs hv;
        double* dr = hv.make(L.PT->A.m);
        double* dc = hv.make(L.PT->A.n);
        PMG_CUDA(cudaMemcpyAsync(dr, rf, sizeof(double) * L.PT->A.m, cudaMemcpyHostToDevice, s.s));
        sell_rowop(L.PT->S, kOpRestrict, dr, nullptr, C.ML, dc, nullptr, s.s);
        PMG_CUDA(cudaMemcpyAsync(rc, dc, sizeof(double) * L.PT->A.n, cudaMemcpyDeviceToHost, s.s));
        PMG_CUDA(cudaStreamSynchronize(s.s));
        return PMG_OK;
    });
}

// diagnostics: enable (1) / disable (0) per-segment tracing of chained sweeps; or (-1) copy the
// trace of the last sweep (6 u64 per segment) into out (cap entries); returns #segments
int pmg_debug_chain_trace(int mode, unsigned long long* out, int cap) {
    if (mode == 1 || mode == 0) {
        g_chain_trace_on = mode == 1;
        return 0;
    }
    if (!g_chain_trace || !out) return 0;
    const int n = std::min(g_chain_trace_n * 6 + kChainTraceExtra, cap);
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpy(out, g_chain_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return g_chain_trace_n;
}

// diagnostics: the same for the skewed-warp sweeps (4 u64 per warp block); returns #blocks
int pmg_debug_skew_trace(int mode, unsigned long long* out, int cap) {
    if (mode == 1 || mode == 0) {
        g_skew_trace_on = mode == 1;
        return 0;
    }
    if (!g_skew_trace || !out) return 0;
    const int n = std::min(g_skew_trace_n * 8, cap);
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpy(out, g_skew_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return g_skew_trace_n;
}

// diagnostics: the same for the rotating-lane sweeps (4 u64 per warp block); returns #blocks
int pmg_debug_wave_trace(int mode, unsigned long long* out, int cap) {
    if (mode == 1 || mode == 0) {
        g_wave_trace_on = mode == 1;
        return 0;
    }
    if (!g_wave_trace || !out) return 0;
    const int n = std::min(g_wave_trace_n * 8, cap);
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpy(out, g_wave_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return g_wave_trace_n;
}

// diagnostics: mode 1/0 turns keeping a copy of every wave sweep's output on/off; mode 2+kind
// copies the last output of that kind (0 L, 1 U, 2 GS; v-space) into out; returns its length
int pmg_debug_wave_dump(int mode, double* out, int cap) {
    if (mode == 0 || mode == 1) {
        g_wave_dump = mode == 1;
        return 0;
    }
    const int k = mode - 2;
    if (k < 0 || k > 2 || !g_wave_dump_buf[k]) return 0;
    const int n = std::min(g_wave_dump_n[k], cap);
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpy(out, g_wave_dump_buf[k], sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return n;
}

// ms_by_class[0..6]: resid(A_p), L-solve(p), U-solve(p), GS(p), p-transfers, coarse (p<finest and
// h-MG), misc; [7] = total launches, [8..14] = launches per class.  enable: n_classes < 0 turns
// profiling on (-1) / off (-2) and resets the counters.
int pmg_work_kernel_times(pmg_work W, double* ms, int n) {
    return guarded([&] {
        if (n < 0) {
            W->collect();
            W->prof = (n == -1);
            for (int c = 0; c < kNumCls; ++c) {
                W->cls_ms[c] = 0;
                W->cls_launches[c] = 0;
            }
            W->launches = 0;
            return PMG_OK;
        }
        W->collect();
        for (int c = 0; c < n && c < kNumCls; ++c) ms[c] = W->cls_ms[c];
        if (n > kNumCls) ms[kNumCls] = double(W->launches);
        for (int c = 0; c < kNumCls && kNumCls + 1 + c < n; ++c) ms[kNumCls + 1 + c] = double(W->cls_launches[c]);
        return PMG_OK;
    });
}

}  // extern "C"
