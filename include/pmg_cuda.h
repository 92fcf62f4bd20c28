/* pmg_cuda.h -- C ABI of the B200 p-multigrid solve path (libpmg_cuda.so).
 *
 * THE DROP-IN BOUNDARY.  The reference declares no solver entry points
 * (proj/include/iga/splines.hpp:1-56 and proj/include/iga/types.hpp:1-44 contain only
 * spline and type declarations); the operations below are the `sparselin` and `pmg`
 * operations of SPEC.md, which the reference's C++ API would expose.  Each entry point
 * names the SPEC operation it replaces.  Host code (include/iga/pmg.hpp, the Python
 * mirror in paper_1901_01685_b200/pmg.py) binds exactly these symbols.
 *
 * Conventions:
 *   - plain pointers and sizes; CSR with int32 offsets/columns, sorted unique columns,
 *     fp64 values (types.hpp:19-20);
 *   - every call returns a status code (PMG_OK, ...); `err_row` (may be NULL) receives
 *     the failing row for PMG_ZERO_PIVOT / PMG_ZERO_DIAG (types.hpp:31-34
 *     FactorizationError{row});
 *   - divergence is a report flag, never an error;
 *   - handles are immutable after creation except pmg_work; one host thread per
 *     pmg_work (SPEC.md:395-396 concurrent solves on one hierarchy);
 *   - no CPU fallback: without a usable CUDA device every call returns PMG_ERR_CUDA.
 */
#ifndef PMG_CUDA_H
#define PMG_CUDA_H

#include <stdint.h>

#include "pmg_asm.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PMG_OK = 0,
    PMG_ZERO_PIVOT = 1, /* ILUT: zero pivot at err_row            */
    PMG_ZERO_DIAG = 2,  /* Gauss-Seidel: zero/missing diagonal     */
    PMG_ERR_DIM = 3,    /* dimension mismatch                      */
    PMG_ERR_CUDA = 4,   /* CUDA runtime failure / no device                      */
    PMG_ERR_OOM = 5,
    PMG_ERR_ARG = 6     /* invalid argument (tau < 0, fillfactor < 1, bad CSR)   */
};

enum { PMG_SMOOTHER_ILUT = 0, PMG_SMOOTHER_GS = 1 };
enum { PMG_ORDER_NONE = 0, PMG_ORDER_RCM = 1 };
enum { PMG_FLAG_CONVERGED = 1, PMG_FLAG_DIVERGED = 2, PMG_FLAG_BREAKDOWN = 4 };

/* read-only host CSR view (borrowed; copied at create) */
typedef struct pmg_csr_view {
    int32_t nrows, ncols;
    const int32_t* rowptr; /* nrows+1 */
    const int32_t* col;    /* rowptr[nrows] */
    const double* val;
} pmg_csr_view;

typedef struct pmg_csr_s* pmg_csr;       /* device CSR (+ sliced layout)        */
typedef struct pmg_factor_s* pmg_factor; /* ILUT factors L, U, perm, level sets */
typedef struct pmg_hier_s* pmg_hier;     /* immutable device hierarchy          */
typedef struct pmg_work_s* pmg_work;     /* per-solve vectors + stream          */

const char* pmg_status_string(int status);
const char* pmg_last_error(void);
int pmg_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- sparselin ---- */
int pmg_csr_create(const pmg_csr_view* A, pmg_csr* out);                           /* SparseMatrixCsr */
int pmg_csr_destroy(pmg_csr A);
int pmg_spmv(pmg_csr A, const double* x, double* y);                               /* spmv, host x/y */
int pmg_residual(pmg_csr A, const double* x, const double* f, double* r, double* norm2); /* r = f - A x, ||r||_2 */
int pmg_gs_sweep(pmg_csr A, double* u, const double* f, int64_t* err_row);         /* gauss_seidel_sweep */
int pmg_rcm_ordering(const pmg_csr_view* A, int32_t* perm);                        /* rcm_ordering, perm[new]=old */
int pmg_ilut_factorize(pmg_csr A, double tau, double fillfactor, int ordering,
                       pmg_factor* out, int64_t* err_row);                         /* ilut_factorize */
int pmg_factor_destroy(pmg_factor F);
int pmg_ilut_apply(pmg_factor F, const double* r, double* e);                      /* ilut_apply */
/* factor introspection: nnz, level counts (north star: level count + rows/level) */
int pmg_factor_stats(pmg_factor F, int64_t* nnz_L, int64_t* nnz_U, int32_t* levels_L, int32_t* levels_U,
                     int32_t* max_row_L, int32_t* max_row_U);
/* which sweep kernels apply_factor uses for F (no reference counterpart; reporting):
 * level-scheduled, chained segments (seg = grid-row length) or skewed warps (lane skew D) */
enum { PMG_SWEEP_LEVELS = 0, PMG_SWEEP_CHAIN = 1, PMG_SWEEP_SKEW = 2, PMG_SWEEP_WAVE = 3 };
int pmg_factor_sweep_info(pmg_factor F, int32_t* kind, int32_t* seg, int32_t* skew_D_L, int32_t* skew_D_U);
/* copy factors to host CSR arrays (L strictly lower, unit diagonal implicit; U with
 * diagonal); pass NULL arrays to query sizes only.  perm may be NULL. */
int pmg_factor_export(pmg_factor F, int32_t* L_rowptr, int32_t* L_col, double* L_val, int32_t* U_rowptr,
                      int32_t* U_col, double* U_val, int32_t* perm);

/* ---- pmg ---- */
typedef struct pmg_hier_desc {
    int n_plevels;               /* p-levels, degree list descending, last is p = 1 */
    const int* degrees;          /* [n_plevels] */
    const pmg_csr_view* A;       /* [n_plevels] rediscretised operators A_k          */
    const double* const* ML;     /* [n_plevels] lumped masses      */
    const pmg_csr_view* P;       /* [n_plevels-1] P[l]: level l+1 -> level l         */
    const pmg_csr_view* PT;      /* [n_plevels-1] transposes (restriction)           */
    int n_hlevels;               /* p=1 h-levels incl. the finest (= last p-level)  */
    const pmg_csr_view* HA;      /* [n_hlevels], HA[0] unused                        */
    const pmg_csr_view* HP;      /* [n_hlevels-1] HP[j]: h-level j+1 -> j            */
    const pmg_csr_view* HPT;     /* [n_hlevels-1]                                    */
    int smoother;                /* PMG_SMOOTHER_* on the p-levels; h-MG always ILUT */
    int nu1, nu2;                /* default 1, 1                       */
    double tau, fillfactor;      /* ILUT(1e-12, 1)                      */
    int ordering;                /* PMG_ORDER_*                                      */
} pmg_hier_desc;

typedef struct pmg_hier_stats {
    double setup_seconds;        /* device setup incl. GPU ILUT factorisations */
    double ilut_seconds;
    int64_t device_bytes;
} pmg_hier_stats;

int pmg_hier_create(const pmg_hier_desc* d, pmg_hier* out, int* err_level, int64_t* err_row); /* build_hierarchy */
int pmg_hier_destroy(pmg_hier H);
int pmg_hier_get_stats(pmg_hier H, pmg_hier_stats* s);
/* factor of p-level l (l < n_plevels-1, ILUT smoother) or h-level j (as n_plevels-1+j) */
int pmg_hier_factor(pmg_hier H, int which, pmg_factor* out);
int pmg_work_create(pmg_hier H, pmg_work* out);
int pmg_work_destroy(pmg_work W);

/* solve: u_inout holds u0 on entry, u on exit (host arrays).
 * rho_hist[0..*cycles] receives ||f-Au_c||/||f-Au_0|| (rho_hist[0] = 1); it must hold
 * max_cycles+1 entries.  flags |= PMG_FLAG_CONVERGED / PMG_FLAG_DIVERGED (>1e10).
 * solve_seconds = device time of the cycle loop (CUDA events), excluding H2D/D2H. */
int pmg_solve(pmg_work W, const double* f, double* u_inout, double tol, int max_cycles, double* rho_hist,
              int* cycles, int* flags, double* solve_seconds);
/* the same with device-resident f/u (pointers into device memory, e.g. torch tensors) */
int pmg_solve_device(pmg_work W, const double* d_f, double* d_u, double tol, int max_cycles, double* rho_hist,
                     int* cycles, int* flags, double* solve_seconds);
/* BiCGSTAB right-preconditioned by one
 * V-cycle from zero guess per preconditioning phase (as_preconditioner).
 * res_hist[0..*iters] receives ||r_i||/||f-Au_0|| of the recursively updated residual
 * (res_hist[0] = 1; max_iter+1 entries); flags |= PMG_FLAG_CONVERGED / PMG_FLAG_DIVERGED /
 * PMG_FLAG_BREAKDOWN (rho = 0, (rh,v) = 0 or omega = 0).  Replaces the
 * reference's bicgstab(A, f, as_preconditioner(hier), tol, max_iter) -> (u, KrylovReport). */
int pmg_bicgstab(pmg_work W, const double* f, double* u_inout, double tol, int max_iter, double* res_hist,
                 int* iters, int* flags, double* solve_seconds);
int pmg_bicgstab_device(pmg_work W, const double* d_f, double* d_u, double tol, int max_iter, double* res_hist,
                        int* iters, int* flags, double* solve_seconds);
/* one cycle at p-level `level` on host vectors (u updated in place) */
int pmg_cycle(pmg_work W, int level, double* u, const double* f);
/* one smoothing step (ILUT or GS, the hierarchy's smoother; p = 1: the ILUT smoother of the
 * finest h-level) / one coarse-grid correction (restrict f - A u, one cycle at level+1 from
 * zero, prolongate and add: PAPER §4 steps 2-4) at p-level `level`, host vectors, u in place.
 * The two halves of the cycle that reduction_factors applies separately. */
int pmg_smooth(pmg_work W, int level, double* u, const double* f);
int pmg_coarse_correction(pmg_work W, int level, double* u, const double* f);
/* prolongate: v_fine = ML_l^-1 P_l v_coarse; restrict */
int pmg_prolongate(pmg_hier H, int level, const double* v_coarse, double* v_fine);
int pmg_restrict(pmg_hier H, int level, const double* r_fine, double* r_coarse);

/* timing helpers for the bench: run `cycles` V-cycles from the state left by the last
 * pmg_solve_device call and report per-kernel-class device time (ms). */
int pmg_work_kernel_times(pmg_work W, double* ms_by_class, int n_classes);

/* ---- discretization: GPU assembly of matrix values (F2) ----
 * assemble_system / assemble_mass / assemble_transfer: the values of one operator on the sparsity
 * pattern and tables of the request (include/pmg_asm.h), element matrices by sum factorisation and a
 * deterministic gather; bit-identical to the host element loop of libiga_host.so.
 * Matches pmg_asm_values_fn: pass it to iga_problem_build_with (include/iga_host.h). */
int pmg_asm_values(const pmg_asm_request* req);

/* diagnostics: mode 1/0 enables/disables per-segment globaltimer tracing of the chained
 * sweeps; mode -1 copies the trace of the last sweep (6 u64 per segment: claim, helpers done,
 * finisher start, finisher end, helper value spins, finisher batch waits) and returns the
 * number of segments */
int pmg_debug_chain_trace(int mode, unsigned long long* out, int cap);
/* the same for the skewed-warp sweeps: 4 u64 per 32-segment warp block */
int pmg_debug_skew_trace(int mode, unsigned long long* out, int cap);
/* the same for the rotating-lane sweeps: 4 u64 per warp block */
int pmg_debug_wave_trace(int mode, unsigned long long* out, int cap);
/* keep (mode 1) / drop (0) a copy of every rotating-lane sweep's output; mode 2 + kind (L 0, U 1,
 * GS 2) copies the last one (v-space) into out; returns its length */
int pmg_debug_wave_dump(int mode, double* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
