/* C ABI of the host-side discretization library (libiga_host.so).
 *
 * This is INPUT GENERATION for the solve path (discretization stays on
 * the host): it assembles the FP64 CSR operators of one problem -- A_k and lumped
 * masses per p-level, transfers P^k_j, the p=1 h-chain with
 * knot-insertion prolongations -- plus f and the initial guess
 * (SPEC.md:516-524).  The reference declares no such entry points (it has no
 * assembler); the names follow SPEC.md's `discretization` module.
 *
 * All functions return 0 on success, -1 on error (message via iga_last_error()).
 */
#ifndef IGA_HOST_H
#define IGA_HOST_H

#include <stdint.h>

#include "pmg_asm.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { IGA_GEOM_SQUARE = 0, IGA_GEOM_ANNULUS = 1, IGA_GEOM_LSHAPE = 2 };
enum { IGA_RHS_SINSIN = 0, IGA_RHS_ANNULUS = 1, IGA_RHS_ONE = 2, IGA_RHS_B1 = 3, IGA_RHS_B2 = 4, IGA_RHS_B3 = 5 };
enum { IGA_MAT_A = 0, IGA_MAT_P = 1, IGA_MAT_PT = 2, IGA_MAT_HA = 3, IGA_MAT_HP = 4, IGA_MAT_HPT = 5 };
enum { IGA_VEC_ML = 0, IGA_VEC_F = 1, IGA_VEC_U0 = 2 };
/* multipatch DOF numbering: patch-major (glued DOFs keep the lower patch's index) or global
 * row-major over the domain's control grid (y, then x ascending) */
enum { IGA_NUMBER_PATCH = 0, IGA_NUMBER_ROWMAJOR = 1 };

typedef struct iga_problem_spec {
    int geometry;        /* IGA_GEOM_* */
    int rhs;             /* IGA_RHS_* */
    double D[4];         /* diffusion tensor, row-major */
    double v[2];         /* velocity */
    double R;            /* reaction */
    int h_exp;           /* h = 2^-h_exp, elements per direction (per patch) = 2^h_exp */
    int coarsest_h_exp;  /* h-MG coarsest level, default 2 (h = 1/4) */
    int n_degrees;       /* degree list, strictly decreasing, ending at 1 */
    int degrees[8];
    int random_guess;    /* 0: u0 = 0; 1: splitmix64(seed) mapped to U[-1,1) */
    uint64_t seed;
    double nitsche_scale; /* multiplies the Nitsche penalty eta = 4 k^2 (0 -> 1) */
    int numbering;        /* IGA_NUMBER_* (multipatch only) */
} iga_problem_spec;

typedef struct iga_problem_s iga_problem;

const char* iga_last_error(void);
void iga_set_num_threads(int n);

/* fill *s with BASELINE.json config `config` (1..5); `degree` selects p for config 2 */
int iga_config_spec(int config, int degree, iga_problem_spec* s);
int iga_problem_build(const iga_problem_spec* s, iga_problem** out);
/* F2: the same build with the matrix VALUES produced by `values` (pmg_asm_values of
 * libpmg_cuda.so: GPU assembly); the host keeps numbering, patterns, tables,
 * the load vector, transposes and the h-chain prolongations.  NULL = host element loop. */
int iga_problem_build_with(const iga_problem_spec* s, pmg_asm_values_fn values, iga_problem** out);
void iga_problem_free(iga_problem* h);

int iga_problem_num_plevels(const iga_problem* h);
int iga_problem_num_hlevels(const iga_problem* h); /* includes the finest (= last p-level) */
int iga_problem_degree(const iga_problem* h, int plevel);

/* kind = IGA_MAT_*; l = p-level (A, P, PT) or h-level (HA, HP, HPT).
 * P of p-level l maps level l+1 -> l; HP of h-level j maps level j+1 -> j. */
int iga_problem_csr_shape(const iga_problem* h, int kind, int l, int32_t* nrows, int32_t* ncols, int64_t* nnz);
int iga_problem_csr_copy(const iga_problem* h, int kind, int l, int32_t* rowptr, int32_t* col, double* val);
/* borrowed pointers into the problem (valid until iga_problem_free): int64 offsets, columns, values */
int iga_problem_csr_arrays(const iga_problem* h, int kind, int l, const int64_t** rowptr, const int32_t** col,
                           const double** val);
int iga_problem_vec_len(const iga_problem* h, int kind, int l);
int iga_problem_vec_copy(const iga_problem* h, int kind, int l, double* out);

/* one operator on one space: kind 0 = CDR operator A (load f=1 in IGA_VEC_F), 1 = mass M,
 * 2 = transfer P^p_{p2}, 3 = mass + lumped mass (IGA_VEC_ML); read it back as p-level 0 */
int iga_matrix_build(int kind, int geometry, int p, int p2, int nel, const double* D, const double* v, double R,
                     double nitsche_scale, iga_problem** out);

int iga_matrix_build_with(int kind, int geometry, int p, int p2, int nel, const double* D, const double* v, double R,
                          double nitsche_scale, pmg_asm_values_fn values, iga_problem** out);

/* MatrixMarket I/O.  Reading accepts coordinate real / integer / pattern
 * matrices, general / symmetric / skew-symmetric (mirrored), and returns sorted CSR with duplicates
 * summed in file order: call iga_mm_read_shape, allocate, then iga_mm_read.  Writing emits
 * "coordinate real general" with %.17g values (exact round trip); comment may be NULL.  Vectors:
 * one-column "array" files or plain text, one value per line.  Return 0 / -1 (iga_mm_last_error). */
const char* iga_mm_last_error(void);
int iga_mm_read_shape(const char* path, int32_t* nrows, int32_t* ncols, int64_t* nnz);
int iga_mm_read(const char* path, int32_t* rowptr, int32_t* col, double* val);
int iga_mm_write(const char* path, int32_t nrows, int32_t ncols, const int32_t* rowptr, const int32_t* col,
                 const double* val, const char* comment);
int iga_mm_write_vector(const char* path, int32_t n, const double* v);
int iga_mm_read_vector_len(const char* path, int32_t* n);
int iga_mm_read_vector(const char* path, double* v);

/* SPEC.md:61-78 and :79-87 (used by the property tests) */
int iga_eval_basis(int p, int spans, double x, int with_deriv, double* N, double* dN);
int iga_geometry_map(int geometry, int patch, double xi, double eta, double* X, double* J);

#ifdef __cplusplus
}
#endif
#endif
