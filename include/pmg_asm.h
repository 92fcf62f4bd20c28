/* pmg_asm.h -- plain-C request of the GPU assembler (F2: SPEC.md:132-167).
 *
 * The reference has no assembler; the operations are SPEC.md's
 * `assemble_system`, `assemble_mass` (:141-149), `assemble_transfer`
 * (:150-158).  The host library (libiga_host.so, include/iga_host.h) keeps the integer
 * structure -- spaces, DOF numbering, sparsity pattern -- the 1D basis tables, the load
 * vector and the orchestration; the matrix VALUES of one operator are produced by whoever
 * implements `pmg_asm_values_fn`: libpmg_cuda.so's `pmg_asm_values` (include/pmg_cuda.h) on the
 * GPU.  The host assembler's own element loop is the CPU path the GPU result must equal bit for
 * bit, so the request carries the host's tables, not formulas.
 *
 * Canonical accumulation order of one matrix entry ("merged deterministically"):
 * patches ascending; inside a patch the element rows ey that touch the entry, those in even
 * blocks of `strip` rows first, then those in odd blocks, ascending inside each; inside an element
 * row the elements ex ascending.  Each element contributes its dense element-matrix entry.
 */
#ifndef PMG_ASM_H
#define PMG_ASM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* one univariate basis evaluated at `npts` abscissae: the (p+1) functions active at each,
 * their first derivatives and the index of the first active function */
typedef struct pmg_asm_table1d {
    int32_t p, npts;
    const double* B;      /* npts * (p+1) */
    const double* dB;     /* npts * (p+1) */
    const int32_t* first; /* npts */
} pmg_asm_table1d;

/* edge ids of a patch: 0 eta=0, 1 xi=1, 2 eta=1, 3 xi=0 */
typedef struct pmg_asm_patch {
    pmg_asm_table1d gx, gy;     /* geometry bases (rational tensor patch) at the abscissae */
    int32_t gnx;                /* control points per net row (index = a + b*gnx) */
    const double *cx, *cy, *w;  /* control net and weights */
    const int32_t* l2g_row;     /* (nel+p_row)^2 local (x fastest) -> global row */
    const int32_t* l2g_col;     /* (nel+p_col)^2 local -> global column */
    int32_t dirichlet_edges;    /* bit e: edge e carries the Nitsche terms (not an interface) */
} pmg_asm_patch;

enum { PMG_ASM_OPERATOR = 0, PMG_ASM_MASS = 1 };

/* abscissae: point e*nq + a is Gauss point a of element e (ascending); points nel*nq and
 * nel*nq + 1 are x = 0 and x = 1 (boundary traces).  wq holds the nel*nq weights (element
 * length included). */
typedef struct pmg_asm_request {
    int32_t kind;            /* PMG_ASM_OPERATOR (row space == column space) or PMG_ASM_MASS (mixed) */
    int32_t nel, nq, npts;   /* elements per direction per patch, Gauss points per direction, nel*nq + 2 */
    int32_t strip;           /* element rows per block of the canonical accumulation order */
    const double* wq;
    pmg_asm_table1d row, col; /* solution bases of the row / column space */
    int32_t n_patches;
    const pmg_asm_patch* patches;
    double D[4], v[2], R;    /* CDR coefficients (operator only) */
    double penalty;          /* Nitsche eta / h (operator only) */
    int32_t nrows, ncols;
    const int64_t* rowptr;   /* sparsity pattern (sorted unique columns) */
    const int32_t* col_idx;
    double* val;             /* out: rowptr[nrows] values (host memory); NULL = not wanted */
    double* lumped;          /* out: nrows row sums, entries added in ascending column order
                                (lump_mass); NULL = not wanted */
} pmg_asm_request;

/* returns 0, or nonzero: 1 = nonpositive Jacobian determinant (geometry error), 2 = entry
 * outside the pattern / bad request, 3 = device failure (message: pmg_last_error()) */
typedef int (*pmg_asm_values_fn)(const pmg_asm_request* req);

#ifdef __cplusplus
}
#endif
#endif
