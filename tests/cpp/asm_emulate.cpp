// CPU emulation of the GPU assembler's kernels (TEST INFRASTRUCTURE ONLY -- never linked into the
// product): runs the __host__ __device__ phases of csrc/cuda/asm_core.cuh serially, element by
// element and CSR entry by CSR entry, exactly as assemble.cu's k_asm_elements / k_asm_gather
// schedule them.  tests/test_assembly_hook.py passes asm_emulate_values to
// iga_problem_build_with and compares with the host element loop: this checks the request
// plumbing, the index logic and the canonical accumulation order where no GPU is present.
#include <cstring>
#include <vector>

#include "../../include/pmg_asm.h"
#include "../../paper_1901_01685_b200/csrc/cuda/asm_core.cuh"

using namespace pmgasm;

static Tab tab(const pmg_asm_table1d& t) { return {t.p, t.B, t.dB, t.first}; }

extern "C" int asm_emulate_values(const pmg_asm_request* rq) {
    const int nel = rq->nel, n1 = rq->row.p + 1, n2 = rq->col.p + 1, nq = rq->nq;
    const int nr = nel + rq->row.p, nc = nel + rq->col.p;
    const int64_t esz = int64_t(n1) * n1 * n2 * n2, nnz = rq->rowptr[rq->nrows];
    Params P{};
    P.kind = rq->kind; P.nel = nel; P.nq = nq; P.strip = rq->strip; P.n1 = n1; P.n2 = n2;
    P.wq = rq->wq; P.row = tab(rq->row); P.col = tab(rq->col);
    std::memcpy(P.D, rq->D, sizeof(P.D));
    P.v[0] = rq->v[0]; P.v[1] = rq->v[1]; P.R = rq->R; P.pen = rq->penalty;
    std::vector<double> own;
    double* val = rq->val;
    if (!val) {
        own.resize(size_t(nnz));
        val = own.data();
    }
    std::memset(val, 0, size_t(nnz) * sizeof(double));
    std::vector<double> E(size_t(nel) * nel * esz);
    std::vector<int32_t> g2l(rq->ncols);
    for (int p = 0; p < rq->n_patches; ++p) {
        const pmg_asm_patch& g = rq->patches[p];
        P.geo = {tab(g.gx), tab(g.gy), g.gnx, g.cx, g.cy, g.w};
        P.dirichlet = g.dirichlet_edges;
        std::fill(g2l.begin(), g2l.end(), -1);
        for (int i = 0; i < nc * nc; ++i) g2l[g.l2g_col[i]] = i;
        for (int ey = 0; ey < nel; ++ey)
            for (int ex = 0; ex < nel; ++ex) {
                Scratch s;
                s.bad = 0;
                double* Ee = E.data() + (int64_t(ey) * nel + ex) * esz;
                if (P.kind == PMG_ASM_OPERATOR) {
                    for (int q = 0; q < nq * nq; ++q) op_point(P, ex, ey, q, s);
                    for (int slot = 0; slot < 4 * nq; ++slot)
                        if (edge_on(P, slot / nq, ex, ey)) op_trace(P, ex, ey, slot, s);
                    for (int it = 0; it < nq * n1 * n1; ++it) op_stage1(P, ex, it, s);
                    const int nn = n1 * n1;
                    for (int k = 0; k < nn * nn; ++k) Ee[k] = op_entry(P, ex, ey, k / nn, k % nn, s);
                } else {
                    for (int q = 0; q < nq * nq; ++q) mass_point(P, ex, ey, q, s);
                    for (int it = 0; it < nq * n1 * n2; ++it) mass_stage1(P, ex, it, s);
                    const int ncl = n2 * n2;
                    for (int k = 0; k < n1 * n1 * ncl; ++k) Ee[k] = mass_entry(P, ey, k / ncl, k % ncl, s);
                }
                if (s.bad) return 1;
            }
        for (int iy = 0; iy < nr; ++iy)
            for (int ix = 0; ix < nr; ++ix) {
                const int32_t row = g.l2g_row[ix + iy * nr];
                for (int64_t k = rq->rowptr[row]; k < rq->rowptr[row + 1]; ++k) {
                    const int32_t lc = g2l[rq->col_idx[k]];
                    if (lc < 0) continue;
                    double acc = val[k];
                    if (gather_entry(P, E.data(), 0, ix, iy, lc % nc, lc / nc, acc)) val[k] = acc;
                }
            }
    }
    if (rq->lumped)
        for (int32_t i = 0; i < rq->nrows; ++i) rq->lumped[i] = row_sum(val, rq->rowptr[i], rq->rowptr[i + 1]);
    return 0;
}
