// assemble.cu -- GPU assembly of the matrix values of A_k, M_k and P^k_j (F2; SPEC.md:132-167,
// PAPER.md:355-357), behind pmg_asm_values (include/pmg_cuda.h, request in include/pmg_asm.h).
//
// Two kernels per chunk of DOF rows of a patch:
//   k_asm_elements : one CTA per element; Gauss-point factors -> stage-1 sums over the xi points ->
//                    element-matrix entries (sum factorisation, plus the Nitsche traces on
//                    Dirichlet edges) written to a chunk buffer in HBM.  FP64, no tensor cores:
//                    (p+1)^4 entries of ~8 (p+1) flops each per element.
//   k_asm_gather   : one warp per matrix row; every CSR entry adds its <= (p+1)^2 element
//                    contributions in the canonical order of include/pmg_asm.h -- the order of the
//                    host loop's coloured strips -- so the merge is deterministic
//                    and the values equal the host assembler's bit for bit.  HBM-bound: each
//                    element-matrix entry is written once and read once.
// The arithmetic lives in asm_core.cuh.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../../include/pmg_cuda.h"
#include "asm_core.cuh"
#include "common.cuh"

namespace pmg {
void set_last_error(const std::string& m);  // capi.cu
}

using namespace pmg;
using namespace pmgasm;

namespace {

constexpr int kElemThreads = 128;

__global__ void __launch_bounds__(kElemThreads) k_asm_elements(Params P, int e0, int nrows_e, double* __restrict__ E,
                                                                int* __restrict__ bad) {
    __shared__ Scratch s;
    const int ex = blockIdx.x % P.nel, eyl = blockIdx.x / P.nel, ey = e0 + eyl;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nq = P.nq, nqq = nq * nq, n1 = P.n1, n2 = P.n2;
    if (tid == 0) s.bad = 0;
    __syncthreads();
    if (P.kind == PMG_ASM_OPERATOR) {
        for (int q = tid; q < nqq; q += nt) op_point(P, ex, ey, q, s);
        bool any_edge = false;
        for (int e = 0; e < 4; ++e) any_edge |= edge_on(P, e, ex, ey);
        if (any_edge)
            for (int slot = tid; slot < 4 * nq; slot += nt)
                if (edge_on(P, slot / nq, ex, ey)) op_trace(P, ex, ey, slot, s);
        __syncthreads();
        for (int it = tid; it < nq * n1 * n1; it += nt) op_stage1(P, ex, it, s);
        __syncthreads();
        const int nn = n1 * n1, ne = nn * nn;
        double* Ee = E + (int64_t(eyl) * P.nel + ex) * ne;
        for (int k = tid; k < ne; k += nt) Ee[k] = op_entry(P, ex, ey, k / nn, k % nn, s);
    } else {
        for (int q = tid; q < nqq; q += nt) mass_point(P, ex, ey, q, s);
        __syncthreads();
        for (int it = tid; it < nq * n1 * n2; it += nt) mass_stage1(P, ex, it, s);
        __syncthreads();
        const int ncl = n2 * n2, ne = n1 * n1 * ncl;
        double* Ee = E + (int64_t(eyl) * P.nel + ex) * ne;
        for (int k = tid; k < ne; k += nt) Ee[k] = mass_entry(P, ey, k / ncl, k % ncl, s);
    }
    if (tid == 0 && s.bad) *bad = 1;
}

// one warp per local row lr = ix + iy*nr, iy in [r0, r1)
__global__ void __launch_bounds__(256) k_asm_gather(Params P, int e0, int r0, int r1, const double* __restrict__ E,
                                                     const int32_t* __restrict__ l2g_row, const int32_t* __restrict__ g2l_col,
                                                     const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                     double* __restrict__ val) {
    const int nr = P.nel + P.n1 - 1, nc = P.nel + P.n2 - 1;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= int64_t(r1 - r0) * nr) return;
    const int iy = r0 + int(w / nr), ix = int(w % nr);
    const int32_t g = l2g_row[ix + iy * nr];
    const int64_t kb = rowptr[g], ke = rowptr[g + 1];
    for (int64_t k = kb + lane; k < ke; k += 32) {
        const int32_t lc = g2l_col[col[k]];
        if (lc < 0) continue;
        double acc = val[k];
        if (gather_entry(P, E, e0, ix, iy, lc % nc, lc / nc, acc)) val[k] = acc;
    }
}

__global__ void k_asm_rowsum(int32_t n, const int64_t* __restrict__ rowptr, const double* __restrict__ val,
                             double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = row_sum(val, rowptr[i], rowptr[i + 1]);
}

__global__ void k_asm_fill(int32_t* a, int64_t n, int32_t v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}
__global__ void k_asm_invert(const int32_t* __restrict__ l2g, int32_t n, int32_t* __restrict__ g2l) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) g2l[l2g[i]] = i;
}

struct DevBuf {  // owning device allocation
    void* p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    void alloc(size_t bytes) { PMG_CUDA(cudaMalloc(&p, bytes ? bytes : 1)); }
    template <class T>
    T* upload(const T* h, size_t n) {
        alloc(n * sizeof(T));
        PMG_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
        return static_cast<T*>(p);
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct DevTab {
    DevBuf B, dB, first;
    Tab view{};
    void upload(const pmg_asm_table1d& t) {
        const size_t n = size_t(t.npts) * (t.p + 1);
        view = {t.p, B.upload(t.B, n), dB.upload(t.dB, n), first.upload(t.first, size_t(t.npts))};
    }
};

void check_request(const pmg_asm_request* rq) {
    auto bad = [](const char* m) { throw std::invalid_argument(std::string("pmg_asm_values: ") + m); };
    if (!rq || !rq->patches || !rq->rowptr || !rq->col_idx || (!rq->val && !rq->lumped) || !rq->wq) bad("null pointer");
    if (rq->kind != PMG_ASM_OPERATOR && rq->kind != PMG_ASM_MASS) bad("unknown kind");
    if (rq->row.p < 1 || rq->row.p > kMaxP || rq->col.p < 1 || rq->col.p > kMaxP) bad("degree outside 1..5");
    if (rq->kind == PMG_ASM_OPERATOR && rq->row.p != rq->col.p) bad("operator needs equal row and column spaces");
    if (rq->nel < 1 || rq->nq < 1 || rq->nq > kMaxN1 || rq->npts != rq->nel * rq->nq + 2) bad("bad quadrature sizes");
    if (rq->strip < std::max(rq->row.p, rq->col.p) + 1) bad("strip shorter than the support of a basis function");
    if (rq->row.npts != rq->npts || rq->col.npts != rq->npts) bad("table size");
    for (int P = 0; P < rq->n_patches; ++P) {
        const pmg_asm_patch& g = rq->patches[P];
        if (g.gx.npts != rq->npts || g.gy.npts != rq->npts || g.gx.p > kMaxP || g.gy.p > kMaxP) bad("geometry table");
        if (!g.cx || !g.cy || !g.w || !g.l2g_row || !g.l2g_col) bad("null patch pointer");
    }
}

int asm_values(const pmg_asm_request* rq) {
    check_request(rq);
    const bool verbose = std::getenv("PMG_VERBOSE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    double t_up = 0, t_kern = 0, t_down = 0;
    auto lap = [&](double& acc) {
        if (!verbose) return;
        cudaDeviceSynchronize();
        auto t = std::chrono::steady_clock::now();
        acc += std::chrono::duration<double>(t - t_last).count();
        t_last = t;
    };
    const int nel = rq->nel, n1 = rq->row.p + 1, n2 = rq->col.p + 1;
    const int nr = nel + rq->row.p, nc = nel + rq->col.p;
    const int64_t nnz = rq->rowptr[rq->nrows];
    const int64_t esz = int64_t(n1) * n1 * n2 * n2;

    DevBuf d_wq, d_rowptr, d_col, d_val, d_bad, d_E, d_g2l;
    DevTab trow, tcol;
    Params P{};
    P.kind = rq->kind; P.nel = nel; P.nq = rq->nq; P.strip = rq->strip; P.n1 = n1; P.n2 = n2;
    P.wq = d_wq.upload(rq->wq, size_t(nel) * rq->nq);
    trow.upload(rq->row);
    tcol.upload(rq->col);
    P.row = trow.view; P.col = tcol.view;
    for (int i = 0; i < 4; ++i) P.D[i] = rq->D[i];
    P.v[0] = rq->v[0]; P.v[1] = rq->v[1]; P.R = rq->R; P.pen = rq->penalty;
    const int64_t* rowptr = d_rowptr.upload(rq->rowptr, size_t(rq->nrows) + 1);
    const int32_t* col = d_col.upload(rq->col_idx, size_t(nnz));
    d_val.alloc(size_t(nnz) * sizeof(double));
    PMG_CUDA(cudaMemset(d_val.p, 0, size_t(nnz) * sizeof(double)));
    d_bad.alloc(sizeof(int));
    PMG_CUDA(cudaMemset(d_bad.p, 0, sizeof(int)));
    d_g2l.alloc(size_t(rq->ncols) * sizeof(int32_t));
    lap(t_up);

    // chunk of DOF rows whose element matrices fit the buffer (default 2 GiB; PMG_ASM_CHUNK_MB)
    static const int chunk_mb = env_int("PMG_ASM_CHUNK_MB", 2048);
    const int64_t row_bytes = int64_t(nel) * esz * 8;
    int rows_e = int(std::max<int64_t>(1, std::min<int64_t>(nel, (int64_t(chunk_mb) << 20) / row_bytes)));
    const int pr = rq->row.p;
    if (rows_e <= pr && nel > rows_e) rows_e = std::min(nel, pr + 1);
    d_E.alloc(size_t(rows_e) * row_bytes);
    const int threads = int(std::min<int64_t>(kElemThreads, ((esz + 31) / 32) * 32));

    for (int p = 0; p < rq->n_patches; ++p) {
        const pmg_asm_patch& g = rq->patches[p];
        DevTab gx, gy;
        DevBuf d_cx, d_cy, d_w, d_l2gr, d_l2gc;
        gx.upload(g.gx);
        gy.upload(g.gy);
        const size_t ncp = size_t(g.gnx) * (size_t(g.gy.first[rq->npts - 1]) + g.gy.p + 1);  // net size: rows reach first(x=1)+p
        P.geo = {gx.view, gy.view, g.gnx, d_cx.upload(g.cx, ncp), d_cy.upload(g.cy, ncp), d_w.upload(g.w, ncp)};
        P.dirichlet = g.dirichlet_edges;
        const int32_t* l2gr = d_l2gr.upload(g.l2g_row, size_t(nr) * nr);
        const int32_t* l2gc = d_l2gc.upload(g.l2g_col, size_t(nc) * nc);
        lap(t_up);
        k_asm_fill<<<ceil_div(rq->ncols, 256), 256>>>(d_g2l.as<int32_t>(), rq->ncols, -1);
        k_asm_invert<<<ceil_div(int64_t(nc) * nc, 256), 256>>>(l2gc, nc * nc, d_g2l.as<int32_t>());
        PMG_LAUNCH_CHECK();
        // DOF rows [r0, r1) need element rows [max(0, r0 - pr), min(nel - 1, r1 - 1)]
        for (int r0 = 0; r0 < nr;) {
            const int e0 = std::max(0, r0 - pr);
            const int e1 = std::min(nel, e0 + rows_e);          // element rows [e0, e1)
            const int r1 = e1 == nel ? nr : e1;                 // rows < e1 are complete (row r needs ey <= r)
            k_asm_elements<<<unsigned(int64_t(e1 - e0) * nel), threads>>>(P, e0, e1 - e0, d_E.as<double>(), d_bad.as<int>());
            PMG_LAUNCH_CHECK();
            const int64_t warps = int64_t(r1 - r0) * nr;
            k_asm_gather<<<unsigned((warps * 32 + 255) / 256), 256>>>(P, e0, r0, r1, d_E.as<double>(), l2gr, d_g2l.as<int32_t>(),
                                                                      rowptr, col, d_val.as<double>());
            PMG_LAUNCH_CHECK();
            r0 = r1;
        }
        PMG_CUDA(cudaDeviceSynchronize());  // patch buffers are freed at the end of the iteration
        lap(t_kern);
    }
    int bad = 0;
    PMG_CUDA(cudaMemcpy(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad) {
        set_last_error("nonpositive Jacobian determinant");
        return 1;
    }
    if (rq->val) PMG_CUDA(cudaMemcpy(rq->val, d_val.p, size_t(nnz) * sizeof(double), cudaMemcpyDeviceToHost));
    if (rq->lumped) {
        DevBuf d_sum;
        d_sum.alloc(size_t(rq->nrows) * sizeof(double));
        k_asm_rowsum<<<ceil_div(rq->nrows, 256), 256>>>(rq->nrows, rowptr, d_val.as<double>(), d_sum.as<double>());
        PMG_LAUNCH_CHECK();
        PMG_CUDA(cudaMemcpy(rq->lumped, d_sum.p, size_t(rq->nrows) * sizeof(double), cudaMemcpyDeviceToHost));
    }
    lap(t_down);
    if (verbose)
        fprintf(stderr, "[pmg] asm kind %d p %d/%d nel %d nnz %lld: upload %.3f s, kernels %.3f s, download %.3f s\n", rq->kind,
                rq->row.p, rq->col.p, nel, (long long)nnz, t_up, t_kern, t_down);
    return 0;
}

}  // namespace

extern "C" int pmg_asm_values(const pmg_asm_request* rq) {
    try {
        return asm_values(rq);
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return 2;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 3;
    }
}
