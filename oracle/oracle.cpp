// CPU ORACLE (test infrastructure only) -- see oracle.h for scope and citations.
//
// Every floating-point expression below fixes the per-row operation order that the CUDA
// kernels reproduce bit-for-bit.  Build with -ffp-contract=off
// so that no multiply-add is contracted.
#include "oracle.h"

#include <algorithm>
#include <functional>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <atomic>
#include <thread>

namespace orc {

// ---- host threads (test infrastructure speed only; every row's arithmetic is unchanged) ----
static int g_threads = 1;
template <class F>
static void par_rows(int32_t n, F&& body) {  // body(i0, i1) over disjoint row blocks
    const int nt = std::max(1, std::min(g_threads, int((n + 4095) / 4096)));
    if (nt == 1) {
        body(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int32_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] { body(std::min(n, t * chunk), std::min(n, (t + 1) * chunk)); });
    for (auto& x : th) x.join();
}

struct Csr {
    int32_t n = 0, m = 0;
    std::vector<int32_t> rp, ci;
    std::vector<double> v;
    static Csr from(const pmg_csr_view& a) {
        Csr c;
        c.n = a.nrows;
        c.m = a.ncols;
        c.rp.assign(a.rowptr, a.rowptr + a.nrows + 1);
        c.ci.assign(a.col, a.col + c.rp.back());
        c.v.assign(a.val, a.val + c.rp.back());
        return c;
    }
};

// ---------------------------------------------------------------- kernels
// y_i = sum_j a_ij x_j, sequential ascending column, s starts at +0 ("ordered summation")
static inline double row_dot(const int32_t* rp, const int32_t* ci, const double* v, int32_t i, const double* x) {
    double s = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) s = s + v[k] * x[ci[k]];
    return s;
}

// y = A x
static void spmv_into(const Csr& A, const double* x, double* y) {
    par_rows(A.n, [&](int32_t i0, int32_t i1) {
        for (int32_t i = i0; i < i1; ++i) y[i] = row_dot(A.rp.data(), A.ci.data(), A.v.data(), i, x);
    });
}

// r_i = f_i - (A x)_i
static void residual(const Csr& A, const double* x, const double* f, double* r) {
    par_rows(A.n, [&](int32_t i0, int32_t i1) {
        for (int32_t i = i0; i < i1; ++i) r[i] = f[i] - row_dot(A.rp.data(), A.ci.data(), A.v.data(), i, x);
    });
}

// ||r||_2 in the canonical blocked order: chunks of 256 entries; inside a chunk eight
// groups of 32 squares are reduced by the xor-butterfly (offsets 16,8,4,2,1), the eight
// group sums are added in order; chunk sums are strided over 256 accumulators
// (acc_t = sum_{k = t mod 256} chunk_k, ascending k, from +0), which are reduced like a chunk.
static double chunk_reduce(const double* v256) {
    double c = 0.0;
    for (int w = 0; w < 8; ++w) {
        double lane[32];
        for (int l = 0; l < 32; ++l) lane[l] = v256[w * 32 + l];
        for (int off = 16; off >= 1; off >>= 1) {
            double nl[32];
            for (int l = 0; l < 32; ++l) nl[l] = lane[l] + lane[l ^ off];
            std::memcpy(lane, nl, sizeof(lane));
        }
        c = (w == 0) ? lane[0] : c + lane[0];
    }
    return c;
}
// (x, y) in the same canonical order, with products x_i * y_i in place of squares
static double dot2(const double* x, const double* y, int64_t n) {
    int64_t nch = (n + 255) / 256;
    std::vector<double> part(nch);
    double buf[256];
    for (int64_t c = 0; c < nch; ++c) {
        for (int t = 0; t < 256; ++t) {
            int64_t i = c * 256 + t;
            buf[t] = i < n ? x[i] * y[i] : 0.0;
        }
        part[c] = chunk_reduce(buf);
    }
    for (int t = 0; t < 256; ++t) {
        double a = 0.0;
        for (int64_t k = t; k < nch; k += 256) a = a + part[k];
        buf[t] = a;
    }
    return chunk_reduce(buf);
}
static double norm2(const double* r, int64_t n) { return std::sqrt(dot2(r, r, n)); }

// Forward lexicographic Gauss-Seidel, u_i <- ((f_i - S_L) - S_U) * (1/a_ii) with S_L over
// j < i (new values) and S_U over j > i (old values), each ascending from +0
// (SPEC.md:233-241).  The diagonal is applied as a multiplication by its IEEE reciprocal
// 1.0/a_ii (computed once per matrix).  Returns -1 or the row with a
// zero/missing diagonal.
static int64_t gs_sweep(const Csr& A, double* u, const double* f) {
    for (int32_t i = 0; i < A.n; ++i) {
        double sl = 0.0, su = 0.0, d = 0.0;
        bool has_d = false;
        for (int32_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            int32_t j = A.ci[k];
            if (j < i) sl = sl + A.v[k] * u[j];
            else if (j > i) su = su + A.v[k] * u[j];
            else { d = A.v[k]; has_d = true; }
        }
        if (!has_d || d == 0.0) return i;
        const double dinv = 1.0 / d;
        u[i] = ((f[i] - sl) - su) * dinv;
    }
    return -1;
}

// Reverse Cuthill-McKee on the symmetrised pattern: per component start at
// the unvisited node of minimum (degree, index); BFS visiting neighbours by ascending
// (degree, index); reverse the concatenated order.  perm[new] = old.
static std::vector<int32_t> rcm(const pmg_csr_view& A) {
    const int32_t n = A.nrows;
    std::vector<std::vector<int32_t>> adj(n);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
            int32_t j = A.col[k];
            if (j == i) continue;
            adj[i].push_back(j);
            adj[j].push_back(i);
        }
    std::vector<int32_t> deg(n);
    for (int32_t i = 0; i < n; ++i) {
        auto& a = adj[i];
        std::sort(a.begin(), a.end());
        a.erase(std::unique(a.begin(), a.end()), a.end());
        deg[i] = int32_t(a.size());
    }
    auto less = [&](int32_t a, int32_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
    std::vector<int32_t> byd(n);
    for (int32_t i = 0; i < n; ++i) byd[i] = i;
    std::sort(byd.begin(), byd.end(), less);
    std::vector<char> seen(n, 0);
    std::vector<int32_t> order;
    order.reserve(n);
    size_t cursor = 0;
    while (int32_t(order.size()) < n) {
        while (seen[byd[cursor]]) ++cursor;
        int32_t s = byd[cursor];
        size_t head = order.size();
        order.push_back(s);
        seen[s] = 1;
        while (head < order.size()) {
            int32_t x = order[head++];
            std::vector<int32_t> nb;
            for (int32_t y : adj[x])
                if (!seen[y]) nb.push_back(y);
            std::sort(nb.begin(), nb.end(), less);
            for (int32_t y : nb) {
                seen[y] = 1;
                order.push_back(y);
            }
        }
    }
    std::reverse(order.begin(), order.end());
    return order;
}

// ---------------------------------------------------------------- ILUT
struct Factor {
    int32_t n = 0;
    Csr L, U;  // L strictly lower (unit diagonal implicit); U row = [diag, off-diagonals ascending]
    std::vector<int32_t> perm, pinv;
    int32_t levL = 0, levU = 0;
    void levels() {
        std::vector<int32_t> lv(n, 0);
        levL = n ? 1 : 0;
        for (int32_t i = 0; i < n; ++i) {
            int32_t m = -1;
            for (int32_t k = L.rp[i]; k < L.rp[i + 1]; ++k) m = std::max(m, lv[L.ci[k]]);
            lv[i] = m + 1;
            levL = std::max(levL, lv[i] + 1);
        }
        levU = n ? 1 : 0;
        for (int32_t i = n - 1; i >= 0; --i) {
            int32_t m = -1;
            for (int32_t k = U.rp[i] + 1; k < U.rp[i + 1]; ++k) m = std::max(m, lv[U.ci[k]]);
            lv[i] = m + 1;
            levU = std::max(levU, lv[i] + 1);
        }
    }
};

struct Cand {
    int32_t c;
    double v;
};
// rule 2: keep the M entries of largest |v|, ties by ascending column; result column-sorted
static void keep_largest(std::vector<Cand>& c, int32_t M) {
    if (int32_t(c.size()) > M) {
        std::sort(c.begin(), c.end(), [](const Cand& a, const Cand& b) {
            double x = std::fabs(a.v), y = std::fabs(b.v);
            return x != y ? x > y : a.c < b.c;
        });
        c.resize(M);
    }
    std::sort(c.begin(), c.end(), [](const Cand& a, const Cand& b) { return a.c < b.c; });
}

// Dual-threshold ILUT(tau, m), IKJ on the symmetrically permuted matrix (SPEC.md:251-259,
// PAPER.md:298-311):
//   tau_i = tau * (sum_j |a_ij| / nnz_i) over the permuted row's stored entries (ascending column);
//   pivots k ascending (including fill): w_k = w_k / u_kk; drop if |w_k| < tau_i (rule 1), else
//     w_j = w_j - w_k * u_kj for the off-diagonal entries of U row k;
//   U entries with |w_j| < tau_i dropped; rule 2 keeps the M = ceil(m nnz/n) largest in L and in U
//   (diagonal always kept); zero diagonal -> error(row).
namespace {
struct RowOut {  // one factor row: L part (ascending) or U part (diagonal first, then ascending)
    std::vector<int32_t> c;
    std::vector<double> v;
};
struct IlutScratch {
    std::vector<double> w;
    std::vector<char> present;
    std::vector<uint64_t> bits;
    std::vector<std::pair<int32_t, double>> row;
    std::vector<int32_t> upos, touched;
    std::vector<Cand> lc, uc;
    explicit IlutScratch(int32_t n) : w(n, 0.0), present(n, 0), bits(size_t(n) / 64 + 2, 0) {}
};
}  // namespace

// one row of the IKJ elimination; U rows of earlier rows are read once their `done` flag is set
static bool ilut_row(int32_t i, const pmg_csr_view& A, const std::vector<int32_t>& perm,
                     const std::vector<int32_t>& pinv, double tau, int32_t M, std::vector<RowOut>& Lr,
                     std::vector<RowOut>& Ur, std::atomic<int>* done, IlutScratch& S) {
    std::vector<double>& w = S.w;
    std::vector<char>& present = S.present;
    std::vector<uint64_t>& bits = S.bits;
    const int32_t old = perm[i];
    S.row.clear();
    for (int32_t k = A.rowptr[old]; k < A.rowptr[old + 1]; ++k) S.row.push_back({pinv[A.col[k]], A.val[k]});
    std::sort(S.row.begin(), S.row.end());
    double asum = 0.0;
    for (auto& e : S.row) asum = asum + std::fabs(e.second);
    const double tau_i = tau * (asum / double(S.row.size()));
    S.upos.clear();
    S.touched.clear();
    int32_t kmin = i;
    for (auto& e : S.row) {
        int32_t c = e.first;
        w[c] = e.second;
        present[c] = 1;
        S.touched.push_back(c);
        if (c < i) { bits[c >> 6] |= 1ull << (c & 63); kmin = std::min(kmin, c); }
        else if (c > i) S.upos.push_back(c);
    }
    S.lc.clear();
    // ascending pivot scan over the L-part bitmap
    int32_t k = kmin;
    while (k < i) {
        int64_t wi = k >> 6;
        uint64_t word = bits[wi] & (~0ull << (k & 63));
        while (word == 0 && (wi + 1) * 64 < int64_t(i)) word = bits[++wi];
        if (word == 0) break;
        k = int32_t(wi * 64 + __builtin_ctzll(word));
        if (k >= i) break;
        bits[k >> 6] &= ~(1ull << (k & 63));
        while (done[k].load(std::memory_order_acquire) == 0) std::this_thread::yield();
        const RowOut& Uk = Ur[k];
        const double wk = w[k] / Uk.v[0];
        if (std::fabs(wk) < tau_i) {
            w[k] = 0.0;
            present[k] = 0;
        } else {
            w[k] = wk;
            S.lc.push_back({k, wk});
            for (size_t q = 1; q < Uk.c.size(); ++q) {
                int32_t j = Uk.c[q];
                if (!present[j]) {
                    present[j] = 1;
                    S.touched.push_back(j);
                    if (j < i) bits[j >> 6] |= 1ull << (j & 63);
                    else if (j > i) S.upos.push_back(j);
                }
                w[j] = w[j] - wk * Uk.v[q];
            }
        }
        ++k;
    }
    const double diag = present[i] ? w[i] : 0.0;
    bool ok = diag != 0.0;
    S.uc.clear();
    for (int32_t j : S.upos)
        if (!(std::fabs(w[j]) < tau_i)) S.uc.push_back({j, w[j]});
    keep_largest(S.lc, M);
    keep_largest(S.uc, M);
    RowOut& L = Lr[i];
    RowOut& U = Ur[i];
    for (auto& e : S.lc) { L.c.push_back(e.c); L.v.push_back(e.v); }
    U.c.push_back(i);
    U.v.push_back(ok ? diag : 1.0);  // 1.0 only keeps later rows running; the error is reported
    for (auto& e : S.uc) { U.c.push_back(e.c); U.v.push_back(e.v); }
    for (int32_t c : S.touched) { w[c] = 0.0; present[c] = 0; }
    done[i].store(1, std::memory_order_release);
    return ok;
}

// Dual-threshold ILUT(tau, m), IKJ on the symmetrically permuted matrix (SPEC.md:251-259,
// PAPER.md:298-311):
//   tau_i = tau * (sum_j |a_ij| / nnz_i) over the permuted row's stored entries (ascending column);
//   pivots k ascending (including fill): w_k = w_k / u_kk; drop if |w_k| < tau_i (rule 1), else
//     w_j = w_j - w_k * u_kj for the off-diagonal entries of U row k;
//   U entries with |w_j| < tau_i dropped; rule 2 keeps the M = ceil(m nnz/n) largest in L and in U
//   (diagonal always kept); zero diagonal -> error(row).
// Rows may be processed by several host threads (rows claimed in ascending order, each waits for
// the U rows it pivots on); every row's arithmetic is the sequential algorithm's.
static std::unique_ptr<Factor> ilut(const pmg_csr_view& A, double tau, double m, int ordering, int64_t* err_row) {
    const int32_t n = A.nrows;
    auto F = std::make_unique<Factor>();
    F->n = n;
    F->perm = ordering == PMG_ORDER_RCM ? rcm(A) : std::vector<int32_t>(n);
    if (ordering != PMG_ORDER_RCM)
        for (int32_t i = 0; i < n; ++i) F->perm[i] = i;
    F->pinv.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) F->pinv[F->perm[i]] = i;
    const int64_t nnz = A.rowptr[n];
    const int32_t M = int32_t(std::ceil(m * double(nnz) / double(n)));
    std::vector<RowOut> Lr(n), Ur(n);
    std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[n]);
    for (int32_t i = 0; i < n; ++i) done[i].store(0, std::memory_order_relaxed);
    std::atomic<int32_t> next{0}, first_bad{INT32_MAX};
    auto worker = [&] {
        IlutScratch S(n);
        for (;;) {
            const int32_t i = next.fetch_add(1);
            if (i >= n) break;
            if (!ilut_row(i, A, F->perm, F->pinv, tau, M, Lr, Ur, done.get(), S)) {
                int32_t cur = first_bad.load();
                while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {
                }
            }
        }
    };
    const int nt = std::max(1, std::min(g_threads, int(n / 256) + 1));
    if (nt == 1) worker();
    else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t) th.emplace_back(worker);
        for (auto& x : th) x.join();
    }
    if (first_bad.load() != INT32_MAX) {
        if (err_row) *err_row = first_bad.load();
        return nullptr;
    }
    F->L.n = F->L.m = F->U.n = F->U.m = n;
    F->L.rp.assign(n + 1, 0);
    F->U.rp.assign(n + 1, 0);
    for (int32_t i = 0; i < n; ++i) {
        F->L.rp[i + 1] = F->L.rp[i] + int32_t(Lr[i].c.size());
        F->U.rp[i + 1] = F->U.rp[i] + int32_t(Ur[i].c.size());
    }
    F->L.ci.reserve(F->L.rp[n]);
    F->L.v.reserve(F->L.rp[n]);
    F->U.ci.reserve(F->U.rp[n]);
    F->U.v.reserve(F->U.rp[n]);
    for (int32_t i = 0; i < n; ++i) {
        F->L.ci.insert(F->L.ci.end(), Lr[i].c.begin(), Lr[i].c.end());
        F->L.v.insert(F->L.v.end(), Lr[i].v.begin(), Lr[i].v.end());
        std::vector<int32_t>().swap(Lr[i].c);
        std::vector<double>().swap(Lr[i].v);
        F->U.ci.insert(F->U.ci.end(), Ur[i].c.begin(), Ur[i].c.end());
        F->U.v.insert(F->U.v.end(), Ur[i].v.begin(), Ur[i].v.end());
        std::vector<int32_t>().swap(Ur[i].c);
        std::vector<double>().swap(Ur[i].v);
    }
    F->levels();
    return F;
}

// PROBE ONLY: the dual-threshold ILUT of the paper's library (PAPER.md:311,
// Eigen's IncompleteLUT), restated from its published algorithm to explain the gap
// between the SPEC's rule and the paper's tables.  Differences from ilut() above:
//   * fill_in = floor(m nnz / n) + 1, and only nnzL = fill_in / 2 entries are kept in L; U keeps
//     min(|U row incl. diagonal|, nnzL) - 1 off-diagonal entries;
//   * a multiplier is dropped when |w_k / u_kk| <= tau (absolute), U entries when
//     |w_j| <= tau * ||row||_2 (2-norm of the original row);
//   * a zero pivot is shifted to sqrt(tau) * ||row||_2 instead of being an error.
// The fill-reducing ordering (the library's AMD) is not restated; `perm` is natural or RCM.
static std::unique_ptr<Factor> ilut_eigen(const pmg_csr_view& A, double tau, double m, int ordering) {
    const int32_t n = A.nrows;
    auto F = std::make_unique<Factor>();
    F->n = n;
    F->perm = ordering == PMG_ORDER_RCM ? rcm(A) : std::vector<int32_t>(n);
    if (ordering != PMG_ORDER_RCM)
        for (int32_t i = 0; i < n; ++i) F->perm[i] = i;
    F->pinv.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) F->pinv[F->perm[i]] = i;
    const int64_t nnz = A.rowptr[n];
    int64_t fill_in = int64_t(double(nnz) * m) / n + 1;
    if (fill_in > n) fill_in = n;
    const int64_t nnzL = fill_in / 2, nnzU = nnzL;
    std::vector<RowOut> Lr(n), Ur(n);
    std::vector<double> w(n, 0.0);
    std::vector<char> present(n, 0);
    std::vector<int32_t> touched;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t old = F->perm[i];
        double rn = 0.0;
        touched.clear();
        std::vector<int32_t> lpos;
        for (int32_t k = A.rowptr[old]; k < A.rowptr[old + 1]; ++k) {
            int32_t c = F->pinv[A.col[k]];
            w[c] = A.val[k];
            present[c] = 1;
            touched.push_back(c);
            if (c < i) lpos.push_back(c);
            rn = rn + A.val[k] * A.val[k];
        }
        rn = std::sqrt(rn);
        std::vector<Cand> lc, uc;
        // pivots in ascending column order, including fill (a min-heap over the L part)
        std::vector<int32_t> heap(lpos.begin(), lpos.end());
        std::make_heap(heap.begin(), heap.end(), std::greater<int32_t>());
        while (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end(), std::greater<int32_t>());
            const int32_t k = heap.back();
            heap.pop_back();
            const RowOut& Uk = Ur[k];
            const double fact = w[k] / Uk.v[0];
            if (std::fabs(fact) <= tau) continue;
            for (size_t q = 1; q < Uk.c.size(); ++q) {
                const int32_t j = Uk.c[q];
                if (!present[j]) {
                    present[j] = 1;
                    w[j] = 0.0;
                    touched.push_back(j);
                    if (j < i) {
                        heap.push_back(j);
                        std::push_heap(heap.begin(), heap.end(), std::greater<int32_t>());
                    }
                }
                w[j] = w[j] - fact * Uk.v[q];
            }
            lc.push_back({k, fact});
        }
        double diag = present[i] ? w[i] : 0.0;
        if (diag == 0.0) diag = std::sqrt(tau) * rn;
        for (int32_t c : touched)
            if (c > i && std::fabs(w[c]) > tau * rn) uc.push_back({c, w[c]});
        keep_largest(lc, int32_t(std::min<int64_t>(int64_t(lc.size()), nnzL)));
        const int64_t keepU = std::min<int64_t>(int64_t(uc.size()) + 1, nnzU) - 1;
        keep_largest(uc, int32_t(std::max<int64_t>(keepU, 0)));
        for (auto& e : lc) { Lr[i].c.push_back(e.c); Lr[i].v.push_back(e.v); }
        Ur[i].c.push_back(i);
        Ur[i].v.push_back(diag);
        for (auto& e : uc) { Ur[i].c.push_back(e.c); Ur[i].v.push_back(e.v); }
        for (int32_t c : touched) { w[c] = 0.0; present[c] = 0; }
    }
    F->L.n = F->L.m = F->U.n = F->U.m = n;
    F->L.rp.assign(n + 1, 0);
    F->U.rp.assign(n + 1, 0);
    for (int32_t i = 0; i < n; ++i) {
        F->L.rp[i + 1] = F->L.rp[i] + int32_t(Lr[i].c.size());
        F->U.rp[i + 1] = F->U.rp[i] + int32_t(Ur[i].c.size());
        F->L.ci.insert(F->L.ci.end(), Lr[i].c.begin(), Lr[i].c.end());
        F->L.v.insert(F->L.v.end(), Lr[i].v.begin(), Lr[i].v.end());
        F->U.ci.insert(F->U.ci.end(), Ur[i].c.begin(), Ur[i].c.end());
        F->U.v.insert(F->U.v.end(), Ur[i].v.begin(), Ur[i].v.end());
    }
    F->levels();
    return F;
}

// e = P^T U^{-1} L^{-1} P r.  L rows ascending, U rows descending.
static void lsolve(const Factor& F, const double* r, double* y) {
    for (int32_t i = 0; i < F.n; ++i) {
        double s = 0.0;
        for (int32_t k = F.L.rp[i]; k < F.L.rp[i + 1]; ++k) s = s + F.L.v[k] * y[F.L.ci[k]];
        y[i] = r[F.perm[i]] - s;
    }
}
// x_i = (y_i - S) * (1/u_ii), S over the off-diagonal entries in DESCENDING column order;
// then u[perm[i]] = u[perm[i]] + x_i.  (1/u_ii: IEEE reciprocal, as in the GS sweep.)
static void usolve_add(const Factor& F, const double* y, double* x, double* u) {
    for (int32_t i = F.n - 1; i >= 0; --i) {
        const int32_t d0 = F.U.rp[i];
        double s = 0.0;
        for (int32_t k = F.U.rp[i + 1] - 1; k > d0; --k) s = s + F.U.v[k] * x[F.U.ci[k]];
        const double dinv = 1.0 / F.U.v[d0];
        x[i] = (y[i] - s) * dinv;
        u[F.perm[i]] = u[F.perm[i]] + x[i];
    }
}

// ---------------------------------------------------------------- dense coarse solve
struct DenseLU {
    int n = 0;
    std::vector<double> a;  // row-major LU
    std::vector<int> piv;
    // partial pivoting, first maximal |a_ik| on ties; l = a_ik / a_kk; a_ij = a_ij - l * a_kj
    bool factor(const Csr& A) {
        n = A.n;
        a.assign(size_t(n) * n, 0.0);
        for (int i = 0; i < n; ++i)
            for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) a[size_t(i) * n + A.ci[k]] = A.v[k];
        piv.resize(n);
        for (int k = 0; k < n; ++k) {
            int p = k;
            for (int i = k + 1; i < n; ++i)
                if (std::fabs(a[size_t(i) * n + k]) > std::fabs(a[size_t(p) * n + k])) p = i;
            piv[k] = p;
            if (p != k)
                for (int j = 0; j < n; ++j) std::swap(a[size_t(k) * n + j], a[size_t(p) * n + j]);
            if (a[size_t(k) * n + k] == 0.0) return false;
            for (int i = k + 1; i < n; ++i) {
                double l = a[size_t(i) * n + k] / a[size_t(k) * n + k];
                a[size_t(i) * n + k] = l;
                for (int j = k + 1; j < n; ++j) a[size_t(i) * n + j] = a[size_t(i) * n + j] - l * a[size_t(k) * n + j];
            }
        }
        return true;
    }
    // b permuted by the pivot sequence; y_i = b_i - sum_{j<i} l_ij y_j; x_i = (y_i - sum_{j>i} u_ij x_j)/u_ii
    void solve(const double* b, double* x) const {
        std::vector<double> y(b, b + n);
        for (int k = 0; k < n; ++k) std::swap(y[k], y[piv[k]]);
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < i; ++j) s = s + a[size_t(i) * n + j] * y[j];
            y[i] = y[i] - s;
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = 0.0;
            for (int j = i + 1; j < n; ++j) s = s + a[size_t(i) * n + j] * x[j];
            x[i] = (y[i] - s) / a[size_t(i) * n + i];
        }
    }
};

// ---------------------------------------------------------------- hierarchy
struct PLev {
    Csr A, P, PT;
    std::vector<double> ML;
    Factor* F = nullptr;
    std::vector<double> u, f, r, y, x;  // work
};
struct HLev {
    const Csr* A = nullptr;
    Csr Aown, P, PT;
    Factor* F = nullptr;
    std::vector<double> e, r, res, y, x;
};
struct Hier {
    int np = 0, nh = 0, smoother = 0, nu1 = 1, nu2 = 1;
    std::vector<PLev> pl;
    std::vector<HLev> hl;
    std::vector<std::unique_ptr<Factor>> owned;
    std::vector<Factor*> factors;  // p-level ILUT factors then h-level factors
    DenseLU coarse;
    double setup_seconds = 0;
};

static void prolong_add(const Csr& P, const double* ML, const double* vc, double* u) {
    par_rows(P.n, [&](int32_t i0, int32_t i1) {
        for (int32_t i = i0; i < i1; ++i) u[i] = u[i] + row_dot(P.rp.data(), P.ci.data(), P.v.data(), i, vc) / ML[i];
    });
}
static void restrict_(const Csr& PT, const double* MLc, const double* rf, double* rc) {
    par_rows(PT.n, [&](int32_t j0, int32_t j1) {
        for (int32_t j = j0; j < j1; ++j) rc[j] = row_dot(PT.rp.data(), PT.ci.data(), PT.v.data(), j, rf) / MLc[j];
    });
}
static void hprolong_add(const Csr& P, const double* ec, double* e) {
    par_rows(P.n, [&](int32_t i0, int32_t i1) {
        for (int32_t i = i0; i < i1; ++i) e[i] = e[i] + row_dot(P.rp.data(), P.ci.data(), P.v.data(), i, ec);
    });
}

// ILUT smoothing step u <- u + U^{-1} L^{-1} (f - A u); `r` may be a
// residual of the current u (reused) or null.
static void ilut_smooth(const Csr& A, const Factor& F, double* u, const double* f, const double* r_known, double* r,
                        double* y, double* x) {
    const double* rr = r_known;
    if (!rr) {
        residual(A, u, f, r);
        rr = r;
    }
    lsolve(F, rr, y);
    usolve_add(F, y, x, u);
}

// one h-MG V(1,1) cycle on h-level j from e = 0
static void hmg(Hier& H, int j, double* e, const double* r) {
    HLev& L = H.hl[j];
    const int32_t n = L.A->n;
    if (j == H.nh - 1) {
        H.coarse.solve(r, e);
        return;
    }
    std::fill(e, e + n, 0.0);
    ilut_smooth(*L.A, *L.F, e, r, r, nullptr, L.y.data(), L.x.data());  // e = 0: residual is r
    residual(*L.A, e, r, L.res.data());
    HLev& C = H.hl[j + 1];
    double* rc = C.r.data();
    for (int32_t q = 0; q < L.PT.n; ++q) rc[q] = row_dot(L.PT.rp.data(), L.PT.ci.data(), L.PT.v.data(), q, L.res.data());
    hmg(H, j + 1, C.e.data(), rc);
    hprolong_add(L.P, C.e.data(), e);
    ilut_smooth(*L.A, *L.F, e, r, nullptr, L.res.data(), L.y.data(), L.x.data());
}

static int64_t smooth(Hier& H, int l, double* u, const double* f, const double* r_known) {
    PLev& L = H.pl[l];
    if (H.smoother == PMG_SMOOTHER_GS) return gs_sweep(L.A, u, f);
    ilut_smooth(L.A, *L.F, u, f, r_known, L.r.data(), L.y.data(), L.x.data());
    return -1;
}

// V-cycle at p-level l.  `zero`: u == 0 on entry (its residual is f).
static int64_t vcycle(Hier& H, int l, double* u, const double* f, const double* r_known, bool zero) {
    if (l == H.np - 1) {  // p = 1: one h-MG V-cycle on the residual equation
        if (zero) {  // u == 0: the correction is the cycle's result itself
            hmg(H, 0, u, f);
            return -1;
        }
        // a hierarchy of p = 1 alone: e = hmg(f - A u), u += e
        PLev& L = H.pl[l];
        const int32_t n = L.A.n;
        const double* r = r_known;
        if (!r) {
            residual(L.A, u, f, L.r.data());
            r = L.r.data();
        }
        hmg(H, 0, L.y.data(), r);
        for (int32_t i = 0; i < n; ++i) u[i] = u[i] + L.y[i];
        return -1;
    }
    PLev& L = H.pl[l];
    for (int s = 0; s < H.nu1; ++s) {
        const double* rk = s == 0 ? (zero ? f : r_known) : nullptr;
        int64_t e = smooth(H, l, u, f, rk);
        if (e >= 0) return e;
    }
    residual(L.A, u, f, L.r.data());
    PLev& C = H.pl[l + 1];
    restrict_(L.PT, C.ML.data(), L.r.data(), C.f.data());
    std::fill(C.u.begin(), C.u.end(), 0.0);
    int64_t e = vcycle(H, l + 1, C.u.data(), C.f.data(), nullptr, true);
    if (e >= 0) return e;
    prolong_add(L.P, L.ML.data(), C.u.data(), u);
    for (int s = 0; s < H.nu2; ++s) {
        e = smooth(H, l, u, f, nullptr);
        if (e >= 0) return e;
    }
    return -1;
}

// Right-preconditioned BiCGSTAB (one V-cycle per
// preconditioning phase).  One iteration = one full step with two preconditioner applications;
// the stop test uses the recursively updated residual, rho_i = ||r_i|| / ||f - A u0||.  Every
// dot product and norm is canonical (dot2 / norm2) and every vector update has the fixed
// operation order below, which the GPU path reproduces bit for bit:
//   p = r (i = 1),  p = r + beta * (p - omega * v)      beta = (rho / rho_prev) * (alpha / omega)
//   s = r - alpha * v;  u = (u + alpha * ph) + omega * sh;  r = s - omega * t
// Breakdown (flag, stop): (rh, r) = 0, (rh, v) = 0, or omega = 0 after the update.
template <class Prec>
static int bicgstab(const Csr& A, const double* f, double* u, double tol, int max_iter, Prec&& prec, double* hist,
                    int* iters, int* flags) {
    const int32_t n = A.n;
    std::vector<double> r(n), rh(n), p(n), v(n), s(n), t(n), ph(n), sh(n);
    residual(A, u, f, r.data());
    const double n0 = norm2(r.data(), n);
    hist[0] = 1.0;
    *iters = 0;
    *flags = 0;
    if (n0 == 0.0) {
        *flags = PMG_FLAG_CONVERGED;
        return PMG_OK;
    }
    rh = r;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (int it = 1; it <= max_iter; ++it) {
        const double rho = dot2(rh.data(), r.data(), n);
        if (rho == 0.0 || !std::isfinite(rho)) {
            *flags |= PMG_FLAG_BREAKDOWN;
            break;
        }
        if (it == 1) {
            p = r;
        } else {
            const double beta = (rho / rho_prev) * (alpha / omega);
            for (int32_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        }
        int rc = prec(p.data(), ph.data());
        if (rc) return rc;
        spmv_into(A, ph.data(), v.data());
        const double rv = dot2(rh.data(), v.data(), n);
        if (rv == 0.0 || !std::isfinite(rv)) {
            *flags |= PMG_FLAG_BREAKDOWN;
            break;
        }
        alpha = rho / rv;
        for (int32_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
        rc = prec(s.data(), sh.data());
        if (rc) return rc;
        spmv_into(A, sh.data(), t.data());
        const double tt = dot2(t.data(), t.data(), n);
        const double ts = dot2(t.data(), s.data(), n);
        omega = tt == 0.0 ? 0.0 : ts / tt;
        for (int32_t i = 0; i < n; ++i) {
            u[i] = (u[i] + alpha * ph[i]) + omega * sh[i];
            r[i] = s[i] - omega * t[i];
        }
        const double res = norm2(r.data(), n) / n0;
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
    return PMG_OK;
}

}  // namespace orc

// =================================================================== C ABI
using namespace orc;

struct orc_factor_s {
    Factor* F;
    bool own;
};
struct orc_hier_s {
    Hier H;
};

extern "C" {

void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

int orc_spmv(const pmg_csr_view* A, const double* x, double* y) {
    for (int32_t i = 0; i < A->nrows; ++i) y[i] = row_dot(A->rowptr, A->col, A->val, i, x);
    return PMG_OK;
}
int orc_residual(const pmg_csr_view* A, const double* x, const double* f, double* r) {
    for (int32_t i = 0; i < A->nrows; ++i) r[i] = f[i] - row_dot(A->rowptr, A->col, A->val, i, x);
    return PMG_OK;
}
double orc_norm2(const double* r, int64_t n) { return norm2(r, n); }
double orc_dot(const double* x, const double* y, int64_t n) { return dot2(x, y, n); }
int orc_gs_sweep(const pmg_csr_view* A, double* u, const double* f, int64_t* err_row) {
    if (A->nrows != A->ncols) return PMG_ERR_DIM;
    Csr c = Csr::from(*A);
    int64_t e = gs_sweep(c, u, f);
    if (e >= 0) {
        if (err_row) *err_row = e;
        return PMG_ZERO_DIAG;
    }
    return PMG_OK;
}
int orc_rcm(const pmg_csr_view* A, int32_t* perm) {
    auto p = rcm(*A);
    std::copy(p.begin(), p.end(), perm);
    return PMG_OK;
}
int orc_ilut(const pmg_csr_view* A, double tau, double fillfactor, int ordering, orc_factor* out, int64_t* err_row) {
    if (A->nrows != A->ncols) return PMG_ERR_DIM;
    if (tau < 0 || fillfactor < 1) return PMG_ERR_ARG;
    auto F = ilut(*A, tau, fillfactor, ordering, err_row);
    if (!F) return PMG_ZERO_PIVOT;
    *out = new orc_factor_s{F.release(), true};
    return PMG_OK;
}
int orc_ilut_eigen(const pmg_csr_view* A, double tau, double fillfactor, int ordering, orc_factor* out) {
    if (A->nrows != A->ncols) return PMG_ERR_DIM;
    *out = new orc_factor_s{ilut_eigen(*A, tau, fillfactor, ordering).release(), true};
    return PMG_OK;
}
int orc_factor_from_arrays(int32_t n, const int32_t* Lrp, const int32_t* Lc, const double* Lv, const int32_t* Urp,
                           const int32_t* Uc, const double* Uv, const int32_t* perm, orc_factor* out) {
    auto* F = new Factor;
    F->n = n;
    F->L.n = F->L.m = F->U.n = F->U.m = n;
    F->L.rp.assign(Lrp, Lrp + n + 1);
    F->L.ci.assign(Lc, Lc + Lrp[n]);
    F->L.v.assign(Lv, Lv + Lrp[n]);
    F->U.rp.assign(Urp, Urp + n + 1);
    F->U.ci.assign(Uc, Uc + Urp[n]);
    F->U.v.assign(Uv, Uv + Urp[n]);
    F->perm.resize(n);
    for (int32_t i = 0; i < n; ++i) F->perm[i] = perm ? perm[i] : i;
    F->pinv.assign(n, 0);
    for (int32_t i = 0; i < n; ++i) F->pinv[F->perm[i]] = i;
    F->levels();
    *out = new orc_factor_s{F, true};
    return PMG_OK;
}
void orc_factor_free(orc_factor F) {
    if (!F) return;
    if (F->own) delete F->F;
    delete F;
}
int orc_factor_stats(orc_factor F, int64_t* nnz_L, int64_t* nnz_U, int32_t* levels_L, int32_t* levels_U) {
    if (nnz_L) *nnz_L = F->F->L.rp.back();
    if (nnz_U) *nnz_U = F->F->U.rp.back();
    if (levels_L) *levels_L = F->F->levL;
    if (levels_U) *levels_U = F->F->levU;
    return PMG_OK;
}
int orc_factor_export(orc_factor h, int32_t* Lrp, int32_t* Lc, double* Lv, int32_t* Urp, int32_t* Uc, double* Uv,
                      int32_t* perm) {
    const Factor& F = *h->F;
    if (Lrp) std::copy(F.L.rp.begin(), F.L.rp.end(), Lrp);
    if (Lc) std::copy(F.L.ci.begin(), F.L.ci.end(), Lc);
    if (Lv) std::copy(F.L.v.begin(), F.L.v.end(), Lv);
    if (Urp) std::copy(F.U.rp.begin(), F.U.rp.end(), Urp);
    if (Uc) std::copy(F.U.ci.begin(), F.U.ci.end(), Uc);
    if (Uv) std::copy(F.U.v.begin(), F.U.v.end(), Uv);
    if (perm) std::copy(F.perm.begin(), F.perm.end(), perm);
    return PMG_OK;
}
int orc_ilut_apply(orc_factor h, const double* r, double* e) {
    const Factor& F = *h->F;
    std::vector<double> y(F.n), x(F.n);
    std::fill(e, e + F.n, 0.0);
    lsolve(F, r, y.data());
    usolve_add(F, y.data(), x.data(), e);
    return PMG_OK;
}
int orc_prolongate(const pmg_csr_view* P, const double* ML, const double* vc, double* vf) {
    for (int32_t i = 0; i < P->nrows; ++i) vf[i] = row_dot(P->rowptr, P->col, P->val, i, vc) / ML[i];
    return PMG_OK;
}
int orc_restrict(const pmg_csr_view* PT, const double* MLc, const double* rf, double* rc) {
    for (int32_t j = 0; j < PT->nrows; ++j) rc[j] = row_dot(PT->rowptr, PT->col, PT->val, j, rf) / MLc[j];
    return PMG_OK;
}

int orc_hier_create(const pmg_hier_desc* d, const orc_factor* ext, orc_hier* out, int* err_level, int64_t* err_row) {
    auto t0 = std::chrono::steady_clock::now();
    auto h = std::make_unique<orc_hier_s>();
    Hier& H = h->H;
    H.np = d->n_plevels;
    H.nh = d->n_hlevels;
    H.smoother = d->smoother;
    H.nu1 = d->nu1;
    H.nu2 = d->nu2;
    H.pl.resize(H.np);
    int next_ext = 0;
    auto get_factor = [&](const Csr& A, const pmg_csr_view& view, int level_tag) -> Factor* {
        if (ext) return ext[next_ext++]->F;
        int64_t er = -1;
        auto F = ilut(view, d->tau, d->fillfactor, d->ordering, &er);
        if (!F) {
            if (err_level) *err_level = level_tag;
            if (err_row) *err_row = er;
            return nullptr;
        }
        (void)A;
        H.owned.push_back(std::move(F));
        return H.owned.back().get();
    };
    for (int l = 0; l < H.np; ++l) {
        PLev& L = H.pl[l];
        L.A = Csr::from(d->A[l]);
        L.ML.assign(d->ML[l], d->ML[l] + L.A.n);
        if (l + 1 < H.np) {
            L.P = Csr::from(d->P[l]);
            L.PT = Csr::from(d->PT[l]);
        }
        L.u.assign(L.A.n, 0.0);
        L.f.assign(L.A.n, 0.0);
        L.r.assign(L.A.n, 0.0);
        L.y.assign(L.A.n, 0.0);
        L.x.assign(L.A.n, 0.0);
    }
    for (int l = 0; l + 1 < H.np; ++l)
        if (H.smoother == PMG_SMOOTHER_ILUT) {
            H.pl[l].F = get_factor(H.pl[l].A, d->A[l], l);
            if (!H.pl[l].F) return PMG_ZERO_PIVOT;
            H.factors.push_back(H.pl[l].F);
        }
    H.hl.resize(H.nh);
    for (int j = 0; j < H.nh; ++j) {
        HLev& L = H.hl[j];
        if (j == 0) L.A = &H.pl.back().A;
        else {
            L.Aown = Csr::from(d->HA[j]);
            L.A = &L.Aown;
        }
        if (j + 1 < H.nh) {
            L.P = Csr::from(d->HP[j]);
            L.PT = Csr::from(d->HPT[j]);
            const pmg_csr_view& v = j == 0 ? d->A[H.np - 1] : d->HA[j];
            L.F = get_factor(*L.A, v, H.np - 1 + j);
            if (!L.F) return PMG_ZERO_PIVOT;
            H.factors.push_back(L.F);
        } else if (!H.coarse.factor(*L.A)) {
            if (err_level) *err_level = H.np - 1 + j;
            return PMG_ZERO_PIVOT;
        }
        int32_t n = L.A->n;
        L.e.assign(n, 0.0);
        L.r.assign(n, 0.0);
        L.res.assign(n, 0.0);
        L.y.assign(n, 0.0);
        L.x.assign(n, 0.0);
    }
    H.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
    return PMG_OK;
}
void orc_hier_free(orc_hier H) { delete H; }
int orc_hier_num_factors(orc_hier H) { return int(H->H.factors.size()); }
orc_factor orc_hier_factor(orc_hier H, int which) { return new orc_factor_s{H->H.factors.at(which), false}; }

// solve: rho_c = ||f - A u_c|| / ||f - A u_0||, stop at
// rho <= tol (converged) or rho > 1e10 / NaN (diverged), at most max_cycles cycles.
int orc_solve(orc_hier h, const double* f, double* u, double tol, int max_cycles, double* hist, int* cycles, int* flags,
              double* solve_seconds, double* setup_seconds) {
    Hier& H = h->H;
    PLev& L = H.pl[0];
    const int32_t n = L.A.n;
    if (setup_seconds) *setup_seconds = H.setup_seconds;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> r(n);
    residual(L.A, u, f, r.data());
    const double n0 = norm2(r.data(), n);
    hist[0] = 1.0;
    *cycles = 0;
    *flags = 0;
    int rc = PMG_OK;
    if (n0 == 0.0) {
        *flags = PMG_FLAG_CONVERGED;
    } else {
        for (int c = 1; c <= max_cycles; ++c) {
            int64_t e = vcycle(H, 0, u, f, r.data(), false);
            if (e >= 0) { rc = PMG_ZERO_DIAG; break; }
            residual(L.A, u, f, r.data());
            const double rho = norm2(r.data(), n) / n0;
            hist[c] = rho;
            *cycles = c;
            if (rho <= tol) { *flags = PMG_FLAG_CONVERGED; break; }
            if (!(rho <= 1e10)) { *flags = PMG_FLAG_DIVERGED; break; }
        }
    }
    if (solve_seconds) *solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

// BiCGSTAB with one V-cycle from zero (right-hand side = the vector) as preconditioner
int orc_bicgstab(orc_hier h, const double* f, double* u, double tol, int max_iter, double* hist, int* iters, int* flags,
                 double* solve_seconds) {
    Hier& H = h->H;
    const int32_t n = H.pl[0].A.n;
    auto t0 = std::chrono::steady_clock::now();
    auto prec = [&](const double* x, double* z) {
        std::fill(z, z + n, 0.0);
        int64_t e = vcycle(H, 0, z, x, x, true);
        return e >= 0 ? int(PMG_ZERO_DIAG) : int(PMG_OK);
    };
    int rc = bicgstab(H.pl[0].A, f, u, tol, max_iter, prec, hist, iters, flags);
    if (solve_seconds) *solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

// BiCGSTAB without preconditioner (SPEC.md:277 example: SPD system vs a dense solve)
int orc_bicgstab_plain(const pmg_csr_view* A, const double* f, double* u, double tol, int max_iter, double* hist,
                       int* iters, int* flags) {
    if (A->nrows != A->ncols) return PMG_ERR_DIM;
    Csr c = Csr::from(*A);
    const int32_t n = c.n;
    auto prec = [&](const double* x, double* z) {
        std::copy(x, x + n, z);
        return int(PMG_OK);
    };
    return bicgstab(c, f, u, tol, max_iter, prec, hist, iters, flags);
}

int orc_cycle(orc_hier h, int level, double* u, const double* f) {
    int64_t e = vcycle(h->H, level, u, f, nullptr, false);
    return e >= 0 ? PMG_ZERO_DIAG : PMG_OK;
}

// one smoothing step at p-level `level` (p = 1: the finest h-level's ILUT smoother), and one
// coarse-grid correction (PAPER §4 steps 2-4: restrict f - A u, one cycle at level+1 from zero,
// prolongate and add) -- the halves of the cycle reduction_factors applies
int orc_smooth(orc_hier h, int level, double* u, const double* f) {
    Hier& H = h->H;
    if (level < 0 || level >= H.np) return PMG_ERR_ARG;
    if (level == H.np - 1) {
        HLev& L = H.hl[0];
        PLev& P = H.pl[level];
        if (!L.F) return PMG_ERR_ARG;  // p = 1 level is the dense coarsest level itself
        ilut_smooth(*L.A, *L.F, u, f, nullptr, P.r.data(), L.y.data(), L.x.data());
        return PMG_OK;
    }
    return smooth(H, level, u, f, nullptr) >= 0 ? PMG_ZERO_DIAG : PMG_OK;
}

int orc_coarse_correction(orc_hier h, int level, double* u, const double* f) {
    Hier& H = h->H;
    if (level < 0 || level >= H.np - 1) return PMG_ERR_ARG;
    PLev& L = H.pl[level];
    PLev& C = H.pl[level + 1];
    residual(L.A, u, f, L.r.data());
    restrict_(L.PT, C.ML.data(), L.r.data(), C.f.data());
    std::fill(C.u.begin(), C.u.end(), 0.0);
    int64_t e = vcycle(H, level + 1, C.u.data(), C.f.data(), nullptr, true);
    if (e >= 0) return PMG_ZERO_DIAG;
    prolong_add(L.P, L.ML.data(), C.u.data(), u);
    return PMG_OK;
}

}  // extern "C"
