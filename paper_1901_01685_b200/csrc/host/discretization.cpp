// Host-side discretization (input generation).  See discretization.hpp.
#include "discretization.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

namespace iga {

// ------------------------------------------------------------------ threads
static int g_threads = 0;
int num_threads() {
    if (g_threads > 0) return g_threads;
    unsigned h = std::thread::hardware_concurrency();
    return h == 0 ? 1 : int(std::min(h, 32u));
}
void set_num_threads(int n) { g_threads = n; }

template <class F>
static void parallel_for(int64_t n, F&& body) {
    int nt = int(std::min<int64_t>(num_threads(), n));
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) body(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (;;) {
                int64_t i = next.fetch_add(1);
                if (i >= n) break;
                body(i);
            }
        });
    for (auto& th : pool) th.join();
}

// ------------------------------------------------------------------ splines
// Open uniform knot vector: p+1 zeros, spans-1 equidistant interior knots, p+1 ones
// (same construction as proj/src/splines.cpp:9-18).
Knots Knots::open_uniform(int p, int spans) {
    if (p < 0 || spans < 1) throw std::invalid_argument("open_uniform: bad degree/spans");
    Knots k;
    k.p = p;
    k.t.assign(p + 1, 0.0);
    for (int i = 1; i < spans; ++i) k.t.push_back(double(i) / spans);
    k.t.insert(k.t.end(), p + 1, 1.0);
    return k;
}

// Span s with t[s] <= x < t[s+1]; x at the right end belongs to the last non-empty
// span (splines.cpp:27-43).
int knot_span(const Knots& kv, double x) {
    const int n = kv.nbasis(), p = kv.p;
    if (!(x >= kv.t.front() && x <= kv.t.back())) throw std::domain_error("knot_span: point outside knot range");
    if (x >= kv.t[n]) return n - 1;
    int lo = p, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        (x < kv.t[mid] ? hi : lo) = mid;
    }
    return lo;
}

// Cox-de Boor triangle; on return B[0..deg] hold the degree-`deg` values of the
// functions active in span s.
static void cox_de_boor(const Knots& kv, int s, double x, int deg, double* B) {
    double left[16], right[16];
    B[0] = 1.0;
    for (int j = 1; j <= deg; ++j) {
        left[j] = x - kv.t[s + 1 - j];
        right[j] = kv.t[s + j] - x;
        double carry = 0.0;
        for (int r = 0; r < j; ++r) {
            double q = B[r] / (right[r + 1] + left[j - r]);
            B[r] = carry + right[r + 1] * q;
            carry = left[j - r] * q;
        }
        B[j] = carry;
    }
}

int basis_values(const Knots& kv, double x, double* N) {
    int s = knot_span(kv, x);
    cox_de_boor(kv, s, x, kv.p, N);
    return s - kv.p;
}

// First derivatives from the degree p-1 values:
//   N'_{i,p} = p ( N_{i,p-1}/(t_{i+p}-t_i) - N_{i+1,p-1}/(t_{i+p+1}-t_{i+1}) )
int basis_values_d1(const Knots& kv, double x, double* N, double* dN) {
    const int p = kv.p;
    int s = knot_span(kv, x);
    cox_de_boor(kv, s, x, p, N);
    if (p == 0) {
        dN[0] = 0.0;
        return s;
    }
    double Nm[16];
    cox_de_boor(kv, s, x, p - 1, Nm);  // functions s-p+1 .. s of degree p-1
    for (int r = 0; r <= p; ++r) {
        int i = s - p + r;
        double a = 0.0, b = 0.0;
        if (r >= 1) a = Nm[r - 1] / (kv.t[i + p] - kv.t[i]);
        if (r <= p - 1) b = Nm[r] / (kv.t[i + p + 1] - kv.t[i + 1]);
        dN[r] = p * (a - b);
    }
    return s - p;
}

// ------------------------------------------------------------------ geometry
NurbsPatch NurbsPatch::affine(double x0, double y0, double sx, double sy) {
    NurbsPatch g;
    g.gx = Knots::open_uniform(1, 1);
    g.gy = Knots::open_uniform(1, 1);
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
            g.cx.push_back(x0 + sx * a);
            g.cy.push_back(y0 + sy * b);
            g.w.push_back(1.0);
        }
    return g;
}

// Exact quarter annulus: linear in xi (radius r_in..r_out), rational quadratic arc in
// eta (weights 1, sqrt(2)/2, 1) -- SPEC.md:86.  xi radial so det J > 0.
NurbsPatch NurbsPatch::quarter_annulus(double r_in, double r_out) {
    NurbsPatch g;
    g.gx = Knots::open_uniform(1, 1);
    g.gy = Knots::open_uniform(2, 1);
    const double arc[3][2] = {{1, 0}, {1, 1}, {0, 1}};
    const double wa[3] = {1.0, std::sqrt(0.5), 1.0};
    for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 2; ++a) {
            double r = a == 0 ? r_in : r_out;
            g.cx.push_back(r * arc[b][0]);
            g.cy.push_back(r * arc[b][1]);
            g.w.push_back(wa[b]);
        }
    return g;
}

void NurbsPatch::map(double xi, double eta, double X[2], double J[2][2]) const {
    double Nx[16], dNx[16], Ny[16], dNy[16];
    int fx = basis_values_d1(gx, xi, Nx, dNx);
    int fy = basis_values_d1(gy, eta, Ny, dNy);
    const int nx = gx.nbasis();
    double W = 0, Wx = 0, Wy = 0, S[2] = {0, 0}, Sx[2] = {0, 0}, Sy[2] = {0, 0};
    for (int b = 0; b <= gy.p; ++b)
        for (int a = 0; a <= gx.p; ++a) {
            int k = (fx + a) + (fy + b) * nx;
            double wk = w[k];
            double v = Nx[a] * Ny[b] * wk, vx = dNx[a] * Ny[b] * wk, vy = Nx[a] * dNy[b] * wk;
            W += v; Wx += vx; Wy += vy;
            S[0] += v * cx[k]; S[1] += v * cy[k];
            Sx[0] += vx * cx[k]; Sx[1] += vx * cy[k];
            Sy[0] += vy * cx[k]; Sy[1] += vy * cy[k];
        }
    for (int r = 0; r < 2; ++r) {
        X[r] = S[r] / W;
        J[r][0] = (Sx[r] - X[r] * Wx) / W;
        J[r][1] = (Sy[r] - X[r] * Wy) / W;
    }
}

bool Domain::is_interface(int patch, int edge) const {
    for (auto& g : glue)
        if ((g.pa == patch && g.ea == edge) || (g.pb == patch && g.eb == edge)) return true;
    return false;
}

// local index of the k-th DOF along edge e of an n x n patch
static int edge_dof(int e, int k, int n) {
    switch (e) {
        case 0: return k;                    // iy = 0
        case 1: return (n - 1) + k * n;      // ix = n-1
        case 2: return k + (n - 1) * n;      // iy = n-1
        default: return k * n;               // ix = 0
    }
}

// Patch-major numbering; a DOF on an interface edge takes the index already given to
// its partner on the lower-numbered patch (SPEC.md:44-49 glue map).
Space Space::build(const Domain& dom, int p, int nel) {
    Space sp;
    sp.p = p;
    sp.nel = nel;
    const int n = nel + p;
    sp.nloc = n * n;
    const int np = int(dom.patches.size());
    sp.l2g.assign(np, std::vector<int32_t>(sp.nloc, -1));
    int32_t next = 0;
    for (int P = 0; P < np; ++P) {
        for (auto& g : dom.glue) {
            int me = -1, other = -1, e_me = -1, e_other = -1;
            if (g.pa == P && g.pb < P) { me = g.pa; e_me = g.ea; other = g.pb; e_other = g.eb; }
            if (g.pb == P && g.pa < P) { me = g.pb; e_me = g.eb; other = g.pa; e_other = g.ea; }
            if (me < 0) continue;
            for (int k = 0; k < n; ++k) {
                int lo = edge_dof(e_other, k, n), lm = edge_dof(e_me, k, n);
                if (sp.l2g[P][lm] < 0) sp.l2g[P][lm] = sp.l2g[other][lo];
            }
        }
        for (int i = 0; i < sp.nloc; ++i)
            if (sp.l2g[P][i] < 0) sp.l2g[P][i] = next++;
    }
    sp.ndof = next;
    if (dom.rowmajor && np > 1) {
        // global row-major renumbering: key (gy, gx) of the DOF in the domain's control grid
        std::vector<int64_t> key(next, -1);
        const int64_t W = int64_t(n) * 8;
        for (int P = 0; P < np; ++P)
            for (int iy = 0; iy < n; ++iy)
                for (int ix = 0; ix < n; ++ix) {
                    const int64_t gx = ix + int64_t(dom.grid_off[P][0]) * (n - 1);
                    const int64_t gy = iy + int64_t(dom.grid_off[P][1]) * (n - 1);
                    const int64_t k = gy * W + gx;
                    int64_t& slot = key[sp.l2g[P][ix + iy * n]];
                    if (slot >= 0 && slot != k) throw AssemblyError("row-major numbering: glue is not conforming");
                    slot = k;
                }
        std::vector<int32_t> order(next);
        for (int32_t i = 0; i < next; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
        std::vector<int32_t> rank(next);
        for (int32_t r = 0; r < next; ++r) rank[order[r]] = r;
        for (auto& m : sp.l2g)
            for (auto& g : m) g = rank[g];
    }
    return sp;
}

// ------------------------------------------------------------------ quadrature
void gauss01(int n, double* x, double* w) {
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int k = 1; k <= n; ++k) {
                double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
            }
            dp = n * (z * p0 - p1) / (z * z - 1.0);
            double dz = p0 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[n - 1 - i] = 0.5 * (1.0 + z);  // ascending nodes on [0,1]
        w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);
    }
}

// ------------------------------------------------------------------ sparsity
// Row pattern: union over the patches containing the row DOF of the tensor band
// [i-lo, i+hi] per direction (basis functions overlap iff their index distance is
// within the band).  rows of space `rs`, columns of space `cs` (same mesh).
static HostCsr make_pattern(const Domain& dom, const Space& rs, const Space& cs) {
    const int np = int(dom.patches.size());
    const int nr = rs.nel + rs.p, nc = cs.nel + cs.p;
    const int lo = rs.p, hi = cs.p;  // col index c overlaps row index r iff r-lo <= c <= r+hi
    // global row -> list of (patch, local)
    std::vector<int32_t> cnt(rs.ndof + 1, 0);
    for (int P = 0; P < np; ++P)
        for (int i = 0; i < rs.nloc; ++i) cnt[rs.l2g[P][i] + 1]++;
    for (int i = 0; i < rs.ndof; ++i) cnt[i + 1] += cnt[i];
    std::vector<int32_t> occ(cnt[rs.ndof]);
    {
        std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
        for (int P = 0; P < np; ++P)
            for (int i = 0; i < rs.nloc; ++i) occ[pos[rs.l2g[P][i]]++] = P * rs.nloc + i;
    }
    HostCsr A;
    A.nrows = rs.ndof;
    A.ncols = cs.ndof;
    A.rowptr.assign(rs.ndof + 1, 0);
    // columns of row g, ascending and unique, into v
    auto row_cols = [&](int32_t g, std::vector<int32_t>& v) {
        v.clear();
        const bool multi = cnt[g + 1] - cnt[g] > 1;
        for (int o = cnt[g]; o < cnt[g + 1]; ++o) {
            int P = occ[o] / rs.nloc, loc = occ[o] % rs.nloc;
            int ix = loc % nr, iy = loc / nr;
            const int32_t* map = cs.l2g[P].data();
            for (int jy = std::max(0, iy - lo); jy <= std::min(nc - 1, iy + hi); ++jy)
                for (int jx = std::max(0, ix - lo); jx <= std::min(nc - 1, ix + hi); ++jx) v.push_back(map[jx + jy * nc]);
        }
        if (multi || np > 1) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        }
    };
    // two passes over blocks of rows (lengths, then columns): no per-row allocations
    const int64_t nblk = (rs.ndof + 1023) / 1024;
    parallel_for(nblk, [&](int64_t blk) {
        std::vector<int32_t> v;
        int32_t r0 = int32_t(blk * 1024), r1 = std::min<int32_t>(rs.ndof, r0 + 1024);
        for (int32_t g = r0; g < r1; ++g) {
            row_cols(g, v);
            A.rowptr[g + 1] = int64_t(v.size());
        }
    });
    for (int32_t g = 0; g < rs.ndof; ++g) A.rowptr[g + 1] += A.rowptr[g];
    A.col.resize(A.rowptr.back());
    A.val.resize(A.rowptr.back());
    parallel_for(nblk, [&](int64_t blk) {
        std::vector<int32_t> v;
        int32_t r0 = int32_t(blk * 1024), r1 = std::min<int32_t>(rs.ndof, r0 + 1024);
        for (int32_t g = r0; g < r1; ++g) {
            row_cols(g, v);
            std::copy(v.begin(), v.end(), A.col.begin() + A.rowptr[g]);
        }
    });
    return A;
}

// the host element loops accumulate into the values: start from +0 (parallel first touch)
static void zero_values(HostCsr& A) {
    const int64_t nnz = A.nnz(), blk = int64_t(1) << 20;
    parallel_for((nnz + blk - 1) / blk, [&](int64_t b) {
        std::fill(A.val.begin() + b * blk, A.val.begin() + std::min(nnz, (b + 1) * blk), 0.0);
    });
}

static inline int64_t find_pos(const HostCsr& A, int32_t row, int32_t col) {
    const int32_t* b = A.col.data() + A.rowptr[row];
    const int32_t* e = A.col.data() + A.rowptr[row + 1];
    const int32_t* it = std::lower_bound(b, e, col);
    if (it == e || *it != col) throw AssemblyError("assembly: entry outside sparsity pattern");
    return it - A.col.data();
}

// ------------------------------------------------------------------ element data
struct Basis1D {  // per element e, per qp a: values/derivs of the p+1 active functions
    int p, nq, nel;
    std::vector<double> xq, wq;      // qp in [0,1] param (global), weights (param length incl.)
    std::vector<double> B, dB;       // [(e*nq + a)*(p+1) + r]
    void build(int p_, int nel_, int nq_) {
        p = p_; nel = nel_; nq = nq_;
        Knots kv = Knots::open_uniform(p, nel);
        double g[32], gw[32];
        gauss01(nq, g, gw);
        xq.resize(size_t(nel) * nq); wq.resize(size_t(nel) * nq);
        B.resize(size_t(nel) * nq * (p + 1)); dB.resize(B.size());
        const double h = 1.0 / nel;
        for (int e = 0; e < nel; ++e)
            for (int a = 0; a < nq; ++a) {
                double x = (e + g[a]) * h;
                xq[e * nq + a] = x;
                wq[e * nq + a] = gw[a] * h;
                int first = basis_values_d1(kv, x, &B[(size_t(e) * nq + a) * (p + 1)], &dB[(size_t(e) * nq + a) * (p + 1)]);
                if (first != e) throw AssemblyError("basis: unexpected span");
            }
    }
    const double* b(int e, int a) const { return &B[(size_t(e) * nq + a) * (p + 1)]; }
    const double* d(int e, int a) const { return &dB[(size_t(e) * nq + a) * (p + 1)]; }
};

// colour-major strip scheduling: blocks of `hgt` element rows, two colours, so no two
// concurrently processed blocks touch a common DOF row.
template <class F>
static void for_each_element_strip(int nel, int hgt, F&& strip) {
    int nblk = (nel + hgt - 1) / hgt;
    for (int colour = 0; colour < 2; ++colour) {
        int m = (nblk - colour + 1) / 2;
        parallel_for(m, [&](int64_t k) {
            int blk = colour + 2 * int(k);
            for (int ey = blk * hgt; ey < std::min(nel, (blk + 1) * hgt); ++ey) strip(ey);
        });
    }
}

static inline void inv2(const double J[2][2], double G[2][2], double& det) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    G[0][0] = J[1][1] / det;  G[0][1] = -J[0][1] / det;
    G[1][0] = -J[1][0] / det; G[1][1] = J[0][0] / det;
}

// scatter a dense element matrix E[(i1 + j1*n1)][(i2 + j2*n2)] into A
static void scatter(HostCsr& A, const std::vector<int32_t>& rmap, const std::vector<int32_t>& cmap, int nr_loc, int nc_loc,
                    int ex, int ey, int n1, int n2, const double* E) {
    const int ncols = n2 * n2;
    for (int j1 = 0; j1 < n1; ++j1)
        for (int i1 = 0; i1 < n1; ++i1) {
            int32_t row = rmap[(ex + i1) + (ey + j1) * nr_loc];
            const double* Er = E + (i1 + j1 * n1) * ncols;
            for (int j2 = 0; j2 < n2; ++j2) {
                int32_t c0 = cmap[ex + (ey + j2) * nc_loc];
                int64_t pos = find_pos(A, row, c0);
                const int64_t rend = A.rowptr[row + 1];
                for (int i2 = 0; i2 < n2; ++i2) {
                    int32_t c = cmap[(ex + i2) + (ey + j2) * nc_loc];
                    if (pos + i2 >= rend || A.col[pos + i2] != c) pos = find_pos(A, row, c) - i2;  // non-monotone glue
                    A.val[pos + i2] += Er[i2 + j2 * n2];
                }
            }
        }
}

// ------------------------------------------------------------------ external values (F2)
// 1D tables of the request (include/pmg_asm.h): a basis at the nel*nq Gauss abscissae followed
// by x = 0 and x = 1, evaluated by the same basis_values_d1 calls the element loop makes.
struct Table1D {
    std::vector<double> B, dB;
    std::vector<int32_t> first;
    pmg_asm_table1d view{};
    void build(const Knots& kv, const std::vector<double>& pts) {
        const int p = kv.p;
        B.assign(pts.size() * (p + 1), 0.0);
        dB.assign(B.size(), 0.0);
        first.resize(pts.size());
        for (size_t i = 0; i < pts.size(); ++i) first[i] = basis_values_d1(kv, pts[i], &B[i * (p + 1)], &dB[i * (p + 1)]);
        view = {p, int32_t(pts.size()), B.data(), dB.data(), first.data()};
    }
};

// NurbsPatch::map with the geometry bases read from tables (the same basis_values_d1 results,
// the same loop: identical X and J)
static void tab_map(const NurbsPatch& g, const Table1D& tx, const Table1D& ty, int ptx, int pty, double X[2], double J[2][2]) {
    const int px = g.gx.p, py = g.gy.p, nx = g.gx.nbasis();
    const double *Nx = &tx.B[size_t(ptx) * (px + 1)], *dNx = &tx.dB[size_t(ptx) * (px + 1)];
    const double *Ny = &ty.B[size_t(pty) * (py + 1)], *dNy = &ty.dB[size_t(pty) * (py + 1)];
    const int fx = tx.first[ptx], fy = ty.first[pty];
    double W = 0, Wx = 0, Wy = 0, S[2] = {0, 0}, Sx[2] = {0, 0}, Sy[2] = {0, 0};
    for (int b = 0; b <= py; ++b)
        for (int a = 0; a <= px; ++a) {
            int k = (fx + a) + (fy + b) * nx;
            double wk = g.w[k];
            double v = Nx[a] * Ny[b] * wk, vx = dNx[a] * Ny[b] * wk, vy = Nx[a] * dNy[b] * wk;
            W += v; Wx += vx; Wy += vy;
            S[0] += v * g.cx[k]; S[1] += v * g.cy[k];
            Sx[0] += vx * g.cx[k]; Sx[1] += vx * g.cy[k];
            Sy[0] += vy * g.cx[k]; Sy[1] += vy * g.cy[k];
        }
    for (int r = 0; r < 2; ++r) {
        X[r] = S[r] / W;
        J[r][0] = (Sx[r] - X[r] * Wx) / W;
        J[r][1] = (Sy[r] - X[r] * Wy) / W;
    }
}

// `pattern` (optional): an operator with the sparsity pattern of the request (M_k has A_k's);
// with `lumped` only the row sums are produced and the returned matrix is empty.
static HostCsr external_values(const Domain& dom, const Space& rs, const Space& cs, const Cdr* c, int nq, int strip,
                               pmg_asm_values_fn values, const HostCsr* pattern = nullptr,
                               std::vector<double>* lumped = nullptr) {
    const bool verbose = std::getenv("IGA_VERBOSE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!verbose) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[iga]   %-18s p %d/%d: %.3f s\n", what, rs.p, cs.p, std::chrono::duration<double>(t - t0).count());
        t0 = t;
    };
    HostCsr A;
    if (!pattern) {
        A = make_pattern(dom, rs, cs);
        pattern = &A;
    }
    if (pattern == &A) zero_values(A);  // parallel first touch of the pages the producer copies into
    lap("pattern");
    if (lumped) lumped->assign(pattern->nrows, 0.0);
    const int nel = rs.nel;
    Basis1D bs;
    bs.build(rs.p, nel, nq);
    std::vector<double> pts(bs.xq);
    pts.push_back(0.0);
    pts.push_back(1.0);
    Table1D tr, tc;
    tr.build(Knots::open_uniform(rs.p, nel), pts);
    tc.build(Knots::open_uniform(cs.p, nel), pts);
    const int np = int(dom.patches.size());
    std::vector<Table1D> gx(np), gy(np);
    std::vector<pmg_asm_patch> pv(np);
    for (int P = 0; P < np; ++P) {
        const NurbsPatch& g = dom.patches[P];
        gx[P].build(g.gx, pts);
        gy[P].build(g.gy, pts);
        int mask = 0;
        for (int e = 0; e < 4; ++e)
            if (!dom.is_interface(P, e)) mask |= 1 << e;
        pv[P] = {gx[P].view, gy[P].view, g.gx.nbasis(), g.cx.data(), g.cy.data(), g.w.data(),
                 rs.l2g[P].data(), cs.l2g[P].data(), mask};
    }
    pmg_asm_request rq{};
    rq.kind = c ? PMG_ASM_OPERATOR : PMG_ASM_MASS;
    rq.nel = nel;
    rq.nq = nq;
    rq.npts = int32_t(pts.size());
    rq.strip = strip;
    rq.wq = bs.wq.data();
    rq.row = tr.view;
    rq.col = tc.view;
    rq.n_patches = np;
    rq.patches = pv.data();
    if (c) {
        for (int i = 0; i < 4; ++i) rq.D[i] = c->D[i / 2][i % 2];
        rq.v[0] = c->v[0];
        rq.v[1] = c->v[1];
        rq.R = c->R;
        rq.penalty = c->nitsche_scale * 4.0 * rs.p * rs.p * nel;
    }
    rq.nrows = pattern->nrows;
    rq.ncols = pattern->ncols;
    rq.rowptr = pattern->rowptr.data();
    rq.col_idx = pattern->col.data();
    rq.val = pattern == &A ? A.val.data() : nullptr;
    rq.lumped = lumped ? lumped->data() : nullptr;
    lap("tables");
    const int rc = values(&rq);
    lap("values (producer)");
    if (rc == 1) throw GeometryError("nonpositive Jacobian determinant");
    if (rc != 0) throw AssemblyError("external assembler failed (status " + std::to_string(rc) + ")");
    return A;
}

// ------------------------------------------------------------------ assembly
// a(u,v) = int (D grad u).grad v + (v.grad u) v + R u v  +  symmetric Nitsche on the
// Dirichlet boundary:  - int (D grad u.n) v - int (D grad v.n) u + (eta/h) int u v,
// eta = 4 p^2, h = 1/nel.  rhs = (f, v), plus the Nitsche
// consistency terms -int (D grad v.n) g + (eta/h) int g v of inhomogeneous Dirichlet data g
// (Benchmark 3).
HostCsr assemble_operator(const Domain& dom, const Space& sp, const Cdr& c, std::vector<double>* rhs,
                          pmg_asm_values_fn values) {
    const int p = sp.p, nel = sp.nel, n1 = p + 1, n = nel + p, nq = p + 1;
    // with an external producer of the values the loop below only forms the load vector
    const bool ext = values != nullptr;
    if (ext && !rhs) return external_values(dom, sp, sp, &c, nq, p + 1, values);
    HostCsr A = ext ? external_values(dom, sp, sp, &c, nq, p + 1, values) : make_pattern(dom, sp, sp);
    if (!ext) zero_values(A);
    Basis1D bs;
    bs.build(p, nel, nq);
    if (rhs) rhs->assign(sp.ndof, 0.0);
    const double pen = c.nitsche_scale * 4.0 * p * p * nel;  // eta / h
    const int nloc2 = n1 * n1;
    for (size_t P = 0; P < dom.patches.size(); ++P) {
        const NurbsPatch& geo = dom.patches[P];
        const auto& l2g = sp.l2g[P];
        Table1D tgx, tgy;  // geometry bases at the abscissae (load-vector-only pass)
        if (ext) {
            tgx.build(geo.gx, bs.xq);
            tgy.build(geo.gy, bs.xq);
        }
        for_each_element_strip(nel, p + 1, [&](int ey) {
            std::vector<double> E(size_t(nloc2) * nloc2), S(4 * size_t(nq) * n1 * n1);
            std::vector<double> K(4 * nq * nq), C(2 * nq * nq), Mr(nq * nq), Fq(nq * nq), Fb(nloc2);
            for (int ex = 0; ex < nel; ++ex) {
                // geometric factors at the (p+1)^2 points
                for (int b = 0; b < nq; ++b)
                    for (int a = 0; a < nq; ++a) {
                        double X[2], J[2][2], G[2][2], det;
                        if (ext) tab_map(geo, tgx, tgy, ex * nq + a, ey * nq + b, X, J);
                        else geo.map(bs.xq[ex * nq + a], bs.xq[ey * nq + b], X, J);
                        inv2(J, G, det);
                        if (!(det > 0)) throw GeometryError("nonpositive Jacobian determinant");
                        double w = bs.wq[ex * nq + a] * bs.wq[ey * nq + b] * det;
                        int q = a + b * nq;
                        if (ext) {  // only the load vector is formed here
                            Fq[q] = c.f ? w * c.f(X[0], X[1]) : 0.0;
                            continue;
                        }
                        // K = w G D G^T (parametric diffusion tensor)
                        for (int r = 0; r < 2; ++r)
                            for (int s = 0; s < 2; ++s) {
                                double acc = 0;
                                for (int m = 0; m < 2; ++m)
                                    for (int l = 0; l < 2; ++l) acc += G[r][m] * c.D[m][l] * G[s][l];
                                K[(r * 2 + s) * nq * nq + q] = w * acc;
                            }
                        for (int r = 0; r < 2; ++r) C[r * nq * nq + q] = w * (G[r][0] * c.v[0] + G[r][1] * c.v[1]);
                        Mr[q] = w * c.R;
                        Fq[q] = c.f ? w * c.f(X[0], X[1]) : 0.0;
                    }
                // stage 1: contract over the xi points
                std::fill(S.begin(), S.end(), 0.0);
                for (int b = 0; b < (ext ? 0 : nq); ++b)
                    for (int a = 0; a < nq; ++a) {
                        int q = a + b * nq;
                        const double *Bx = bs.b(ex, a), *dBx = bs.d(ex, a);
                        double k00 = K[0 * nq * nq + q], k01 = K[1 * nq * nq + q], k10 = K[2 * nq * nq + q], k11 = K[3 * nq * nq + q];
                        double c0 = C[q], c1 = C[nq * nq + q], m = Mr[q];
                        double* Syy = &S[((0 * nq + b) * n1) * n1];
                        double* Syd = &S[((1 * nq + b) * n1) * n1];
                        double* Sdy = &S[((2 * nq + b) * n1) * n1];
                        double* Sdd = &S[((3 * nq + b) * n1) * n1];
                        for (int i1 = 0; i1 < n1; ++i1)
                            for (int i2 = 0; i2 < n1; ++i2) {
                                Syy[i1 * n1 + i2] += k00 * dBx[i1] * dBx[i2] + c0 * Bx[i1] * dBx[i2] + m * Bx[i1] * Bx[i2];
                                Syd[i1 * n1 + i2] += k01 * dBx[i1] * Bx[i2] + c1 * Bx[i1] * Bx[i2];
                                Sdy[i1 * n1 + i2] += k10 * Bx[i1] * dBx[i2];
                                Sdd[i1 * n1 + i2] += k11 * Bx[i1] * Bx[i2];
                            }
                    }
                // stage 2: contract over the eta points
                std::fill(E.begin(), E.end(), 0.0);
                for (int b = 0; b < (ext ? 0 : nq); ++b) {
                    const double *By = bs.b(ey, b), *dBy = bs.d(ey, b);
                    const double* Syy = &S[((0 * nq + b) * n1) * n1];
                    const double* Syd = &S[((1 * nq + b) * n1) * n1];
                    const double* Sdy = &S[((2 * nq + b) * n1) * n1];
                    const double* Sdd = &S[((3 * nq + b) * n1) * n1];
                    for (int j1 = 0; j1 < n1; ++j1)
                        for (int j2 = 0; j2 < n1; ++j2) {
                            double yy = By[j1] * By[j2], yd = By[j1] * dBy[j2], dy = dBy[j1] * By[j2], dd = dBy[j1] * dBy[j2];
                            for (int i1 = 0; i1 < n1; ++i1) {
                                double* Er = &E[size_t(i1 + j1 * n1) * nloc2 + j2 * n1];
                                const int o = i1 * n1;
                                for (int i2 = 0; i2 < n1; ++i2)
                                    Er[i2] += yy * Syy[o + i2] + yd * Syd[o + i2] + dy * Sdy[o + i2] + dd * Sdd[o + i2];
                            }
                        }
                }
                // Nitsche terms on Dirichlet edges touched by this element
                std::fill(Fb.begin(), Fb.end(), 0.0);
                for (int edge = 0; edge < 4; ++edge) {
                    bool on = (edge == 0 && ey == 0) || (edge == 1 && ex == nel - 1) || (edge == 2 && ey == nel - 1) ||
                              (edge == 3 && ex == 0);
                    if (!on || dom.is_interface(int(P), edge)) continue;
                    Knots kv = Knots::open_uniform(p, nel);
                    for (int a = 0; a < nq; ++a) {
                        bool horiz = (edge == 0 || edge == 2);
                        int e_along = horiz ? ex : ey;
                        double s = bs.xq[e_along * nq + a], ws = bs.wq[e_along * nq + a];
                        double xi = horiz ? s : (edge == 1 ? 1.0 : 0.0);
                        double eta = horiz ? (edge == 2 ? 1.0 : 0.0) : s;
                        double X[2], J[2][2], G[2][2], det;
                        geo.map(xi, eta, X, J);
                        inv2(J, G, det);
                        double t[2] = {horiz ? J[0][0] : J[0][1], horiz ? J[1][0] : J[1][1]};
                        double tl = std::sqrt(t[0] * t[0] + t[1] * t[1]);
                        double nv[2];
                        if (edge == 0 || edge == 1) { nv[0] = t[1] / tl; nv[1] = -t[0] / tl; }
                        else { nv[0] = -t[1] / tl; nv[1] = t[0] / tl; }
                        double Nx[16], dNx[16], Ny[16], dNy[16];
                        int fx = basis_values_d1(kv, xi, Nx, dNx), fy = basis_values_d1(kv, eta, Ny, dNy);
                        if (fx != ex || fy != ey) throw AssemblyError("boundary basis span mismatch");
                        double phi[64], flux[64];
                        for (int j = 0; j < n1; ++j)
                            for (int i = 0; i < n1; ++i) {
                                double g0 = dNx[i] * Ny[j], g1 = Nx[i] * dNy[j];
                                double gx0 = G[0][0] * g0 + G[1][0] * g1, gx1 = G[0][1] * g0 + G[1][1] * g1;  // G^T grad
                                double dg0 = c.D[0][0] * gx0 + c.D[0][1] * gx1, dg1 = c.D[1][0] * gx0 + c.D[1][1] * gx1;
                                phi[i + j * n1] = Nx[i] * Ny[j];
                                flux[i + j * n1] = dg0 * nv[0] + dg1 * nv[1];
                            }
                        double w = ws * tl;
                        for (int te = 0; te < (ext ? 0 : nloc2); ++te)
                            for (int tr = 0; tr < nloc2; ++tr)
                                E[size_t(te) * nloc2 + tr] += w * (-flux[tr] * phi[te] - flux[te] * phi[tr] + pen * phi[te] * phi[tr]);
                        if (rhs && c.g) {  // consistency terms of inhomogeneous data: -int (D grad v.n) g + (eta/h) int g v
                            const double gv = c.g(X[0], X[1]);
                            for (int te = 0; te < nloc2; ++te) Fb[te] += w * (-flux[te] * gv + pen * phi[te] * gv);
                        }
                    }
                }
                if (!ext) scatter(A, l2g, l2g, n, n, ex, ey, n1, n1, E.data());
                if (rhs) {
                    for (int j1 = 0; j1 < n1; ++j1)
                        for (int i1 = 0; i1 < n1; ++i1) {
                            double acc = 0;
                            for (int b = 0; b < nq; ++b)
                                for (int a = 0; a < nq; ++a) acc += Fq[a + b * nq] * bs.b(ex, a)[i1] * bs.b(ey, b)[j1];
                            (*rhs)[l2g[(ex + i1) + (ey + j1) * n]] += acc + Fb[i1 + j1 * n1];
                        }
                }
            }
        });
    }
    return A;
}

// Mixed mass  P_ij = int phi_i^{(k)} phi_j^{(j)} dOmega over a common mesh; with the same
// space on both sides this is the mass matrix M_k (eq. (24)).
static HostCsr assemble_mixed_mass(const Domain& dom, const Space& rs, const Space& cs, pmg_asm_values_fn values) {
    if (rs.nel != cs.nel) throw AssemblyError("transfer: spaces on different meshes");
    if (values) return external_values(dom, rs, cs, nullptr, std::max(rs.p, cs.p) + 1, std::max(rs.p, cs.p) + 1, values);
    HostCsr A = make_pattern(dom, rs, cs);
    zero_values(A);
    const int nel = rs.nel, n1 = rs.p + 1, n2 = cs.p + 1, nq = std::max(rs.p, cs.p) + 1;
    const int nr = nel + rs.p, nc = nel + cs.p;
    Basis1D br, bc;
    br.build(rs.p, nel, nq);
    bc.build(cs.p, nel, nq);
    for (size_t P = 0; P < dom.patches.size(); ++P) {
        const NurbsPatch& geo = dom.patches[P];
        for_each_element_strip(nel, std::max(rs.p, cs.p) + 1, [&](int ey) {
            std::vector<double> E(size_t(n1 * n1) * n2 * n2), S(size_t(nq) * n1 * n2), W(nq * nq);
            for (int ex = 0; ex < nel; ++ex) {
                for (int b = 0; b < nq; ++b)
                    for (int a = 0; a < nq; ++a) {
                        double X[2], J[2][2];
                        geo.map(br.xq[ex * nq + a], br.xq[ey * nq + b], X, J);
                        double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
                        if (!(det > 0)) throw GeometryError("nonpositive Jacobian determinant");
                        W[a + b * nq] = br.wq[ex * nq + a] * br.wq[ey * nq + b] * det;
                    }
                std::fill(S.begin(), S.end(), 0.0);
                for (int b = 0; b < nq; ++b)
                    for (int a = 0; a < nq; ++a) {
                        const double *Bx = br.b(ex, a), *Cx = bc.b(ex, a);
                        double w = W[a + b * nq];
                        for (int i1 = 0; i1 < n1; ++i1)
                            for (int i2 = 0; i2 < n2; ++i2) S[(b * n1 + i1) * n2 + i2] += w * Bx[i1] * Cx[i2];
                    }
                std::fill(E.begin(), E.end(), 0.0);
                const int ncl = n2 * n2;
                for (int b = 0; b < nq; ++b) {
                    const double *By = br.b(ey, b), *Cy = bc.b(ey, b);
                    for (int j1 = 0; j1 < n1; ++j1)
                        for (int j2 = 0; j2 < n2; ++j2) {
                            double yy = By[j1] * Cy[j2];
                            for (int i1 = 0; i1 < n1; ++i1)
                                for (int i2 = 0; i2 < n2; ++i2)
                                    E[size_t(i1 + j1 * n1) * ncl + i2 + j2 * n2] += yy * S[(b * n1 + i1) * n2 + i2];
                        }
                }
                scatter(A, rs.l2g[P], cs.l2g[P], nr, nc, ex, ey, n1, n2, E.data());
            }
        });
    }
    return A;
}

HostCsr assemble_mass(const Domain& dom, const Space& sp, pmg_asm_values_fn values) {
    return assemble_mixed_mass(dom, sp, sp, values);
}
HostCsr assemble_transfer(const Domain& dom, const Space& fine_p, const Space& coarse_p, pmg_asm_values_fn values) {
    return assemble_mixed_mass(dom, fine_p, coarse_p, values);
}

// Row-sum lumping M^L_ii = sum_j M_ij, ascending column order.
std::vector<double> lump(const HostCsr& M) {
    std::vector<double> d(M.nrows);
    for (int32_t i = 0; i < M.nrows; ++i) {
        double s = 0.0;
        for (int64_t k = M.rowptr[i]; k < M.rowptr[i + 1]; ++k) s += M.val[k];
        if (!(s > 0)) throw AssemblyError("lump_mass: nonpositive row sum");
        d[i] = s;
    }
    return d;
}
std::vector<double> lumped_mass(const Domain& dom, const Space& sp, pmg_asm_values_fn values, const HostCsr* pattern) {
    if (!values) return lump(assemble_mass(dom, sp));
    // external producer: M_k's values stay with it, only the row sums come back
    std::vector<double> d;
    external_values(dom, sp, sp, nullptr, sp.p + 1, sp.p + 1, values, pattern, &d);
    for (double s : d)
        if (!(s > 0)) throw AssemblyError("lump_mass: nonpositive row sum");
    return d;
}

// p = 1 knot insertion (coarse nel -> 2 nel): coarse hat J = fine hat 2J + (fine hats 2J+-1)/2,
// i.e. linear interpolation of nodal coefficients.
HostCsr hrefine_p1(const Domain& dom, const Space& fine, const Space& coarse) {
    if (fine.p != 1 || coarse.p != 1 || fine.nel != 2 * coarse.nel) throw AssemblyError("hrefine_p1: bad spaces");
    const int nf = fine.nel + 1, nc = coarse.nel + 1;
    auto q1 = [&](int i, int* J, double* v) -> int {  // 1D row i of Q
        if (i % 2 == 0) { J[0] = i / 2; v[0] = 1.0; return 1; }
        J[0] = i / 2; J[1] = i / 2 + 1; v[0] = 0.5; v[1] = 0.5; return 2;
    };
    std::vector<std::vector<std::pair<int32_t, double>>> rows(fine.ndof);
    std::vector<char> done(fine.ndof, 0);
    for (size_t P = 0; P < dom.patches.size(); ++P)
        for (int iy = 0; iy < nf; ++iy)
            for (int ix = 0; ix < nf; ++ix) {
                int32_t g = fine.l2g[P][ix + iy * nf];
                if (done[g]) continue;
                done[g] = 1;
                int Jx[2], Jy[2];
                double vx[2], vy[2];
                int mx = q1(ix, Jx, vx), my = q1(iy, Jy, vy);
                for (int b = 0; b < my; ++b)
                    for (int a = 0; a < mx; ++a) rows[g].push_back({coarse.l2g[P][Jx[a] + Jy[b] * nc], vx[a] * vy[b]});
                std::sort(rows[g].begin(), rows[g].end());
            }
    HostCsr Q;
    Q.nrows = fine.ndof;
    Q.ncols = coarse.ndof;
    Q.rowptr.assign(fine.ndof + 1, 0);
    for (int32_t g = 0; g < fine.ndof; ++g) Q.rowptr[g + 1] = Q.rowptr[g] + int64_t(rows[g].size());
    for (auto& r : rows)
        for (auto& e : r) { Q.col.push_back(e.first); Q.val.push_back(e.second); }
    return Q;
}

// CSR transpose; rows of the result list entries in ascending original-row order.  Output rows
// are independent: counts by one pass, then every block of output rows scatters its own entries
// (threads scan disjoint row ranges of A and keep the entries that fall into their column block
// -- done per block through a column-bucketed index so A is read once per pass).
HostCsr transpose(const HostCsr& A) {
    HostCsr T;
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    T.rowptr.assign(size_t(A.ncols) + 1, 0);
    const int nt = std::max(1, num_threads());
    // pass 1: per-thread column counts over contiguous row ranges of A
    const int64_t nchunk = nt;
    std::vector<std::vector<int32_t>> cnt(nchunk);
    auto range = [&](int64_t c, int32_t& r0, int32_t& r1) {
        r0 = int32_t(int64_t(A.nrows) * c / nchunk);
        r1 = int32_t(int64_t(A.nrows) * (c + 1) / nchunk);
    };
    parallel_for(nchunk, [&](int64_t c) {
        int32_t r0, r1;
        range(c, r0, r1);
        auto& v = cnt[c];
        v.assign(size_t(A.ncols), 0);
        for (int64_t k = A.rowptr[r0]; k < A.rowptr[r1]; ++k) v[A.col[k]]++;
    });
    // offsets: column j's entries of chunk c start at rowptr[j] + sum_{c' < c} cnt[c'][j]
    for (int32_t j = 0; j < A.ncols; ++j) {
        int64_t tot = 0;
        for (int64_t c = 0; c < nchunk; ++c) {
            int32_t t = cnt[c][j];
            cnt[c][j] = int32_t(tot);
            tot += t;
        }
        T.rowptr[j + 1] = T.rowptr[j] + tot;
    }
    T.col.resize(A.nnz());
    T.val.resize(A.nnz());
    // pass 2: every chunk scatters its rows (ascending) into its own slots: ascending original rows
    parallel_for(nchunk, [&](int64_t c) {
        int32_t r0, r1;
        range(c, r0, r1);
        auto& pos = cnt[c];
        for (int32_t i = r0; i < r1; ++i)
            for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
                const int32_t j = A.col[k];
                const int64_t o = T.rowptr[j] + pos[j]++;
                T.col[o] = i;
                T.val[o] = A.val[k];
            }
    });
    return T;
}

}  // namespace iga
