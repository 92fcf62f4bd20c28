// C++ API (include/iga/pmg.hpp) over the C ABI of libpmg_cuda.so: status codes are mapped
// to the reference's exception types (types.hpp:23-42); no arithmetic happens here.
#include "iga/pmg.hpp"

#include <mutex>

namespace iga {

namespace {

[[noreturn]] void fail(int st, const char* what, int64_t row = -1) {
    std::string msg = std::string(what) + ": " + pmg_status_string(st) + " -- " + pmg_last_error();
    switch (st) {
        case PMG_ZERO_PIVOT: throw FactorizationError(msg, row);
        case PMG_ZERO_DIAG: throw SmootherError(msg, row);
        case PMG_ERR_DIM: throw DimensionError(msg);
        case PMG_ERR_ARG: throw std::invalid_argument(msg);
        default: throw DeviceError(msg, st);
    }
}
inline void check(int st, const char* what, int64_t row = -1) {
    if (st != PMG_OK) fail(st, what, row);
}

std::shared_ptr<pmg_csr_s> device_csr(const CsrMatrix& A) {
    pmg_csr h = nullptr;
    pmg_csr_view v = A.view();
    check(pmg_csr_create(&v, &h), "csr_create");
    return std::shared_ptr<pmg_csr_s>(h, [](pmg_csr p) { pmg_csr_destroy(p); });
}

void need(size_t got, size_t want, const char* what) {
    if (got != want) throw DimensionError(std::string(what) + ": dimension mismatch");
}

}  // namespace

Vector spmv(const CsrMatrix& A, const Vector& x) {
    need(x.size(), size_t(A.ncols), "spmv");
    auto d = device_csr(A);
    Vector y(A.nrows);
    check(pmg_spmv(d.get(), x.data(), y.data()), "spmv");
    return y;
}

void gauss_seidel_sweep(const CsrMatrix& A, Vector& u, const Vector& f) {
    if (A.nrows != A.ncols) throw DimensionError("gauss_seidel_sweep: matrix not square");
    need(u.size(), size_t(A.nrows), "gauss_seidel_sweep");
    need(f.size(), size_t(A.nrows), "gauss_seidel_sweep");
    auto d = device_csr(A);
    int64_t row = -1;
    int st = pmg_gs_sweep(d.get(), u.data(), f.data(), &row);
    if (st != PMG_OK) fail(st, "gauss_seidel_sweep", row);
}

std::vector<int32_t> rcm_ordering(const CsrMatrix& A) {
    std::vector<int32_t> p(A.nrows);
    pmg_csr_view v = A.view();
    check(pmg_rcm_ordering(&v, p.data()), "rcm_ordering");
    return p;
}

IlutFactorization ilut_factorize(const CsrMatrix& A, double tau, double fillfactor, Ordering ordering) {
    if (A.nrows != A.ncols) throw DimensionError("ilut_factorize: matrix not square");
    IlutFactorization F;
    F.A_ = device_csr(A);
    pmg_factor h = nullptr;
    int64_t row = -1;
    int st = pmg_ilut_factorize(F.A_.get(), tau, fillfactor, int(ordering), &h, &row);
    if (st != PMG_OK) fail(st, "ilut_factorize", row);
    F.h_ = std::shared_ptr<pmg_factor_s>(h, [](pmg_factor p) { pmg_factor_destroy(p); });
    F.n_ = A.nrows;
    F.tau = tau;
    F.fillfactor = fillfactor;
    return F;
}

IlutFactorization::Stats IlutFactorization::stats() const {
    Stats s{};
    pmg_factor_stats(h_.get(), &s.nnz_L, &s.nnz_U, &s.levels_L, &s.levels_U, &s.max_row_L, &s.max_row_U);
    return s;
}

CsrMatrix IlutFactorization::L() const {
    Stats s = stats();
    CsrMatrix M;
    M.nrows = M.ncols = n_;
    M.row_offsets.resize(n_ + 1);
    M.col_indices.resize(s.nnz_L);
    M.values.resize(s.nnz_L);
    check(pmg_factor_export(h_.get(), M.row_offsets.data(), M.col_indices.data(), M.values.data(), nullptr, nullptr,
                            nullptr, nullptr),
          "factor_export");
    return M;
}

CsrMatrix IlutFactorization::U() const {
    Stats s = stats();
    CsrMatrix M;
    M.nrows = M.ncols = n_;
    M.row_offsets.resize(n_ + 1);
    M.col_indices.resize(s.nnz_U);
    M.values.resize(s.nnz_U);
    check(pmg_factor_export(h_.get(), nullptr, nullptr, nullptr, M.row_offsets.data(), M.col_indices.data(),
                            M.values.data(), nullptr),
          "factor_export");
    return M;
}

std::vector<int32_t> IlutFactorization::perm() const {
    std::vector<int32_t> p(n_);
    check(pmg_factor_export(h_.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, p.data()), "factor_export");
    return p;
}

std::vector<int32_t> IlutFactorization::perm_inverse() const {
    auto p = perm();
    std::vector<int32_t> q(n_);
    for (int32_t i = 0; i < n_; ++i) q[p[i]] = i;
    return q;
}

Vector ilut_apply(const IlutFactorization& fac, const Vector& r) {
    need(r.size(), size_t(fac.size()), "ilut_apply");
    Vector e(r.size());
    check(pmg_ilut_apply(fac.handle(), r.data(), e.data()), "ilut_apply");
    return e;
}

// ------------------------------------------------------------------ pmg
namespace {
struct WorkPool {  // one pmg_work per hierarchy (calls on a hierarchy are serialised here)
    std::mutex m;
    pmg_work w = nullptr;
};
}  // namespace

PmgHierarchy build_hierarchy(const HierarchyInputs& in, Smoother smoother, int nu1, int nu2, double tau,
                             double fillfactor, Ordering ordering) {
    const int np = int(in.plevels.size()), nh = int(in.hlevels.size());
    std::vector<int> degrees(np);
    std::vector<pmg_csr_view> A(np), P(std::max(np - 1, 1)), PT(std::max(np - 1, 1));
    std::vector<const double*> ML(np);
    for (int l = 0; l < np; ++l) {
        degrees[l] = in.plevels[l].degree;
        A[l] = in.plevels[l].A.view();
        ML[l] = in.plevels[l].lumped_mass.data();
        if (l + 1 < np) {
            P[l] = in.plevels[l].P.view();
            PT[l] = in.plevels[l].PT.view();
        }
    }
    std::vector<pmg_csr_view> HA(nh), HP(std::max(nh - 1, 1)), HPT(std::max(nh - 1, 1));
    for (int j = 0; j < nh; ++j) {
        HA[j] = j == 0 ? A[np - 1] : in.hlevels[j].A.view();
        if (j + 1 < nh) {
            HP[j] = in.hlevels[j].P.view();
            HPT[j] = in.hlevels[j].PT.view();
        }
    }
    pmg_hier_desc d{np,       degrees.data(), A.data(),  ML.data(), P.data(), PT.data(),      nh,    HA.data(),
                    HP.data(), HPT.data(),     int(smoother), nu1, nu2, tau, fillfactor, int(ordering)};
    pmg_hier h = nullptr;
    int lvl = -1;
    int64_t row = -1;
    int st = pmg_hier_create(&d, &h, &lvl, &row);
    if (st != PMG_OK) fail(st, "build_hierarchy", row);
    PmgHierarchy H;
    H.h_ = std::shared_ptr<pmg_hier_s>(h, [](pmg_hier p) { pmg_hier_destroy(p); });
    H.n_ = in.plevels[0].A.nrows;
    for (auto& l : in.plevels) H.sizes_.push_back(l.A.nrows);
    return H;
}

// ------------------------------------------------------------------ problem assembly (host)
namespace {
[[noreturn]] void host_fail(const char* what) {
    throw std::runtime_error(std::string(what) + ": " + iga_last_error());
}
CsrMatrix host_csr(const iga_problem* h, int kind, int l) {
    CsrMatrix M;
    int64_t nnz = 0;
    if (iga_problem_csr_shape(h, kind, l, &M.nrows, &M.ncols, &nnz)) host_fail("assemble");
    M.row_offsets.resize(size_t(M.nrows) + 1);
    M.col_indices.resize(size_t(nnz));
    M.values.resize(size_t(nnz));
    if (iga_problem_csr_copy(h, kind, l, M.row_offsets.data(), M.col_indices.data(), M.values.data()))
        host_fail("assemble");
    return M;
}
Vector host_vec(const iga_problem* h, int kind, int l) {
    Vector v(size_t(iga_problem_vec_len(h, kind, l)));
    if (iga_problem_vec_copy(h, kind, l, v.data())) host_fail("assemble");
    return v;
}
}  // namespace

ProblemSpec config_spec(int config, int degree) {
    ProblemSpec s{};
    if (iga_config_spec(config, degree, &s)) host_fail("config_spec");
    return s;
}

Problem assemble(const ProblemSpec& spec, Assembly assembly) {
    iga_problem* h = nullptr;
    if (iga_problem_build_with(&spec, assembly == Assembly::gpu ? &pmg_asm_values : nullptr, &h)) host_fail("assemble");
    std::unique_ptr<iga_problem, void (*)(iga_problem*)> guard(h, iga_problem_free);
    Problem pb;
    const int np = iga_problem_num_plevels(h), nh = iga_problem_num_hlevels(h);
    for (int l = 0; l < np; ++l) {
        PLevelInput L;
        L.degree = iga_problem_degree(h, l);
        L.A = host_csr(h, IGA_MAT_A, l);
        L.lumped_mass = host_vec(h, IGA_VEC_ML, l);
        if (l + 1 < np) {
            L.P = host_csr(h, IGA_MAT_P, l);
            L.PT = host_csr(h, IGA_MAT_PT, l);
        }
        pb.inputs.plevels.push_back(std::move(L));
    }
    for (int j = 0; j < nh; ++j) {
        HLevelInput L;
        if (j > 0) L.A = host_csr(h, IGA_MAT_HA, j);
        if (j + 1 < nh) {
            L.P = host_csr(h, IGA_MAT_HP, j);
            L.PT = host_csr(h, IGA_MAT_HPT, j);
        }
        pb.inputs.hlevels.push_back(std::move(L));
    }
    pb.f = host_vec(h, IGA_VEC_F, 0);
    pb.u0 = host_vec(h, IGA_VEC_U0, 0);
    return pb;
}

PmgHierarchy build_hierarchy(const ProblemSpec& spec, Smoother smoother, int nu1, int nu2, double tau,
                             double fillfactor, Ordering ordering, Assembly assembly) {
    return build_hierarchy(assemble(spec, assembly).inputs, smoother, nu1, nu2, tau, fillfactor, ordering);
}

double PmgHierarchy::setup_seconds() const {
    pmg_hier_stats s{};
    pmg_hier_get_stats(h_.get(), &s);
    return s.setup_seconds;
}

namespace {
std::shared_ptr<pmg_work_s> make_work(const PmgHierarchy& H) {
    pmg_work w = nullptr;
    check(pmg_work_create(H.handle(), &w), "work_create");
    return std::shared_ptr<pmg_work_s>(w, [](pmg_work p) { pmg_work_destroy(p); });
}
}  // namespace

Vector prolongate(const PmgHierarchy& H, int level, const Vector& v) {
    if (level < 0 || level + 1 >= int(H.sizes_.size())) throw std::invalid_argument("prolongate: bad level");
    need(v.size(), size_t(H.sizes_[level + 1]), "prolongate");
    Vector out(H.sizes_[level]);
    check(pmg_prolongate(H.handle(), level, v.data(), out.data()), "prolongate");
    return out;
}

Vector restrict(const PmgHierarchy& H, int level, const Vector& r) {
    if (level < 0 || level + 1 >= int(H.sizes_.size())) throw std::invalid_argument("restrict: bad level");
    need(r.size(), size_t(H.sizes_[level]), "restrict");
    Vector out(H.sizes_[level + 1]);
    check(pmg_restrict(H.handle(), level, r.data(), out.data()), "restrict");
    return out;
}

void cycle(const PmgHierarchy& H, int level, Vector& u, const Vector& f) {
    if (level < 0 || level >= int(H.sizes_.size())) throw std::invalid_argument("cycle: bad level");
    need(u.size(), size_t(H.sizes_[level]), "cycle");
    need(f.size(), size_t(H.sizes_[level]), "cycle");
    auto w = make_work(H);  // each call owns its vectors
    check(pmg_cycle(w.get(), level, u.data(), f.data()), "cycle");
}

std::pair<Vector, SolveReport> solve(const PmgHierarchy& H, const Vector& f, double tol, int max_cycles,
                                     const Vector* guess) {
    need(f.size(), size_t(H.n_), "solve");
    Vector u = guess ? *guess : Vector(H.n_, 0.0);
    need(u.size(), size_t(H.n_), "solve");
    auto w = make_work(H);
    SolveReport rep;
    std::vector<double> hist(size_t(max_cycles) + 1);
    int cycles = 0, flags = 0;
    double secs = 0;
    check(pmg_solve(w.get(), f.data(), u.data(), tol, max_cycles, hist.data(), &cycles, &flags, &secs), "solve");
    rep.cycles = cycles;
    rep.residual_history.assign(hist.begin(), hist.begin() + cycles + 1);
    rep.converged = flags & PMG_FLAG_CONVERGED;
    rep.diverged = flags & PMG_FLAG_DIVERGED;
    rep.setup_seconds = H.setup_seconds();
    rep.solve_seconds = secs;
    return {std::move(u), std::move(rep)};
}

std::pair<Vector, KrylovReport> bicgstab(const PmgHierarchy& H, const Vector& f, double tol, int max_iter,
                                         const Vector* guess) {
    need(f.size(), size_t(H.n_), "bicgstab");
    Vector u = guess ? *guess : Vector(H.n_, 0.0);
    need(u.size(), size_t(H.n_), "bicgstab");
    auto w = make_work(H);
    KrylovReport rep;
    std::vector<double> hist(size_t(max_iter) + 1);
    int iters = 0, flags = 0;
    double secs = 0;
    check(pmg_bicgstab(w.get(), f.data(), u.data(), tol, max_iter, hist.data(), &iters, &flags, &secs), "bicgstab");
    rep.iterations = iters;
    rep.residual_history.assign(hist.begin(), hist.begin() + iters + 1);
    rep.converged = flags & PMG_FLAG_CONVERGED;
    rep.diverged = flags & PMG_FLAG_DIVERGED;
    rep.breakdown = flags & PMG_FLAG_BREAKDOWN;
    rep.solve_seconds = secs;
    return {std::move(u), std::move(rep)};
}

}  // namespace iga
