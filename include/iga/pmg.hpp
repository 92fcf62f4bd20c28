// iga/pmg.hpp -- C++ solver API of the p-multigrid solve path, B200 backend.
//
// Mirrors the reference's C++ conventions (proj/include/iga/types.hpp:11-42: namespace
// iga, Index, Scalar = double, CSR with sorted columns, exceptions derived from
// std::runtime_error, FactorizationError carrying `row`) and the SPEC operations the
// reference would declare for this path.  Eigen is absent from the
// reference tree, so the CSR and vector types are plain std::vector based.
//
// Every call runs on the GPU through the C ABI of include/pmg_cuda.h (libpmg_cuda.so).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../iga_host.h"
#include "../pmg_cuda.h"

namespace iga {

using Index = std::int64_t;  // types.hpp:11 (Eigen::Index)
using Scalar = double;       // types.hpp:12
using Vector = std::vector<Scalar>;

// types.hpp:23-42
struct FactorizationError : std::runtime_error {
    Index row;
    FactorizationError(const std::string& msg, Index r) : std::runtime_error(msg), row(r) {}
};
struct SmootherError : std::runtime_error {
    Index row;
    SmootherError(const std::string& msg, Index r) : std::runtime_error(msg), row(r) {}
};
struct DimensionError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DeviceError : std::runtime_error {
    int status;
    DeviceError(const std::string& msg, int s) : std::runtime_error(msg), status(s) {}
};

// SparseMatrixCsr: strictly increasing columns per row
struct CsrMatrix {
    std::int32_t nrows = 0, ncols = 0;
    std::vector<std::int32_t> row_offsets, col_indices;
    std::vector<Scalar> values;
    pmg_csr_view view() const { return {nrows, ncols, row_offsets.data(), col_indices.data(), values.data()}; }
};

enum class Smoother { ilut = PMG_SMOOTHER_ILUT, gauss_seidel = PMG_SMOOTHER_GS };
enum class Ordering { none = PMG_ORDER_NONE, rcm = PMG_ORDER_RCM };

// IlutFactorization
class IlutFactorization {
   public:
    CsrMatrix L() const;  // strictly lower, unit diagonal implicit
    CsrMatrix U() const;  // upper with diagonal
    std::vector<std::int32_t> perm() const;
    std::vector<std::int32_t> perm_inverse() const;
    double tau = 0, fillfactor = 1;
    struct Stats {
        std::int64_t nnz_L, nnz_U;
        std::int32_t levels_L, levels_U, max_row_L, max_row_U;
    };
    Stats stats() const;
    pmg_factor handle() const { return h_.get(); }
    std::int32_t size() const { return n_; }

   private:
    friend IlutFactorization ilut_factorize(const CsrMatrix&, double, double, Ordering);
    std::shared_ptr<pmg_factor_s> h_;
    std::shared_ptr<pmg_csr_s> A_;
    std::int32_t n_ = 0;
};

Vector spmv(const CsrMatrix& A, const Vector& x);
void gauss_seidel_sweep(const CsrMatrix& A, Vector& u, const Vector& f);
std::vector<std::int32_t> rcm_ordering(const CsrMatrix& A);
IlutFactorization ilut_factorize(const CsrMatrix& A, double tau = 1e-12, double fillfactor = 1.0,
                                 Ordering ordering = Ordering::rcm);
Vector ilut_apply(const IlutFactorization& fac, const Vector& r);

// inputs of build_hierarchy: the rediscretised operators, lumped masses and transfers of
// every p-level (degree list descending to 1) and the p=1 h-chain
struct PLevelInput {
    int degree;
    CsrMatrix A;
    Vector lumped_mass;
    CsrMatrix P, PT;  // from the next (lower-degree) level; empty on the last level
};
struct HLevelInput {
    CsrMatrix A;      // unused for the finest h-level (= the degree-1 p-level)
    CsrMatrix P, PT;  // from the next coarser h-level; empty on the coarsest
};
struct HierarchyInputs {
    std::vector<PLevelInput> plevels;
    std::vector<HLevelInput> hlevels;
};

struct SolveReport {
    int cycles = 0;
    std::vector<double> residual_history;
    bool converged = false, diverged = false;
    double setup_seconds = 0, solve_seconds = 0;
};

struct KrylovReport {
    int iterations = 0;
    std::vector<double> residual_history;  // [0] = 1
    bool converged = false, diverged = false, breakdown = false;
    double solve_seconds = 0;
};

class PmgHierarchy {  // SPEC.md:313-316, immutable after construction
   public:
    pmg_hier handle() const { return h_.get(); }
    double setup_seconds() const;

   private:
    friend PmgHierarchy build_hierarchy(const HierarchyInputs&, Smoother, int, int, double, double, Ordering);
    std::shared_ptr<pmg_hier_s> h_;
    std::int32_t n_ = 0;
    std::vector<std::int32_t> sizes_;
    friend Vector prolongate(const PmgHierarchy&, int, const Vector&);
    friend Vector restrict(const PmgHierarchy&, int, const Vector&);
    friend void cycle(const PmgHierarchy&, int, Vector&, const Vector&);
    friend std::pair<Vector, SolveReport> solve(const PmgHierarchy&, const Vector&, double, int, const Vector*);
    friend std::pair<Vector, KrylovReport> bicgstab(const PmgHierarchy&, const Vector&, double, int, const Vector*);
};

PmgHierarchy build_hierarchy(const HierarchyInputs& in, Smoother smoother = Smoother::ilut, int nu1 = 1, int nu2 = 1,
                             double tau = 1e-12, double fillfactor = 1.0,
                             Ordering ordering = Ordering::none);

// The problem side of SPEC.md:327's build_hierarchy(spec, p, h, ...): the benchmark / geometry,
// coefficients, degree list and h of iga_problem_spec (include/iga_host.h).  Numbering, sparsity
// patterns and the load vector come from libiga_host.so; the matrix values of A_k, M_k, P^k_j
// (assemble_system / assemble_mass / assemble_transfer) from the host element loop
// or from the GPU assembler (pmg_asm_values) -- bit-identical either way.
using ProblemSpec = iga_problem_spec;
enum class Assembly { host, gpu };
struct Problem {
    HierarchyInputs inputs;
    Vector f, u0;  // load vector and initial guess
};
ProblemSpec config_spec(int config, int degree = 0);  // BASELINE.json config 1..5 (degree: config 2's p)
Problem assemble(const ProblemSpec& spec, Assembly assembly = Assembly::host);
// assemble + build_hierarchy in one call (build_hierarchy(spec, p, h, smoother, nu1, nu2))
PmgHierarchy build_hierarchy(const ProblemSpec& spec, Smoother smoother = Smoother::ilut, int nu1 = 1, int nu2 = 1,
                             double tau = 1e-12, double fillfactor = 1.0, Ordering ordering = Ordering::none,
                             Assembly assembly = Assembly::host);
Vector prolongate(const PmgHierarchy& H, int level, const Vector& v_coarse);
Vector restrict(const PmgHierarchy& H, int level, const Vector& r_fine);
// (`restrict` is a C99 keyword, not a C++ one; the former spelling stays as an alias)
inline Vector restrict_(const PmgHierarchy& H, int level, const Vector& r_fine) { return restrict(H, level, r_fine); }
void cycle(const PmgHierarchy& H, int level, Vector& u, const Vector& f);
// SPEC.md:363-371; guess == nullptr -> zero initial guess
std::pair<Vector, SolveReport> solve(const PmgHierarchy& H, const Vector& f, double tol = 1e-8, int max_cycles = 200,
                                     const Vector* guess = nullptr);
// SPEC.md:269-277 with as_preconditioner(H): BiCGSTAB, one V-cycle from zero
// per preconditioning phase; guess == nullptr -> zero initial guess
std::pair<Vector, KrylovReport> bicgstab(const PmgHierarchy& H, const Vector& f, double tol = 1e-8, int max_iter = 200,
                                         const Vector* guess = nullptr);

}  // namespace iga
