// Host-side input generation for the p-multigrid solve path: B-spline bases,
// NURBS geometry, Galerkin/Nitsche assembly of the CDR operator, mass, transfer
// and h-refinement operators.  This is SETUP code (discretization
// stays on the host); the solve phase runs in libpmg_cuda.so.
//
// Behaviour follows the reference spec:
//   splines        SPEC.md:20-108, proj/src/splines.cpp:9-125 (span search with a
//                  right-closed last span, Cox-de Boor values, first derivatives)
//   discretization SPEC.md:110-198 (CDR bilinear form, (p+1)^2 Gauss points,
//                  symmetric Nitsche with eta = 4 k^2 / h, mass, transfer, lumping)
//   multipatch     SPEC.md:44-49, SPEC.md:99 (L-shape as 3 conforming patches,
//                  DOF identification; patch-major numbering)
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "../../../include/pmg_asm.h"

namespace iga {

// ---- errors (conventions of proj/include/iga/types.hpp:23-42) ----
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct AssemblyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };

// allocator whose resize() leaves new elements uninitialised: the big CSR arrays are written in
// full by parallel loops (or by the external producer of the values), so a serial zero fill --
// and with it the first touch of every page by one thread -- would only cost time
template <class T>
struct NoInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        if constexpr (sizeof...(Args) == 0) ::new (static_cast<void*>(p)) U;
        else ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};

// ---- host CSR (int32 offsets/columns, fp64 values) ----
struct HostCsr {
    int32_t nrows = 0, ncols = 0;
    std::vector<int64_t> rowptr;  // nrows+1 (int64 on the host; device uses int32 where it fits)
    std::vector<int32_t, NoInitAlloc<int32_t>> col;
    std::vector<double, NoInitAlloc<double>> val;  // make_pattern leaves it uninitialised
    int64_t nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

// ---- splines (splines.hpp:10-54) ----
struct Knots {
    int p = 0;
    std::vector<double> t;
    static Knots open_uniform(int p, int spans);
    int nbasis() const { return int(t.size()) - p - 1; }
    int nspans() const { return nbasis() - p; }
};
int knot_span(const Knots& kv, double x);                       // right-closed last span
int basis_values(const Knots& kv, double x, double* N);        // returns first active index
int basis_values_d1(const Knots& kv, double x, double* N, double* dN);

// ---- geometry: rational tensor patch on [0,1]^2 ----
struct NurbsPatch {
    Knots gx, gy;                    // geometry bases (independent of solution degree)
    std::vector<double> cx, cy, w;   // control net, x fastest: index a + b*nx
    void map(double xi, double eta, double X[2], double J[2][2]) const;  // J[r][c] = dX_r/dxi_c
    static NurbsPatch affine(double x0, double y0, double sx, double sy);
    static NurbsPatch quarter_annulus(double r_in, double r_out);  // xi radial, eta angular
};

// ---- problem coefficients ----
struct Cdr {
    double D[2][2] = {{1, 0}, {0, 1}};
    double v[2] = {0, 0};
    double R = 0;
    double nitsche_scale = 1.0;
    std::function<double(double, double)> f;
    std::function<double(double, double)> g;  // Dirichlet data (null: homogeneous)
};

// edge ids: 0 eta=0 (iy=0), 1 xi=1 (ix=n-1), 2 eta=1 (iy=n-1), 3 xi=0 (ix=0)
struct Interface { int pa, ea, pb, eb; };  // edge ea of patch pa == edge eb of pb, same direction

struct Domain {
    std::vector<NurbsPatch> patches;
    std::vector<Interface> glue;     // conforming interfaces (pb < pa: pa's DOFs take pb's index)
    // Optional global DOF numbering for multipatch domains whose patches tile a grid of unit
    // squares: patch P sits at grid cell grid_off[P] = {cx, cy}; DOFs are then numbered
    // row-major over the whole domain (y, then x ascending) instead of patch-major.
    std::vector<std::array<int, 2>> grid_off;
    bool rowmajor = false;
    bool is_interface(int patch, int edge) const;
};

// spline space of degree p with nel elements per direction on every patch
struct Space {
    int p = 1, nel = 1;
    int nloc = 0;                            // (nel+p)^2 local DOFs per patch
    std::vector<std::vector<int32_t>> l2g;   // per patch local -> global
    int32_t ndof = 0;
    static Space build(const Domain& dom, int p, int nel);
};

// Assembly.  All routines are deterministic and independent of
// the number of worker threads (element strips coloured so no two concurrent strips
// touch the same row; colour-major accumulation order).
//
// `values` (optional, F2): an external producer of the matrix values -- the GPU assembler
// pmg_asm_values of libpmg_cuda.so (include/pmg_asm.h).  The host then builds only the integer
// structure, the 1D tables and the load vector; the values must equal the host loop's bit for bit.
HostCsr assemble_operator(const Domain& dom, const Space& sp, const Cdr& c, std::vector<double>* rhs,
                          pmg_asm_values_fn values = nullptr);
HostCsr assemble_mass(const Domain& dom, const Space& sp, pmg_asm_values_fn values = nullptr);
// row sums of M; `pattern` (optional, external values only): an operator on the same space, whose
// sparsity pattern M shares
std::vector<double> lumped_mass(const Domain& dom, const Space& sp, pmg_asm_values_fn values = nullptr,
                                const HostCsr* pattern = nullptr);
std::vector<double> lump(const HostCsr& M);                            // row sums of an assembled M
HostCsr assemble_transfer(const Domain& dom, const Space& fine_p, const Space& coarse_p,
                          pmg_asm_values_fn values = nullptr);  // P^k_j
HostCsr hrefine_p1(const Domain& dom, const Space& fine, const Space& coarse);  // knot insertion, p=1
HostCsr transpose(const HostCsr& A);

// Gauss-Legendre on [0,1]
void gauss01(int n, double* x, double* w);

int num_threads();
void set_num_threads(int n);

}  // namespace iga
