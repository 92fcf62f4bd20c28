// Drives the C++ solver API (include/iga/pmg.hpp, libiga_pmg.so) end to end on BASELINE config 1:
// assemble + build_hierarchy(spec, ...), solve, ilut_factorize / ilut_apply, bicgstab, restrict /
// prolongate, and the FactorizationError path.  Writes the results as raw float64 files into
// argv[1] for tests/test_cpp_api.py, which compares them with the CPU oracle bit for bit.
#include <cstdio>
#include <cstring>
#include <string>

#include "iga/pmg.hpp"

static void dump(const std::string& path, const std::vector<double>& v) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f || std::fwrite(v.data(), sizeof(double), v.size(), f) != v.size()) std::exit(3);
    std::fclose(f);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string out = argv[1];
    const iga::ProblemSpec spec = iga::config_spec(1);
    const iga::Problem pb = iga::assemble(spec);
    const iga::PmgHierarchy H = iga::build_hierarchy(spec, iga::Smoother::ilut);

    auto [u, rep] = iga::solve(H, pb.f, 1e-8, 200, &pb.u0);
    dump(out + "/solve_u.bin", u);
    dump(out + "/solve_hist.bin", rep.residual_history);

    const iga::CsrMatrix& A = pb.inputs.plevels[0].A;
    const iga::IlutFactorization F = iga::ilut_factorize(A, 1e-12, 1.0, iga::Ordering::none);
    dump(out + "/ilut_apply.bin", iga::ilut_apply(F, pb.f));

    auto [ub, kr] = iga::bicgstab(H, pb.f, 1e-8, 200, &pb.u0);
    dump(out + "/bicgstab_u.bin", ub);
    dump(out + "/bicgstab_hist.bin", kr.residual_history);

    const iga::Vector rc = iga::restrict(H, 0, pb.f);
    dump(out + "/restrict.bin", rc);
    dump(out + "/prolongate.bin", iga::prolongate(H, 0, rc));

    // a zero pivot raises FactorizationError carrying the row
    iga::CsrMatrix Z;
    Z.nrows = Z.ncols = 2;
    Z.row_offsets = {0, 2, 3};
    Z.col_indices = {0, 1, 0};
    Z.values = {0.0, 1.0, 1.0};
    long long zrow = -2;
    try {
        (void)iga::ilut_factorize(Z, 0.0, 1.0, iga::Ordering::none);
    } catch (const iga::FactorizationError& e) {
        zrow = e.row;
    }
    std::printf("{\"cycles\": %d, \"converged\": %d, \"bicgstab_iterations\": %d, \"zero_pivot_row\": %lld}\n",
                rep.cycles, int(rep.converged), kr.iterations, zrow);
    return 0;
}
