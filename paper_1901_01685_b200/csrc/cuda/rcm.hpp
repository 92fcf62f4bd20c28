#pragma once
#include <cstdint>
#include <vector>

namespace pmg_host {
std::vector<int32_t> rcm_ordering(int32_t n, const int32_t* rowptr, const int32_t* col);
int32_t permute_symmetric(int32_t n, const int32_t* rowptr, const int32_t* col, const double* val,
                          const std::vector<int32_t>& perm, std::vector<int32_t>& brp, std::vector<int32_t>& bci,
                          std::vector<double>& bv);
int32_t bandwidth(int32_t n, const int32_t* rowptr, const int32_t* col);
}  // namespace pmg_host
