// Reverse Cuthill-McKee ordering and symmetric permutation (host setup for ILUT).
//
// rcm_ordering: symmetrised pattern without the diagonal;
// every component starts at the unvisited node of minimum (degree, index); the BFS
// appends each node's unvisited neighbours in ascending (degree, index); the concatenated
// Cuthill-McKee sequence is reversed.  perm[new] = old.
#include "rcm.hpp"

#include <algorithm>
#include <numeric>

namespace pmg_host {

std::vector<int32_t> rcm_ordering(int32_t n, const int32_t* rowptr, const int32_t* col) {
    // symmetrised adjacency in CSR form: count, fill, sort + unique per row
    std::vector<int64_t> cnt(size_t(n) + 1, 0);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (col[k] != i) {
                cnt[i + 1]++;
                cnt[col[k] + 1]++;
            }
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    std::vector<int32_t> adj(cnt[n]);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (col[k] != i) {
                adj[fill[i]++] = col[k];
                adj[fill[col[k]]++] = i;
            }
    std::vector<int32_t> deg(n), beg(n), end(n);
    for (int32_t i = 0; i < n; ++i) {
        auto b = adj.begin() + cnt[i], e = adj.begin() + cnt[i + 1];
        std::sort(b, e);
        e = std::unique(b, e);
        beg[i] = int32_t(cnt[i]);
        end[i] = int32_t(e - adj.begin());
        deg[i] = end[i] - beg[i];
    }
    // (degree, index) key: a strict total order
    auto key = [&](int32_t v) { return (int64_t(deg[v]) << 32) | uint32_t(v); };
    std::vector<int32_t> starts(n);
    std::iota(starts.begin(), starts.end(), 0);
    std::sort(starts.begin(), starts.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });

    std::vector<uint8_t> seen(n, 0);
    std::vector<int32_t> q;
    q.reserve(n);
    std::vector<int32_t> nb;
    size_t s = 0;
    while (q.size() < size_t(n)) {
        while (seen[starts[s]]) ++s;
        size_t head = q.size();
        q.push_back(starts[s]);
        seen[starts[s]] = 1;
        for (; head < q.size(); ++head) {
            const int32_t x = q[head];
            nb.clear();
            for (int32_t k = beg[x]; k < end[x]; ++k)
                if (!seen[adj[k]]) nb.push_back(adj[k]);
            std::sort(nb.begin(), nb.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });
            for (int32_t y : nb) {
                seen[y] = 1;
                q.push_back(y);
            }
        }
    }
    return std::vector<int32_t>(q.rbegin(), q.rend());
}

// B = P A P^T with B[i][j] = A[perm[i]][perm[j]], columns sorted; returns the bandwidth
int32_t permute_symmetric(int32_t n, const int32_t* rowptr, const int32_t* col, const double* val,
                          const std::vector<int32_t>& perm, std::vector<int32_t>& brp, std::vector<int32_t>& bci,
                          std::vector<double>& bv) {
    std::vector<int32_t> pinv(n);
    for (int32_t i = 0; i < n; ++i) pinv[perm[i]] = i;
    brp.assign(size_t(n) + 1, 0);
    for (int32_t i = 0; i < n; ++i) brp[i + 1] = brp[i] + (rowptr[perm[i] + 1] - rowptr[perm[i]]);
    bci.resize(brp[n]);
    bv.resize(brp[n]);
    int32_t band = 0;
    std::vector<std::pair<int32_t, double>> row;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t o = perm[i];
        row.clear();
        for (int32_t k = rowptr[o]; k < rowptr[o + 1]; ++k) row.emplace_back(pinv[col[k]], val[k]);
        std::sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
        for (size_t q = 0; q < row.size(); ++q) {
            bci[brp[i] + q] = row[q].first;
            bv[brp[i] + q] = row[q].second;
            band = std::max(band, std::abs(row[q].first - i));
        }
    }
    return band;
}

int32_t bandwidth(int32_t n, const int32_t* rowptr, const int32_t* col) {
    int32_t band = 0;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) band = std::max(band, std::abs(col[k] - i));
    return band;
}

}  // namespace pmg_host
