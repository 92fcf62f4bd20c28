// MatrixMarket import / export ("Matrix export: MatrixMarket coordinate format for
// A, M_k, P^k_{k-1}", "MatrixMarket import/export for matrices; vectors as
// one-column MatrixMarket or plain text, one value per line").
//
// Reading accepts `matrix coordinate {real|integer|pattern} {general|symmetric|skew-symmetric}`
// (symmetric parts are mirrored, pattern entries are 1.0) and returns sorted CSR with duplicate
// entries summed in file order.  Writing emits `coordinate real general`, 1-based, row-major, with
// %.17g values, so every double survives a round trip bit for bit.  Vectors: `array real
// general` with one column, or plain text with one value per line.
// Exposed through the C ABI in include/iga_host.h.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/iga_host.h"

namespace {

struct Triplets {
    int32_t nrows = 0, ncols = 0;
    std::vector<int64_t> key;  // row * ncols + col, in file order (after mirroring)
    std::vector<double> val;
};

std::string lower(std::string s) {
    for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// CSR of the triplets: sorted by (row, col); duplicates summed in file order
struct Csr {
    int32_t nrows = 0, ncols = 0;
    std::vector<int32_t> rowptr, col;
    std::vector<double> val;
};

Csr to_csr(const Triplets& t) {
    std::vector<int64_t> order(t.key.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = int64_t(i);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return t.key[a] < t.key[b]; });
    Csr c;
    c.nrows = t.nrows;
    c.ncols = t.ncols;
    c.rowptr.assign(size_t(t.nrows) + 1, 0);
    for (size_t q = 0; q < order.size();) {
        const int64_t k = t.key[order[q]];
        double s = t.val[order[q]];
        size_t r = q + 1;
        for (; r < order.size() && t.key[order[r]] == k; ++r) s = s + t.val[order[r]];
        const int32_t i = int32_t(k / t.ncols), j = int32_t(k % t.ncols);
        c.col.push_back(j);
        c.val.push_back(s);
        ++c.rowptr[size_t(i) + 1];
        q = r;
    }
    for (int32_t i = 0; i < t.nrows; ++i) c.rowptr[size_t(i) + 1] += c.rowptr[size_t(i)];
    return c;
}

// C stdio only: this library is loaded into processes that may already hold another
// libstdc++ (e.g. next to torch), whose iostreams must not be mixed with ours
struct File {
    FILE* fp = nullptr;
    explicit File(const std::string& path, const char* mode) : fp(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (fp) std::fclose(fp);
    }
};

bool next_line(FILE* fp, std::string& line) {
    line.clear();
    int ch;
    while ((ch = std::fgetc(fp)) != EOF && ch != '\n') line.push_back(char(ch));
    return ch != EOF || !line.empty();
}

std::vector<std::string> words(const std::string& line) {
    std::vector<std::string> w;
    size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        size_t j = i;
        while (j < line.size() && !std::isspace(static_cast<unsigned char>(line[j]))) ++j;
        if (j > i) w.push_back(lower(line.substr(i, j - i)));
        i = j;
    }
    return w;
}

// the first non-comment, non-empty line after the banner
std::string size_line(FILE* fp) {
    std::string line;
    while (next_line(fp, line))
        if (!line.empty() && line[0] != '%') return line;
    return std::string();
}

Triplets read_coordinate(const std::string& path) {
    File f(path, "r");
    if (!f.fp) throw std::runtime_error("cannot open " + path + ": " + std::strerror(errno));
    std::string line;
    if (!next_line(f.fp, line)) throw std::runtime_error(path + ": empty file");
    const std::vector<std::string> h = words(line);
    if (h.size() < 5 || h[0] != "%%matrixmarket" || h[1] != "matrix" || h[2] != "coordinate")
        throw std::runtime_error(path + ": not a MatrixMarket coordinate matrix (header: " + line + ")");
    const std::string& field = h[3];
    const std::string& symmetry = h[4];
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer" && field != "double")
        throw std::runtime_error(path + ": unsupported field '" + field + "'");
    const bool sym = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
    if (!sym && !skew && symmetry != "general")
        throw std::runtime_error(path + ": unsupported symmetry '" + symmetry + "'");
    line = size_line(f.fp);
    Triplets t;
    long long nnz = 0, m = 0, n = 0;
    if (std::sscanf(line.c_str(), "%lld %lld %lld", &m, &n, &nnz) != 3 || m < 0 || n < 0 || nnz < 0 ||
        m > INT32_MAX || n > INT32_MAX)
        throw std::runtime_error(path + ": bad size line '" + line + "'");
    t.nrows = int32_t(m);
    t.ncols = int32_t(n);
    t.key.reserve(size_t(nnz) * (sym || skew ? 2 : 1));
    t.val.reserve(t.key.capacity());
    for (long long e = 0; e < nnz; ++e) {
        long long i, j;
        double v = 1.0;
        if (std::fscanf(f.fp, "%lld %lld", &i, &j) != 2)
            throw std::runtime_error(path + ": truncated after " + std::to_string(e) + " entries");
        if (!pattern && std::fscanf(f.fp, "%lf", &v) != 1)
            throw std::runtime_error(path + ": missing value of entry " + std::to_string(e));
        if (i < 1 || i > m || j < 1 || j > n) throw std::runtime_error(path + ": entry out of range");
        t.key.push_back((i - 1) * n + (j - 1));
        t.val.push_back(v);
        if ((sym || skew) && i != j) {
            t.key.push_back((j - 1) * n + (i - 1));
            t.val.push_back(skew ? -v : v);
        }
    }
    return t;
}

std::vector<double> read_vector(const std::string& path) {
    File f(path, "r");
    if (!f.fp) throw std::runtime_error("cannot open " + path + ": " + std::strerror(errno));
    std::vector<double> v;
    std::string line;
    if (next_line(f.fp, line) && lower(line).rfind("%%matrixmarket", 0) == 0) {
        const std::vector<std::string> h = words(line);
        if (h.size() < 3 || h[2] != "array") throw std::runtime_error(path + ": vectors must be MatrixMarket arrays");
        line = size_line(f.fp);
        long long m = 0, n = 0;
        if (std::sscanf(line.c_str(), "%lld %lld", &m, &n) != 2 || n != 1 || m < 0)
            throw std::runtime_error(path + ": a vector is an m x 1 array");
        v.resize(size_t(m));
        for (long long i = 0; i < m; ++i)
            if (std::fscanf(f.fp, "%lf", &v[size_t(i)]) != 1) throw std::runtime_error(path + ": truncated vector");
        return v;
    }
    std::rewind(f.fp);  // plain text, one value per line
    double x;
    int r;
    while ((r = std::fscanf(f.fp, "%lf", &x)) == 1) v.push_back(x);
    if (r != EOF) throw std::runtime_error(path + ": not a number in the vector file");
    return v;
}

std::string g_mm_err;
// the last matrix read (shape query, then copy), per thread
std::string g_cache_path;
Csr g_cache;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_mm_err = e.what();
        return -1;
    }
}

const Csr& cached(const char* path) {
    if (g_cache_path != path) {
        g_cache = to_csr(read_coordinate(path));
        g_cache_path = path;
    }
    return g_cache;
}

}  // namespace

extern "C" {

const char* iga_mm_last_error(void) { return g_mm_err.c_str(); }

int iga_mm_read_shape(const char* path, int32_t* nrows, int32_t* ncols, int64_t* nnz) {
    return guarded([&] {
        g_cache_path.clear();  // re-read: the file may have changed
        const Csr& c = cached(path);
        *nrows = c.nrows;
        *ncols = c.ncols;
        *nnz = int64_t(c.col.size());
    });
}

int iga_mm_read(const char* path, int32_t* rowptr, int32_t* col, double* val) {
    return guarded([&] {
        const Csr& c = cached(path);
        std::copy(c.rowptr.begin(), c.rowptr.end(), rowptr);
        std::copy(c.col.begin(), c.col.end(), col);
        std::copy(c.val.begin(), c.val.end(), val);
    });
}

int iga_mm_write(const char* path, int32_t nrows, int32_t ncols, const int32_t* rowptr, const int32_t* col,
                 const double* val, const char* comment) {
    return guarded([&] {
        FILE* fp = std::fopen(path, "w");
        if (!fp) throw std::runtime_error(std::string("cannot write ") + path + ": " + std::strerror(errno));
        std::fprintf(fp, "%%%%MatrixMarket matrix coordinate real general\n");
        if (comment && *comment) std::fprintf(fp, "%% %s\n", comment);
        std::fprintf(fp, "%d %d %d\n", nrows, ncols, rowptr[nrows]);
        for (int32_t i = 0; i < nrows; ++i)
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) std::fprintf(fp, "%d %d %.17g\n", i + 1, col[k] + 1, val[k]);
        if (std::fclose(fp) != 0) throw std::runtime_error(std::string("write failed: ") + path);
    });
}

int iga_mm_write_vector(const char* path, int32_t n, const double* v) {
    return guarded([&] {
        FILE* fp = std::fopen(path, "w");
        if (!fp) throw std::runtime_error(std::string("cannot write ") + path + ": " + std::strerror(errno));
        std::fprintf(fp, "%%%%MatrixMarket matrix array real general\n%d 1\n", n);
        for (int32_t i = 0; i < n; ++i) std::fprintf(fp, "%.17g\n", v[i]);
        if (std::fclose(fp) != 0) throw std::runtime_error(std::string("write failed: ") + path);
    });
}

int iga_mm_read_vector_len(const char* path, int32_t* n) {
    return guarded([&] { *n = int32_t(read_vector(path).size()); });
}

int iga_mm_read_vector(const char* path, double* v) {
    return guarded([&] {
        const std::vector<double> x = read_vector(path);
        std::copy(x.begin(), x.end(), v);
    });
}

}  // extern "C"
