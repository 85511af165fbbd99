// CPU check of the drop-in's host generators (include/krylov_b200/io.hpp:
// gen_laplace2d 5/9-point, gen_laplace3d) against the reference's
// (oracle/_ref, kref_laplace*): identical CSR structure and values, bit for
// bit.  Built and run by tests/test_host_cpp.py (no GPU needed).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "krylov_b200/io.hpp"

extern "C" {
int kref_laplace2d_size(int64_t nx, int64_t ny, int stencil, int64_t* n, int64_t* nnz);
int kref_laplace2d(int64_t nx, int64_t ny, int stencil, int64_t* rp, int64_t* ci, double* v);
int kref_laplace3d_size(int64_t nx, int64_t ny, int64_t nz, int64_t* n, int64_t* nnz);
int kref_laplace3d(int64_t nx, int64_t ny, int64_t nz, int64_t* rp, int64_t* ci, double* v);
}

namespace {
int failures = 0;

void compare(const char* what, const krylov_b200::CsrMatrix& a, int64_t n, const std::vector<int64_t>& rp,
             const std::vector<int64_t>& ci, const std::vector<double>& v) {
    bool ok = static_cast<int64_t>(a.n) == n && a.row_ptr.size() == rp.size() && a.col_idx.size() == ci.size();
    for (size_t i = 0; ok && i < rp.size(); ++i) ok = static_cast<int64_t>(a.row_ptr[i]) == rp[i];
    for (size_t k = 0; ok && k < ci.size(); ++k)
        ok = static_cast<int64_t>(a.col_idx[k]) == ci[k] && std::memcmp(&a.vals[k], &v[k], 8) == 0;
    std::printf("%s %s\n", ok ? "OK  " : "FAIL", what);
    failures += ok ? 0 : 1;
}

void check2d(int64_t nx, int64_t ny, int stencil) {
    int64_t n = 0, nnz = 0;
    kref_laplace2d_size(nx, ny, stencil, &n, &nnz);
    std::vector<int64_t> rp(n + 1), ci(nnz);
    std::vector<double> v(nnz);
    kref_laplace2d(nx, ny, stencil, rp.data(), ci.data(), v.data());
    char what[96];
    std::snprintf(what, sizeof what, "gen_laplace2d(%lld, %lld, %d)", static_cast<long long>(nx),
                  static_cast<long long>(ny), stencil);
    compare(what, krylov_b200::gen_laplace2d(nx, ny, stencil), n, rp, ci, v);
}

void check3d(int64_t nx, int64_t ny, int64_t nz) {
    int64_t n = 0, nnz = 0;
    kref_laplace3d_size(nx, ny, nz, &n, &nnz);
    std::vector<int64_t> rp(n + 1), ci(nnz);
    std::vector<double> v(nnz);
    kref_laplace3d(nx, ny, nz, rp.data(), ci.data(), v.data());
    char what[96];
    std::snprintf(what, sizeof what, "gen_laplace3d(%lld, %lld, %lld)", static_cast<long long>(nx),
                  static_cast<long long>(ny), static_cast<long long>(nz));
    compare(what, krylov_b200::gen_laplace3d(nx, ny, nz), n, rp, ci, v);
}
}  // namespace

int main() {
    for (int st : {5, 9})
        for (auto [nx, ny] : {std::pair<int64_t, int64_t>{2, 2}, {3, 7}, {12, 12}, {100, 37}, {257, 3}}) check2d(nx, ny, st);
    for (auto d : {std::vector<int64_t>{2, 2, 2}, {5, 3, 4}, {17, 9, 11}, {40, 33, 2}}) check3d(d[0], d[1], d[2]);
    bool threw = false;
    try {
        krylov_b200::gen_laplace2d(4, 4, 7);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    std::printf("%s stencil 7 rejected\n", threw ? "OK  " : "FAIL");
    failures += threw ? 0 : 1;
    std::printf("%d failures\n", failures);
    return failures == 0 ? 0 : 1;
}
