// TEST INFRASTRUCTURE — what the reference's own unit tests need beyond the
// drop-in API, for compiling them unchanged (tests/cpp/Makefile):
//   * their input generators — gen_glued / gen_logscaled (matgen.hpp:48-128)
//     and the Householder Q behind their random_orthonormal helper
//     (dense_kernels.hpp:164) — taken from the reference itself through the
//     oracle (oracle/_ref/libkrylov_ref.so, kref_* entries), so the tests see
//     the very matrices the reference's tests see;
//   * mat_mul with transpose flags (dense_kernels.hpp:54), a host product
//     the tests use to build and check their inputs.
// Everything under test (CholQR, BCGS-PIP, BCGS2, the BasisStore, the MPK,
// ortho_error) comes from the product, include/krylov_b200.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "krylov_b200/io.hpp"
#include "krylov_b200/krylov.hpp"

extern "C" {
int kref_gen_glued(int64_t n, int64_t p, int64_t s, double kappa_panel, double growth, double coupling,
                   uint64_t seed, double* out);
int kref_gen_logscaled(int64_t n, int64_t k, double kappa, uint64_t seed, double* out);
int kref_householder_q(int64_t rows, int64_t cols, const double* a, double* q);
const char* kref_last_error(void);
}

namespace krylov {
using namespace krylov_b200;

struct Seed {
    std::uint64_t value = 0;
};
struct LogscaledPanel {
    DenseMatrix matrix;
    std::vector<double> planted_sigma;
};
struct GluedMatrix {
    DenseMatrix matrix;
    index_t panels = 0, panel_cols = 0;
};
struct QrResult {
    DenseMatrix q;
};

namespace refcompat_detail {
inline void ok(int rc) {
    if (rc == 0) return;
    const std::string msg = kref_last_error();
    if (rc == KRY_DIMENSION_MISMATCH) throw DimensionMismatch(msg);
    throw std::invalid_argument(msg);
}
}  // namespace refcompat_detail

inline LogscaledPanel gen_logscaled(index_t n, index_t k, double kappa, Seed seed) {
    LogscaledPanel p{DenseMatrix(n, k), {}};
    refcompat_detail::ok(kref_gen_logscaled(static_cast<int64_t>(n), static_cast<int64_t>(k), kappa, seed.value,
                                            p.matrix.data()));
    return p;
}
inline GluedMatrix gen_glued(index_t n, index_t p, index_t s, double kappa_panel, double growth, double coupling,
                             Seed seed) {
    GluedMatrix g{DenseMatrix(n, p * s), p, s};
    refcompat_detail::ok(kref_gen_glued(static_cast<int64_t>(n), static_cast<int64_t>(p), static_cast<int64_t>(s),
                                        kappa_panel, growth, coupling, seed.value, g.matrix.data()));
    return g;
}
inline QrResult householder_qr(ConstMatrixView a) {
    QrResult r{DenseMatrix(a.rows(), a.cols())};
    refcompat_detail::ok(kref_householder_q(static_cast<int64_t>(a.rows()), static_cast<int64_t>(a.cols()), a.data(),
                                            r.q.data()));
    return r;
}

enum class Op { None, Trans };
inline DenseMatrix mat_mul(ConstMatrixView a, ConstMatrixView b, Op oa = Op::None, Op ob = Op::None) {
    const index_t m = oa == Op::None ? a.rows() : a.cols(), k = oa == Op::None ? a.cols() : a.rows();
    const index_t kb = ob == Op::None ? b.rows() : b.cols(), nn = ob == Op::None ? b.cols() : b.rows();
    if (k != kb) throw DimensionMismatch("mat_mul inner dimensions");
    DenseMatrix c(m, nn);
    for (index_t j = 0; j < nn; ++j)
        for (index_t l = 0; l < k; ++l) {
            const double blj = ob == Op::None ? b(l, j) : b(j, l);
            for (index_t i = 0; i < m; ++i) c(i, j) += (oa == Op::None ? a(i, l) : a(l, i)) * blj;
        }
    return c;
}
}  // namespace krylov
