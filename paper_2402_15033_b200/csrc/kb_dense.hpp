// Host-side small dense algebra of the hot path: the O(w³)/O(m³) pieces the
// paper replicates on every rank — Pythagorean Cholesky,
// R combinations, Hessenberg assembly, Givens least squares — plus the
// breakdown-only spectral diagnostic.  Each routine follows the reference
// algorithm operation for operation (file:line on each), so identical Gram
// entries give bit-identical factors on every rank.
#pragma once

#include <cstdint>
#include <vector>

#include "kb_common.hpp"

namespace kb {

// Column-major dense matrix (host).
struct Mat {
    i64 rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(i64 r, i64 c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(i64 i, i64 j) { return a[static_cast<size_t>(i + j * rows)]; }
    double operator()(i64 i, i64 j) const { return a[static_cast<size_t>(i + j * rows)]; }
    double* col(i64 j) { return a.data() + j * rows; }
    const double* col(i64 j) const { return a.data() + j * rows; }
};

// Square upper-triangular factor, entries below the diagonal are zero
// (UpperTriangular, dense_matrix.hpp:101-131).
struct Upper {
    i64 dim = 0;
    std::vector<double> a;
    Upper() = default;
    explicit Upper(i64 d) : dim(d), a(static_cast<size_t>(d * d), 0.0) {}
    double& at(i64 i, i64 j) { return a[static_cast<size_t>(i + j * dim)]; }
    double operator()(i64 i, i64 j) const { return a[static_cast<size_t>(i + j * dim)]; }
};

// BlockRecord (basis_store.hpp:28-34).
struct BlockRecord {
    i64 c0 = 0;
    i64 width = 0;
    bool overlap = false;
    std::vector<double> carried;
    double carried_diag = 1.0;
};

// Sequential dot in index order (dense_matrix.hpp:133-137).
double dot_seq(const double* a, const double* b, i64 n);
// try_cholesky (dense_kernels.hpp:111-127): 0 or the 1-based failing pivot.
i64 try_cholesky(const Mat& s, Upper& r);
// tri_mul (dense_kernels.hpp:261-272).
Upper tri_mul(const Upper& a, const Upper& b);
// mat_mul(A, B) (dense_kernels.hpp:63-70): column-wise axpy, zero entries skipped.
Mat mat_mul_nn(const Mat& a, const Mat& b);
// assemble_hessenberg with the monomial change of basis (gmres.hpp:40-49, 100-136).
Mat assemble_hessenberg(const Upper& r, i64 m, const std::vector<BlockRecord>& blocks);
// solve_hessenberg_lsq (gmres.hpp:146-185).
struct Lsq {
    std::vector<double> y;
    double implicit_residual = 0.0;
    i64 valid_cols = 0;
};
Lsq solve_hessenberg_lsq(const Mat& h, double gamma);
// accumulated_cond(Q, X).cond (spectral.hpp:151-176) on host copies; used
// only on a breakdown for AppendOutcome::kappa_estimate (basis_store.hpp:383-387).
double accumulated_cond(const Mat& q, const Mat& x);

}  // namespace kb
