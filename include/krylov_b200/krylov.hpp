// krylov_b200/krylov.hpp — C++ drop-in for the hot path of the CPU reference
// (/root/reference/proj/include/krylov).  Header-only, over the C ABI of
// krylov_b200.h (link libkrylov_b200.so).  Names, signatures, value
// semantics and exception types follow the reference so that caller code
// switches by changing `#include "krylov/gmres.hpp"` + `krylov::` to this
// header + `krylov_b200::`:
//
//   reference                                   here
//   sstep_gmres(CsrMatrix, span b, span x0, cfg) gmres.hpp:396      same
//   standard_gmres(...)                          gmres.hpp:404      same
//   bcgs_pip / bcgs_pip_partial / bcgs_pip2      block_ortho.hpp:152-208 same
//   cholqr / cholqr2 / bcgs_project / bcgs2      block_ortho.hpp:49-137 same (HHQR intra: one column)
//   ortho_error                                  spectral.hpp:104   same (device Gram)
//   try_cholesky                                 dense_kernels.hpp:111 same
//   spmv / mpk_monomial                          csr_matrix.hpp:69, gmres.hpp:80 same
//   BasisStore                                   basis_store.hpp:42  same members (device-resident Q)
//   SyncCounter, OrthoKind, OrthoScheme, SolverConfig, SolveReport, AppendOutcome,
//   BlockRecord, PanelState, DenseMatrix, ConstMatrixView, UpperTriangular, CsrMatrix
//
// Everything computes on the GPU; without a device the calls throw
// DeviceError (there is no CPU fallback).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../krylov_b200.h"

namespace krylov_b200 {

using index_t = std::size_t;

// ---- exceptions (types.hpp) ---------------------------------------------
class DimensionMismatch : public std::invalid_argument {
public:
    explicit DimensionMismatch(const std::string& w) : std::invalid_argument(w) {}
};
class NotPositiveDefinite : public std::runtime_error {
public:
    explicit NotPositiveDefinite(index_t p)
        : std::runtime_error("matrix not positive definite at pivot " + std::to_string(p)), pivot(p) {}
    index_t pivot;
};
class SingularFactor : public std::runtime_error {
public:
    SingularFactor() : std::runtime_error("triangular factor has a zero diagonal entry") {}
};
class SingularR : public std::runtime_error {
public:
    explicit SingularR(index_t c)
        : std::runtime_error("basis coefficient matrix singular at column " + std::to_string(c)), column(c) {}
    index_t column;
};
class DeviceError : public std::runtime_error {
public:
    DeviceError(int code, const std::string& w) : std::runtime_error(w), code(code) {}
    int code;
};

namespace detail {
inline void check(int rc, int64_t aux = 0) {
    if (rc == KRY_OK) return;
    const std::string msg = kry_last_error();
    switch (rc) {
        case KRY_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case KRY_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(static_cast<index_t>(aux));
        case KRY_SINGULAR_FACTOR: throw SingularFactor();
        case KRY_SINGULAR_R: throw SingularR(static_cast<index_t>(aux));
        case KRY_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw DeviceError(rc, std::string(kry_status_name(rc)) + ": " + msg);
    }
}
}  // namespace detail

// ---- containers (dense_matrix.hpp) ---------------------------------------
class ConstMatrixView {
public:
    ConstMatrixView() = default;
    ConstMatrixView(const double* d, index_t r, index_t c) : data_(d), rows_(r), cols_(c) {}
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    bool empty() const { return rows_ == 0 || cols_ == 0; }
    const double* data() const { return data_; }
    const double* col(index_t j) const { return data_ + j * rows_; }
    double operator()(index_t i, index_t j) const { return data_[i + j * rows_]; }
    ConstMatrixView col_range(index_t first, index_t count) const {
        return ConstMatrixView(data_ + first * rows_, rows_, count);
    }

private:
    const double* data_ = nullptr;
    index_t rows_ = 0, cols_ = 0;
};

class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(index_t r, index_t c) : rows_(r), cols_(c), data_(r * c, 0.0) {}
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t size() const { return data_.size(); }
    bool empty() const { return data_.empty(); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double* col(index_t j) { return data_.data() + j * rows_; }
    const double* col(index_t j) const { return data_.data() + j * rows_; }
    double& operator()(index_t i, index_t j) { return data_[i + j * rows_]; }
    double operator()(index_t i, index_t j) const { return data_[i + j * rows_]; }
    operator ConstMatrixView() const { return view(); }
    ConstMatrixView view() const { return ConstMatrixView(data_.data(), rows_, cols_); }
    ConstMatrixView col_range(index_t f, index_t c) const { return view().col_range(f, c); }
    void set_col(index_t j, const double* src) { std::memcpy(col(j), src, rows_ * sizeof(double)); }
    double frobenius_norm() const {
        double s = 0.0;
        for (double x : data_) s += x * x;
        return std::sqrt(s);
    }

private:
    index_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// Host vector helpers of dense_matrix.hpp:133-150 (input preparation and
// checks on host copies; the solver's vector work runs on the GPU).
inline double dot(const double* a, const double* b, index_t n) {
    double s = 0.0;
    for (index_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
inline double norm2(const double* a, index_t n) { return std::sqrt(dot(a, a, n)); }
inline double norm2(const std::vector<double>& a) { return norm2(a.data(), a.size()); }
inline void axpy(double alpha, const double* x, double* y, index_t n) {
    for (index_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}
inline constexpr double machine_eps = std::numeric_limits<double>::epsilon();  // spectral.hpp:14

class UpperTriangular {
public:
    UpperTriangular() = default;
    explicit UpperTriangular(index_t d) : dim_(d), data_(d * d, 0.0) {}
    index_t dim() const { return dim_; }
    double& at(index_t i, index_t j) { return data_[i + j * dim_]; }
    double operator()(index_t i, index_t j) const { return data_[i + j * dim_]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    ConstMatrixView view() const { return ConstMatrixView(data_.data(), dim_, dim_); }

private:
    index_t dim_ = 0;
    std::vector<double> data_;
};

struct CsrMatrix {  // csr_matrix.hpp:17-65 (indices stored as the reference's size_t)
    index_t n = 0;
    std::vector<index_t> row_ptr, col_idx;
    std::vector<double> vals;
    index_t nnz() const { return vals.size(); }
    // Triplets (row, col, value) → CSR with ascending columns per row,
    // duplicate entries summed in the order given (csr_matrix.hpp:42).
    static CsrMatrix from_triplets(index_t n, std::vector<std::tuple<index_t, index_t, double>> trip) {
        for (const auto& t : trip)
            if (std::get<0>(t) >= n || std::get<1>(t) >= n) throw DimensionMismatch("dimension mismatch: triplet index");
        std::stable_sort(trip.begin(), trip.end(), [](const auto& a, const auto& b) {
            return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                                    : std::get<1>(a) < std::get<1>(b);
        });
        CsrMatrix m;
        m.n = n;
        m.row_ptr.assign(n + 1, 0);
        for (std::size_t k = 0; k < trip.size(); ++k) {
            const auto& [r, c, v] = trip[k];
            if (k > 0 && std::get<0>(trip[k - 1]) == r && std::get<1>(trip[k - 1]) == c) {
                m.vals.back() += v;
                continue;
            }
            m.col_idx.push_back(c);
            m.vals.push_back(v);
            ++m.row_ptr[r + 1];
        }
        for (index_t i = 0; i < n; ++i) m.row_ptr[i + 1] += m.row_ptr[i];
        return m;
    }
};

// ---- scheme / telemetry types (block_ortho.hpp, basis_store.hpp, gmres.hpp) ----
struct SyncCounter {
    long long reduces = 0;
    std::vector<long long> per_block, per_big_panel;
    void add(long long k = 1) { reduces += k; }
};
enum class OrthoKind { Bcgs2Hhqr = KRY_ORTHO_BCGS2_HHQR, Bcgs2Cholqr2 = KRY_ORTHO_BCGS2_CHOLQR2,
                       BcgsPip2 = KRY_ORTHO_BCGS_PIP2, TwoStage = KRY_ORTHO_TWO_STAGE };
struct OrthoScheme {
    OrthoKind kind = OrthoKind::BcgsPip2;
    index_t big_panel_size = 0;
};
inline const char* ortho_kind_name(OrthoKind k) {  // block_ortho.hpp:33-41
    switch (k) {
        case OrthoKind::Bcgs2Hhqr: return "bcgs2-hhqr";
        case OrthoKind::Bcgs2Cholqr2: return "bcgs2-cholqr2";
        case OrthoKind::BcgsPip2: return "bcgs-pip2";
        case OrthoKind::TwoStage: return "two-stage";
    }
    return "?";
}
enum class PanelState { Raw, Preprocessed, Final };
struct AppendOutcome {
    index_t committed = 0;
    bool truncated = false, breakdown = false;
    index_t pivot = 0;
    double kappa_estimate = 0;
};
struct BlockRecord {
    index_t c0 = 0, width = 0;
    bool overlap = false;
    std::vector<double> carried;
    double carried_diag = 1.0;
};
struct BlockOrthoResult {
    DenseMatrix q, r_col;
    UpperTriangular r_jj;
};
struct PipOutcome {
    DenseMatrix r_col;
    UpperTriangular r_chol;
    DenseMatrix q;
    index_t bad_pivot = 0;
};
struct BlockQr {
    DenseMatrix q;
    UpperTriangular r;
};

struct SolverConfig {
    index_t restart_len = 60, step = 5, big_step = 0;
    OrthoScheme scheme{OrthoKind::BcgsPip2, 0};
    double rel_tol = 1e-6;
    index_t max_iters = 500000;
    index_t effective_big_step() const { return big_step == 0 ? restart_len : big_step; }
    kry_solver_config to_c() const {
        kry_solver_config c{};
        c.restart_len = static_cast<int64_t>(restart_len);
        c.step = static_cast<int64_t>(step);
        c.big_step = static_cast<int64_t>(big_step);
        c.scheme_kind = static_cast<int32_t>(scheme.kind);
        c.scheme_big_panel_size = static_cast<int64_t>(scheme.big_panel_size);
        c.rel_tol = rel_tol;
        c.max_iters = static_cast<int64_t>(max_iters);
        return c;
    }
};
enum class SolveStatus { Converged, MaxIters, OrthoBreakdown, Stagnation };
struct SolveReport {
    SolveStatus status = SolveStatus::MaxIters;
    index_t iterations = 0, restarts = 0;
    double initial_residual = 0.0, final_relative_residual = 0.0;
    std::vector<double> cycle_residuals;
    bool breakdown = false;
    double breakdown_kappa = 0.0;
    SyncCounter sync;
    double reduces_per_iteration = 0.0, wall_seconds = 0.0;
    std::vector<double> solution;
};

// ---- device context and operators ------------------------------------------
class Context {
public:
    explicit Context(int device = 0, int nranks = 1, int rank = 0, const void* nccl_id = nullptr) {
        kry_ctx* c = nullptr;
        detail::check(kry_ctx_create(device, nranks, rank, nccl_id, &c));
        h_.reset(c);
    }
    kry_ctx* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(kry_ctx* c) const { kry_ctx_destroy(c); }
    };
    std::unique_ptr<kry_ctx, Del> h_;
};

inline Context& default_context() {
    static Context ctx(0);
    return ctx;
}

class Operator {
public:
    static Operator csr(const CsrMatrix& a, Context& ctx = default_context()) {
        std::vector<int64_t> rp(a.row_ptr.begin(), a.row_ptr.end()), ci(a.col_idx.begin(), a.col_idx.end());
        kry_operator* o = nullptr;
        detail::check(kry_operator_create_csr(ctx.get(), static_cast<int64_t>(a.n), 0, static_cast<int64_t>(a.n),
                                              rp.data(), ci.data(), a.vals.data(), &o));
        return Operator(o, ctx);
    }
    static Operator laplace2d(index_t nx, index_t ny, Context& ctx = default_context()) {
        kry_operator* o = nullptr;
        detail::check(kry_operator_create_laplace2d(ctx.get(), static_cast<int64_t>(nx), static_cast<int64_t>(ny), &o));
        return Operator(o, ctx);
    }
    static Operator laplace3d(index_t nx, index_t ny, index_t nz, Context& ctx = default_context()) {
        kry_operator* o = nullptr;
        detail::check(kry_operator_create_laplace3d(ctx.get(), static_cast<int64_t>(nx), static_cast<int64_t>(ny),
                                                    static_cast<int64_t>(nz), &o));
        return Operator(o, ctx);
    }
    index_t rows() const {
        int64_t ng = 0, rb = 0, nl = 0;
        detail::check(kry_operator_rows(h_.get(), &ng, &rb, &nl));
        return static_cast<index_t>(nl);
    }
    kry_operator* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    struct Del {
        void operator()(kry_operator* o) const { kry_operator_destroy(o); }
    };
    Operator(kry_operator* o, Context& c) : h_(o), ctx_(&c) {}
    std::unique_ptr<kry_operator, Del> h_;
    Context* ctx_;
};

// ---- kernels ---------------------------------------------------------------------
inline std::vector<double> spmv(const Operator& a, std::span<const double> x) {
    if (x.size() != a.rows()) throw DimensionMismatch("spmv vector length");
    std::vector<double> y(x.size());
    detail::check(kry_spmv(a.context().get(), a.get(), x.data(), y.data()));
    return y;
}
inline std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x) { return spmv(Operator::csr(a), x); }

inline DenseMatrix mpk_monomial(const Operator& a, std::span<const double> start, index_t s) {
    if (start.size() != a.rows()) throw DimensionMismatch("mpk start vector length");
    DenseMatrix v(a.rows(), s + 1);
    detail::check(kry_mpk(a.context().get(), a.get(), start.data(), static_cast<int64_t>(s), v.data()));
    return v;
}
inline DenseMatrix mpk_monomial(const CsrMatrix& a, std::span<const double> start, index_t s) {
    return mpk_monomial(Operator::csr(a), start, s);
}

inline index_t try_cholesky(ConstMatrixView s, UpperTriangular& r) {
    if (s.rows() != s.cols()) throw DimensionMismatch("cholesky needs a square matrix");
    r = UpperTriangular(s.rows());
    int64_t piv = 0;
    detail::check(kry_try_cholesky(static_cast<int64_t>(s.rows()), s.data(), r.data(), &piv));
    return static_cast<index_t>(piv);
}

// ---- block orthogonalization (block_ortho.hpp) --------------------------------------
inline PipOutcome bcgs_pip_partial(ConstMatrixView q_prev, ConstMatrixView v, SyncCounter& sync,
                                   Context& ctx = default_context()) {
    const index_t c0 = q_prev.empty() ? 0 : q_prev.cols(), w = v.cols(), n = v.rows();
    PipOutcome out;
    out.r_col = DenseMatrix(c0, w);
    out.r_chol = UpperTriangular(w);
    DenseMatrix q(n, w);
    int64_t bad = 0, red = 0;
    detail::check(kry_bcgs_pip_partial(ctx.get(), static_cast<int64_t>(n), c0 ? q_prev.data() : nullptr,
                                       static_cast<int64_t>(c0), v.data(), static_cast<int64_t>(w), q.data(),
                                       out.r_col.data(), out.r_chol.data(), &bad, &red));
    sync.add(red);
    out.bad_pivot = static_cast<index_t>(bad);
    if (bad == 0) out.q = std::move(q);
    return out;
}

inline BlockOrthoResult bcgs_pip(ConstMatrixView q_prev, ConstMatrixView v, SyncCounter& sync,
                                 Context& ctx = default_context()) {
    PipOutcome p = bcgs_pip_partial(q_prev, v, sync, ctx);
    if (p.bad_pivot != 0) throw NotPositiveDefinite(p.bad_pivot);
    return BlockOrthoResult{std::move(p.q), std::move(p.r_col), std::move(p.r_chol)};
}

inline BlockOrthoResult bcgs_pip2(ConstMatrixView q_prev, ConstMatrixView v, SyncCounter& sync,
                                  Context& ctx = default_context()) {
    const index_t c0 = q_prev.empty() ? 0 : q_prev.cols(), w = v.cols(), n = v.rows();
    BlockOrthoResult out{DenseMatrix(n, w), DenseMatrix(c0, w), UpperTriangular(w)};
    int64_t piv = 0, red = 0;
    const int rc = kry_bcgs_pip2(ctx.get(), static_cast<int64_t>(n), c0 ? q_prev.data() : nullptr,
                                 static_cast<int64_t>(c0), v.data(), static_cast<int64_t>(w), out.q.data(),
                                 out.r_col.data(), out.r_jj.data(), &piv, &red);
    sync.add(red);
    detail::check(rc, piv);
    return out;
}

inline BlockQr cholqr(ConstMatrixView v, SyncCounter& sync, Context& ctx = default_context()) {
    BlockOrthoResult r = bcgs_pip(ConstMatrixView(), v, sync, ctx);
    return BlockQr{std::move(r.q), std::move(r.r_jj)};
}

// The BCGS2 baseline (block_ortho.hpp:57-137) on the device.
inline BlockQr cholqr2(ConstMatrixView v, SyncCounter& sync, Context& ctx = default_context()) {
    const index_t n = v.rows(), w = v.cols();
    BlockQr out{DenseMatrix(n, w), UpperTriangular(w)};
    int64_t piv = 0, red = 0;
    const int rc = kry_cholqr2(ctx.get(), static_cast<int64_t>(n), v.data(), static_cast<int64_t>(w), out.q.data(),
                               out.r.data(), &piv, &red);
    sync.add(red);
    detail::check(rc, piv);
    return out;
}

struct ProjectResult {
    DenseMatrix vhat;     // V − Q_prev·(Q_prevᵀV)
    DenseMatrix r_block;  // Q_prevᵀV
};
inline ProjectResult bcgs_project(ConstMatrixView q_prev, ConstMatrixView v, SyncCounter& sync,
                                  Context& ctx = default_context()) {
    const index_t c0 = q_prev.empty() ? 0 : q_prev.cols(), w = v.cols(), n = v.rows();
    ProjectResult out{DenseMatrix(n, w), DenseMatrix(c0, w)};
    int64_t red = 0;
    detail::check(kry_bcgs_project(ctx.get(), static_cast<int64_t>(n), c0 ? q_prev.data() : nullptr,
                                   static_cast<int64_t>(c0), v.data(), static_cast<int64_t>(w), out.vhat.data(),
                                   out.r_block.data(), &red));
    sync.add(red);
    return out;
}

enum class IntraKind { Hhqr, Cholqr2 };  // Hhqr: one column only on the device path
inline BlockOrthoResult bcgs2(ConstMatrixView q_prev, ConstMatrixView v, IntraKind intra, SyncCounter& sync,
                              Context& ctx = default_context()) {
    const index_t c0 = q_prev.empty() ? 0 : q_prev.cols(), w = v.cols(), n = v.rows();
    BlockOrthoResult out{DenseMatrix(n, w), DenseMatrix(c0, w), UpperTriangular(w)};
    int64_t piv = 0, red = 0;
    const int rc = kry_bcgs2(ctx.get(), static_cast<int64_t>(n), c0 ? q_prev.data() : nullptr,
                             static_cast<int64_t>(c0), v.data(), static_cast<int64_t>(w),
                             intra == IntraKind::Hhqr ? 0 : 1, out.q.data(), out.r_col.data(), out.r_jj.data(),
                             &piv, &red);
    sync.add(red);
    detail::check(rc, piv);
    return out;
}

// ‖I − QᵀQ‖₂ (spectral.hpp:104): the Gram QᵀQ on the device, the 2-norm of
// the small symmetric deviation by cyclic Jacobi rotations on the host.
inline double ortho_error(ConstMatrixView q, Context& ctx = default_context()) {
    if (q.empty()) return 0.0;
    const index_t k = q.cols();
    if (k > 512) throw DimensionMismatch("ortho_error capped at 512 columns");
    std::vector<double> a(k * k);
    detail::check(kry_gram_full(ctx.get(), static_cast<int64_t>(q.rows()), q.data(), static_cast<int64_t>(k), a.data()));
    auto at = [&](index_t i, index_t j) -> double& { return a[i + j * k]; };
    for (index_t j = 0; j < k; ++j)
        for (index_t i = 0; i < k; ++i) at(i, j) = (i == j ? 1.0 : 0.0) - at(i, j);
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (index_t i = 0; i < k; ++i) diag = std::max(diag, std::abs(at(i, i)));
        for (index_t p = 0; p + 1 < k; ++p)
            for (index_t r = p + 1; r < k; ++r) {
                const double apr = at(p, r);
                if (apr == 0.0) continue;
                off = std::max(off, std::abs(apr));
                // rotation zeroing (p, r): t = tan θ, the smaller root
                const double theta = (at(r, r) - at(p, p)) / (2.0 * apr);
                const double t = theta == 0.0 ? 1.0
                                              : std::copysign(1.0, theta) / (std::abs(theta) + std::hypot(1.0, theta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (index_t i = 0; i < k; ++i) {  // columns p, r
                    const double x = at(i, p), y = at(i, r);
                    at(i, p) = c * x - sn * y;
                    at(i, r) = sn * x + c * y;
                }
                for (index_t i = 0; i < k; ++i) {  // rows p, r
                    const double x = at(p, i), y = at(r, i);
                    at(p, i) = c * x - sn * y;
                    at(r, i) = sn * x + c * y;
                }
            }
        if (off <= machine_eps * std::max(diag, 1e-300)) break;
    }
    double norm = 0.0;
    for (index_t i = 0; i < k; ++i) norm = std::max(norm, std::abs(at(i, i)));
    return norm;
}

// ---- basis store (basis_store.hpp:42-401), device-resident -----------------------------
class BasisStore {
public:
    BasisStore(index_t n, index_t m, index_t panel_size, index_t big_panel_size, Context& ctx = default_context())
        : n_(n), m_(m) {
        kry_store* s = nullptr;
        detail::check(kry_store_create(ctx.get(), static_cast<int64_t>(n), static_cast<int64_t>(m),
                                       static_cast<int64_t>(panel_size), static_cast<int64_t>(big_panel_size), &s));
        h_.reset(s);
    }
    index_t rows() const { return n_; }
    index_t capacity() const { return info().capacity; }
    index_t filled() const { return info().filled; }
    index_t finalized_count() const { return info().finalized; }
    index_t big_panel_start() const { return info().big_panel_start; }
    index_t panel_size() const { return info().panel_size; }
    index_t big_panel_size() const { return info().big_panel_size; }
    bool big_panel_open() const { return info().big_panel_open != 0; }
    bool big_panel_full() const { return info().big_panel_full != 0; }
    bool has_seam_column() const { return info().seam_valid != 0; }

    void reset() { detail::check(kry_store_reset(h_.get())); }
    void seed_unit_column(const double* v) { detail::check(kry_store_seed_unit_column(h_.get(), v)); }

    AppendOutcome append_block(ConstMatrixView v, bool overlap, const OrthoScheme& scheme, SyncCounter& sync) {
        if (v.rows() != n_) throw DimensionMismatch("block row count");
        kry_append_outcome o{};
        int64_t d = 0;
        detail::check(kry_store_append_block(h_.get(), v.data(), static_cast<int64_t>(v.cols()), overlap ? 1 : 0,
                                             static_cast<int32_t>(scheme.kind),
                                             static_cast<int64_t>(scheme.big_panel_size), &o, &d));
        sync.add(d);
        sync.per_block.push_back(d);
        return outcome(o);
    }
    AppendOutcome preprocess_block(ConstMatrixView v, bool overlap, SyncCounter& sync) {
        return append_block(v, overlap, OrthoScheme{OrthoKind::TwoStage, big_panel_size()}, sync);
    }
    AppendOutcome finalize_big_panel(SyncCounter& sync) {
        const bool open = big_panel_open();
        kry_append_outcome o{};
        int64_t d = 0;
        detail::check(kry_store_finalize_big_panel(h_.get(), &o, &d));
        if (open) {
            sync.add(d);
            sync.per_big_panel.push_back(d);
        }
        return outcome(o);
    }

    UpperTriangular coefficients() const {
        UpperTriangular r(m_ + 1);
        detail::check(kry_store_coefficients(h_.get(), r.data()));
        return r;
    }
    // A host copy of column j (the basis lives on the GPU); converts to the
    // reference's `const double*` for the duration of the full expression.
    struct HostColumn : std::vector<double> {
        using std::vector<double>::vector;
        operator const double*() const { return data(); }
    };
    HostColumn column(index_t j) const {
        HostColumn c(n_);
        detail::check(kry_store_column(h_.get(), static_cast<int64_t>(j), c.data()));
        return c;
    }
    DenseMatrix all() const {
        const index_t f = filled();
        DenseMatrix q(n_, f);
        if (f) detail::check(kry_store_columns(h_.get(), 0, static_cast<int64_t>(f), q.data()));
        return q;
    }
    std::vector<PanelState> panel_states() const {
        std::vector<int32_t> s(info().n_panel_states);
        detail::check(kry_store_panel_states(h_.get(), s.data()));
        std::vector<PanelState> out;
        for (int32_t v : s) out.push_back(static_cast<PanelState>(v));
        return out;
    }
    std::vector<BlockRecord> block_records() const {
        std::vector<BlockRecord> out;
        for (int64_t i = 0; i < info().n_records; ++i) {
            int64_t c0 = 0, w = 0;
            int32_t ov = 0;
            double diag = 0;
            std::vector<double> carried(m_ + 2);
            detail::check(kry_store_block_record(h_.get(), i, &c0, &w, &ov, carried.data(), &diag));
            carried.resize(ov ? static_cast<size_t>(c0) : 0);
            out.push_back(BlockRecord{static_cast<index_t>(c0), static_cast<index_t>(w), ov != 0,
                                      std::move(carried), diag});
        }
        return out;
    }

private:
    kry_store_info info() const {
        kry_store_info i{};
        detail::check(kry_store_get_info(h_.get(), &i));
        return i;
    }
    static AppendOutcome outcome(const kry_append_outcome& o) {
        return AppendOutcome{static_cast<index_t>(o.committed), o.truncated != 0, o.breakdown != 0,
                             static_cast<index_t>(o.pivot), o.kappa_estimate};
    }
    struct Del {
        void operator()(kry_store* s) const { kry_store_destroy(s); }
    };
    std::unique_ptr<kry_store, Del> h_;
    index_t n_, m_;
};

// ---- solvers (gmres.hpp:396-411) -------------------------------------------------------
namespace detail {
inline SolveReport solve(bool standard, const Operator& a, std::span<const double> b, std::span<const double> x0,
                         const SolverConfig& cfg) {
    const index_t n = a.rows();
    if (b.size() != n) throw DimensionMismatch("rhs length");
    if (!x0.empty() && x0.size() != n) throw DimensionMismatch("x0 length");
    SolveReport rep;
    rep.solution.assign(n, 0.0);
    // The reference's SolveReport keeps every entry: size the history
    // buffers from max_iters (one per-block entry per s iterations, at most
    // one cycle per s iterations) and, should a run still report more
    // entries than fit, re-run with buffers of the reported size.
    const int64_t step = standard ? 1 : std::max<int64_t>(1, static_cast<int64_t>(cfg.step));
    const int64_t iters = static_cast<int64_t>(std::min<index_t>(cfg.max_iters, index_t(1) << 40));
    int64_t cap_c = std::min<int64_t>(iters / step + 64, int64_t(1) << 24);
    int64_t cap_b = std::min<int64_t>(2 * (iters / step) + 64, int64_t(1) << 25);
    std::vector<double> cyc;
    std::vector<int64_t> pb, pbp;
    kry_report r{};
    const kry_solver_config c = cfg.to_c();
    auto fn = standard ? kry_standard_gmres : kry_sstep_gmres;
    for (int attempt = 0;; ++attempt) {
        cyc.assign(static_cast<size_t>(cap_c), 0.0);
        pb.assign(static_cast<size_t>(cap_b), 0);
        pbp.assign(static_cast<size_t>(cap_c), 0);
        r = kry_report{};
        r.cycle_residuals = cyc.data();
        r.cycle_residuals_cap = cap_c;
        r.per_block = pb.data();
        r.per_block_cap = cap_b;
        r.per_big_panel = pbp.data();
        r.per_big_panel_cap = cap_c;
        check(fn(a.context().get(), a.get(), b.data(), x0.empty() ? nullptr : x0.data(), &c, &r,
                 rep.solution.data()));
        if ((r.n_cycle_residuals <= cap_c && r.n_per_block <= cap_b && r.n_per_big_panel <= cap_c) || attempt > 0)
            break;
        cap_c = std::max({cap_c, r.n_cycle_residuals, r.n_per_big_panel});
        cap_b = std::max(cap_b, r.n_per_block);
    }
    rep.status = static_cast<SolveStatus>(r.status);
    rep.iterations = static_cast<index_t>(r.iterations);
    rep.restarts = static_cast<index_t>(r.restarts);
    rep.initial_residual = r.initial_residual;
    rep.final_relative_residual = r.final_relative_residual;
    rep.cycle_residuals.assign(cyc.begin(), cyc.begin() + std::min<int64_t>(r.n_cycle_residuals, r.cycle_residuals_cap));
    rep.breakdown = r.breakdown != 0;
    rep.breakdown_kappa = r.breakdown_kappa;
    rep.sync.reduces = r.reduces;
    rep.sync.per_block.assign(pb.begin(), pb.begin() + std::min<int64_t>(r.n_per_block, r.per_block_cap));
    rep.sync.per_big_panel.assign(pbp.begin(), pbp.begin() + std::min<int64_t>(r.n_per_big_panel, r.per_big_panel_cap));
    rep.reduces_per_iteration = r.reduces_per_iteration;
    rep.wall_seconds = r.wall_seconds;
    return rep;
}
}  // namespace detail

inline SolveReport sstep_gmres(const Operator& a, std::span<const double> b, std::span<const double> x0,
                               const SolverConfig& cfg) {
    return detail::solve(false, a, b, x0, cfg);
}
inline SolveReport sstep_gmres(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                               const SolverConfig& cfg) {
    return detail::solve(false, Operator::csr(a), b, x0, cfg);
}
inline SolveReport standard_gmres(const Operator& a, std::span<const double> b, std::span<const double> x0,
                                  const SolverConfig& cfg) {
    return detail::solve(true, a, b, x0, cfg);
}
inline SolveReport standard_gmres(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                                  const SolverConfig& cfg) {
    return detail::solve(true, Operator::csr(a), b, x0, cfg);
}

}  // namespace krylov_b200
