// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/krylov, compiled where they lie; nothing is
// copied into this repo).  Built by oracle/Makefile into oracle/_ref/
// libkrylov_ref.so with the reference's own Release flags (-O3 -DNDEBUG,
// gnu++20, no -march; proj/CMakeLists.txt:3-8).  Used only by tests/, by
// tests/golden/make_golden.py and by bench.py's cpu_baseline / reference
// arm.  The product (paper_2402_15033_b200/) never links or loads it.
//
// Every kref_* entry mirrors the product's kry_* entry of the same name and
// fills the same structs (include/krylov_b200.h), so parity tests compare
// like with like.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "krylov/basis_store.hpp"
#include "krylov/block_ortho.hpp"
#include "krylov/csr_matrix.hpp"
#include "krylov/dense_kernels.hpp"
#include "krylov/gmres.hpp"
#include "krylov/matgen.hpp"
#include "krylov/spectral.hpp"

#include "../include/krylov_b200.h"

using namespace krylov;

namespace {

thread_local std::string g_err;
thread_local int64_t g_pivot = 0;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return KRY_OK;
    } catch (const NotPositiveDefinite& e) {
        g_err = e.what();
        g_pivot = static_cast<int64_t>(e.pivot);
        return KRY_NOT_POSITIVE_DEFINITE;
    } catch (const DimensionMismatch& e) {
        g_err = e.what();
        return KRY_DIMENSION_MISMATCH;
    } catch (const SingularFactor& e) {
        g_err = e.what();
        return KRY_SINGULAR_FACTOR;
    } catch (const SingularR& e) {
        g_err = e.what();
        g_pivot = static_cast<int64_t>(e.column);
        return KRY_SINGULAR_R;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return KRY_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KRY_INTERNAL;
    }
}

CsrMatrix make_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
    CsrMatrix a;
    a.n = static_cast<index_t>(n);
    a.row_ptr.assign(rp, rp + n + 1);
    const int64_t nnz = rp[n];
    a.col_idx.assign(ci, ci + nnz);
    a.vals.assign(v, v + nnz);
    a.validate();
    return a;
}

void copy_mat(const DenseMatrix& m, double* out) {
    if (out && m.size() > 0) std::memcpy(out, m.data(), m.size() * sizeof(double));
}

void copy_upper(const UpperTriangular& r, double* out) {
    if (out && r.dim() > 0) std::memcpy(out, r.data(), r.dim() * r.dim() * sizeof(double));
}

void fill_report(const SolveReport& rep, kry_report* out) {
    out->status = static_cast<int32_t>(rep.status);
    out->breakdown = rep.breakdown ? 1 : 0;
    out->iterations = static_cast<int64_t>(rep.iterations);
    out->restarts = static_cast<int64_t>(rep.restarts);
    out->initial_residual = rep.initial_residual;
    out->final_relative_residual = rep.final_relative_residual;
    out->breakdown_kappa = rep.breakdown_kappa;
    out->reduces = rep.sync.reduces;
    out->reduces_per_iteration = rep.reduces_per_iteration;
    out->wall_seconds = rep.wall_seconds;
    out->n_cycle_residuals = static_cast<int64_t>(rep.cycle_residuals.size());
    for (int64_t i = 0; i < out->n_cycle_residuals && i < out->cycle_residuals_cap; ++i)
        out->cycle_residuals[i] = rep.cycle_residuals[i];
    out->n_per_block = static_cast<int64_t>(rep.sync.per_block.size());
    for (int64_t i = 0; i < out->n_per_block && i < out->per_block_cap; ++i)
        out->per_block[i] = rep.sync.per_block[i];
    out->n_per_big_panel = static_cast<int64_t>(rep.sync.per_big_panel.size());
    for (int64_t i = 0; i < out->n_per_big_panel && i < out->per_big_panel_cap; ++i)
        out->per_big_panel[i] = rep.sync.per_big_panel[i];
}

SolverConfig make_cfg(const kry_solver_config* c) {
    SolverConfig cfg;
    cfg.restart_len = static_cast<index_t>(c->restart_len);
    cfg.step = static_cast<index_t>(c->step);
    cfg.big_step = static_cast<index_t>(c->big_step);
    cfg.scheme.kind = static_cast<OrthoKind>(c->scheme_kind);
    cfg.scheme.big_panel_size = static_cast<index_t>(c->scheme_big_panel_size);
    cfg.rel_tol = c->rel_tol;
    cfg.max_iters = static_cast<index_t>(c->max_iters);
    return cfg;
}

void fill_outcome(const AppendOutcome& a, kry_append_outcome* o) {
    if (!o) return;
    o->committed = static_cast<int64_t>(a.committed);
    o->truncated = a.truncated ? 1 : 0;
    o->breakdown = a.breakdown ? 1 : 0;
    o->pivot = static_cast<int64_t>(a.pivot);
    o->kappa_estimate = a.kappa_estimate;
}

struct RefStore {
    BasisStore store;
    index_t n;
    RefStore(index_t n_, index_t m, index_t s, index_t shat) : store(n_, m, s, shat), n(n_) {}
};

ConstMatrixView view(const double* p, int64_t n, int64_t k) {
    return (k == 0 || p == nullptr) ? ConstMatrixView() : ConstMatrixView(p, n, k);
}

}  // namespace

extern "C" {

const char* kref_last_error(void) { return g_err.c_str(); }
int64_t kref_last_pivot(void) { return g_pivot; }

// ---- generators (matgen.hpp) ---------------------------------------------
int kref_laplace2d_size(int64_t nx, int64_t ny, int stencil, int64_t* n, int64_t* nnz) {
    return guarded([&] {
        CsrMatrix a = gen_laplace2d(nx, ny, stencil);
        *n = a.n;
        *nnz = a.nnz();
    });
}
int kref_laplace2d(int64_t nx, int64_t ny, int stencil, int64_t* rp, int64_t* ci, double* v) {
    return guarded([&] {
        CsrMatrix a = gen_laplace2d(nx, ny, stencil);
        for (index_t i = 0; i <= a.n; ++i) rp[i] = a.row_ptr[i];
        for (index_t k = 0; k < a.nnz(); ++k) {
            ci[k] = a.col_idx[k];
            v[k] = a.vals[k];
        }
    });
}
int kref_laplace3d_size(int64_t nx, int64_t ny, int64_t nz, int64_t* n, int64_t* nnz) {
    return guarded([&] {
        CsrMatrix a = gen_laplace3d(nx, ny, nz);
        *n = a.n;
        *nnz = a.nnz();
    });
}
int kref_laplace3d(int64_t nx, int64_t ny, int64_t nz, int64_t* rp, int64_t* ci, double* v) {
    return guarded([&] {
        CsrMatrix a = gen_laplace3d(nx, ny, nz);
        for (index_t i = 0; i <= a.n; ++i) rp[i] = a.row_ptr[i];
        for (index_t k = 0; k < a.nnz(); ++k) {
            ci[k] = a.col_idx[k];
            v[k] = a.vals[k];
        }
    });
}
int kref_gen_glued(int64_t n, int64_t p, int64_t s, double kappa_panel, double growth,
                   double coupling, uint64_t seed, double* out) {
    return guarded([&] {
        GluedMatrix g = gen_glued(n, p, s, kappa_panel, growth, coupling, Seed{seed});
        copy_mat(g.matrix, out);
    });
}
int kref_gen_logscaled(int64_t n, int64_t k, double kappa, uint64_t seed, double* out) {
    return guarded([&] {
        LogscaledPanel p = gen_logscaled(n, k, kappa, Seed{seed});
        copy_mat(p.matrix, out);
    });
}

// ---- kernels -------------------------------------------------------------
int kref_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
              double* y) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, rp, ci, v);
        std::vector<double> r = spmv(a, std::span<const double>(x, n));
        std::memcpy(y, r.data(), n * sizeof(double));
    });
}
int kref_mpk(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* start,
             int64_t s, double* out) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, rp, ci, v);
        DenseMatrix m = mpk_monomial(a, std::span<const double>(start, n), s);
        copy_mat(m, out);
    });
}
int kref_gram(int64_t n, int64_t k, const double* v, double* g) {
    return guarded([&] { copy_mat(gram(ConstMatrixView(v, n, k)), g); });
}
int kref_mat_mul_tn(int64_t n, int64_t ka, const double* a, int64_t kb, const double* b, double* c) {
    return guarded([&] {
        copy_mat(mat_mul(ConstMatrixView(a, n, ka), ConstMatrixView(b, n, kb), Op::Trans, Op::None), c);
    });
}
int kref_try_cholesky(int64_t k, const double* s, double* r, int64_t* pivot) {
    return guarded([&] {
        UpperTriangular rr;
        *pivot = static_cast<int64_t>(try_cholesky(ConstMatrixView(s, k, k), rr));
        copy_upper(rr, r);
    });
}
int kref_tri_solve_right(int64_t n, int64_t k, const double* v, const double* r, double* x) {
    return guarded([&] {
        UpperTriangular rr(k);
        for (int64_t j = 0; j < k; ++j)
            for (int64_t i = 0; i <= j; ++i) rr.at(i, j) = r[i + j * k];
        copy_mat(tri_solve_right(ConstMatrixView(v, n, k), rr), x);
    });
}
int kref_ortho_error(int64_t n, int64_t k, const double* q, double* err) {
    return guarded([&] { *err = ortho_error(view(q, n, k)); });
}

// ---- block orthogonalization (block_ortho.hpp) ----------------------------
int kref_bcgs_pip_partial(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w,
                          double* q, double* r_col, double* r_chol, int64_t* bad_pivot,
                          int64_t* reduces) {
    return guarded([&] {
        SyncCounter sync;
        PipOutcome o = bcgs_pip_partial(view(qp, n, c0), ConstMatrixView(v, n, w), sync);
        copy_mat(o.r_col, r_col);
        copy_upper(o.r_chol, r_chol);
        if (o.bad_pivot == 0) copy_mat(o.q, q);
        *bad_pivot = static_cast<int64_t>(o.bad_pivot);
        if (reduces) *reduces += sync.reduces;
    });
}
int kref_bcgs_pip(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* q,
                  double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    SyncCounter sync;
    g_pivot = 0;
    int rc = guarded([&] {
        BlockOrthoResult res = bcgs_pip(view(qp, n, c0), ConstMatrixView(v, n, w), sync);
        copy_mat(res.q, q);
        copy_mat(res.r_col, r_col);
        copy_upper(res.r_jj, r_jj);
    });
    if (pivot) *pivot = (rc == KRY_NOT_POSITIVE_DEFINITE) ? g_pivot : 0;
    if (reduces) *reduces += sync.reduces;
    return rc;
}
int kref_bcgs_pip2(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* q,
                   double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    SyncCounter sync;
    g_pivot = 0;
    int rc = guarded([&] {
        BlockOrthoResult res = bcgs_pip2(view(qp, n, c0), ConstMatrixView(v, n, w), sync);
        copy_mat(res.q, q);
        copy_mat(res.r_col, r_col);
        copy_upper(res.r_jj, r_jj);
    });
    if (pivot) *pivot = (rc == KRY_NOT_POSITIVE_DEFINITE) ? g_pivot : 0;
    if (reduces) *reduces += sync.reduces;
    return rc;
}
int kref_cholqr(int64_t n, const double* v, int64_t w, double* q, double* r, int64_t* pivot,
                int64_t* reduces) {
    SyncCounter sync;
    g_pivot = 0;
    int rc = guarded([&] {
        BlockQr qr = cholqr(ConstMatrixView(v, n, w), sync);
        copy_mat(qr.q, q);
        copy_upper(qr.r, r);
    });
    if (pivot) *pivot = (rc == KRY_NOT_POSITIVE_DEFINITE) ? g_pivot : 0;
    if (reduces) *reduces += sync.reduces;
    return rc;
}

// The BCGS2 baseline pieces (block_ortho.hpp:57-137).
int kref_cholqr2(int64_t n, const double* v, int64_t w, double* q, double* r, int64_t* pivot,
                 int64_t* reduces) {
    SyncCounter sync;
    g_pivot = 0;
    int rc = guarded([&] {
        BlockQr qr = cholqr2(ConstMatrixView(v, n, w), sync);
        copy_mat(qr.q, q);
        copy_upper(qr.r, r);
    });
    if (pivot) *pivot = (rc == KRY_NOT_POSITIVE_DEFINITE) ? g_pivot : 0;
    if (reduces) *reduces += sync.reduces;
    return rc;
}
int kref_bcgs_project(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* vhat,
                      double* r_block, int64_t* reduces) {
    SyncCounter sync;
    int rc = guarded([&] {
        ProjectResult pr = bcgs_project(view(qp, n, c0), ConstMatrixView(v, n, w), sync);
        copy_mat(pr.vhat, vhat);
        copy_mat(pr.r_block, r_block);
    });
    if (reduces) *reduces += sync.reduces;
    return rc;
}
int kref_bcgs2(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, int32_t intra, double* q,
               double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    SyncCounter sync;
    g_pivot = 0;
    int rc = guarded([&] {
        BlockOrthoResult res = bcgs2(view(qp, n, c0), ConstMatrixView(v, n, w),
                                     intra == 0 ? IntraKind::Hhqr : IntraKind::Cholqr2, sync);
        copy_mat(res.q, q);
        copy_mat(res.r_col, r_col);
        copy_upper(res.r_jj, r_jj);
    });
    if (pivot) *pivot = (rc == KRY_NOT_POSITIVE_DEFINITE) ? g_pivot : 0;
    if (reduces) *reduces += sync.reduces;
    return rc;
}
// Thin Q of the reference's Householder QR (dense_kernels.hpp:164): input
// generator of the reference's own unit tests (tests/cpp refcompat).
int kref_householder_q(int64_t rows, int64_t cols, const double* a, double* q) {
    return guarded([&] {
        DenseMatrix m(rows, cols);
        std::memcpy(m.data(), a, static_cast<size_t>(rows * cols) * sizeof(double));
        copy_mat(householder_qr(m).q, q);
    });
}

// ---- basis store (basis_store.hpp) ------------------------------------------
int kref_store_create(int64_t n, int64_t m, int64_t s, int64_t shat, void** out) {
    return guarded([&] { *out = new RefStore(n, m, s, shat); });
}
void kref_store_destroy(void* st) { delete static_cast<RefStore*>(st); }
int kref_store_reset(void* st) {
    return guarded([&] { static_cast<RefStore*>(st)->store.reset(); });
}
int kref_store_seed_unit_column(void* st, const double* v) {
    return guarded([&] { static_cast<RefStore*>(st)->store.seed_unit_column(v); });
}
int kref_store_append_block(void* st, const double* v, int64_t w, int overlap, int32_t kind,
                            int64_t shat, kry_append_outcome* out, int64_t* delta) {
    return guarded([&] {
        RefStore* s = static_cast<RefStore*>(st);
        SyncCounter sync;
        AppendOutcome a = s->store.append_block(ConstMatrixView(v, s->n, w), overlap != 0,
                                                OrthoScheme{static_cast<OrthoKind>(kind),
                                                            static_cast<index_t>(shat)},
                                                sync);
        fill_outcome(a, out);
        if (delta) *delta = sync.reduces;
    });
}
int kref_store_preprocess_block(void* st, const double* v, int64_t w, int overlap,
                                kry_append_outcome* out, int64_t* delta) {
    return guarded([&] {
        RefStore* s = static_cast<RefStore*>(st);
        SyncCounter sync;
        AppendOutcome a = s->store.preprocess_block(ConstMatrixView(v, s->n, w), overlap != 0, sync);
        fill_outcome(a, out);
        if (delta) *delta = sync.reduces;
    });
}
int kref_store_finalize_big_panel(void* st, kry_append_outcome* out, int64_t* delta) {
    return guarded([&] {
        RefStore* s = static_cast<RefStore*>(st);
        SyncCounter sync;
        AppendOutcome a = s->store.finalize_big_panel(sync);
        fill_outcome(a, out);
        if (delta) *delta = sync.reduces;
    });
}
int kref_store_get_info(void* st, kry_store_info* info) {
    return guarded([&] {
        const BasisStore& b = static_cast<RefStore*>(st)->store;
        std::memset(info, 0, sizeof(*info));
        info->rows = b.rows();
        info->capacity = b.capacity();
        info->filled = b.filled();
        info->finalized = b.finalized_count();
        info->big_panel_start = b.big_panel_start();
        info->panel_size = b.panel_size();
        info->big_panel_size = b.big_panel_size();
        info->seam_valid = b.has_seam_column();
        info->big_panel_open = b.big_panel_open();
        info->big_panel_full = b.big_panel_full();
        info->n_records = static_cast<int64_t>(b.block_records().size());
        info->n_panel_states = static_cast<int64_t>(b.panel_states().size());
        info->ld = b.rows();
    });
}
int kref_store_coefficients(void* st, double* r) {
    return guarded([&] { copy_upper(static_cast<RefStore*>(st)->store.coefficients(), r); });
}
int kref_store_columns(void* st, int64_t first, int64_t count, double* out) {
    return guarded([&] {
        RefStore* s = static_cast<RefStore*>(st);
        for (int64_t j = 0; j < count; ++j)
            std::memcpy(out + j * s->n, s->store.column(first + j), s->n * sizeof(double));
    });
}
int kref_store_panel_states(void* st, int32_t* states) {
    return guarded([&] {
        const auto& ps = static_cast<RefStore*>(st)->store.panel_states();
        for (size_t i = 0; i < ps.size(); ++i) states[i] = static_cast<int32_t>(ps[i]);
    });
}
int kref_store_block_record(void* st, int64_t idx, int64_t* c0, int64_t* width, int32_t* overlap,
                            double* carried, double* carried_diag) {
    return guarded([&] {
        const BlockRecord& r = static_cast<RefStore*>(st)->store.block_records().at(idx);
        *c0 = r.c0;
        *width = r.width;
        *overlap = r.overlap;
        if (carried)
            for (size_t i = 0; i < r.carried.size(); ++i) carried[i] = r.carried[i];
        *carried_diag = r.carried_diag;
    });
}
int kref_store_hessenberg(void* st, int64_t k, double* h) {
    return guarded([&] {
        const BasisStore& b = static_cast<RefStore*>(st)->store;
        DenseMatrix hh = assemble_hessenberg(b.coefficients(), ChangeOfBasis::monomial(k), k,
                                             b.block_records());
        copy_mat(hh, h);
    });
}
int kref_hessenberg_lsq(int64_t k, const double* h, double gamma, double* y, double* implicit,
                        int64_t* valid) {
    return guarded([&] {
        LsqResult l = solve_hessenberg_lsq(ConstMatrixView(h, k + 1, k), gamma);
        for (size_t i = 0; i < l.y.size(); ++i) y[i] = l.y[i];
        *implicit = l.implicit_residual;
        *valid = static_cast<int64_t>(l.valid_cols);
    });
}

// ---- solver (gmres.hpp) -----------------------------------------------------
int kref_sstep_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b,
                     const double* x0, const kry_solver_config* cfg, kry_report* report,
                     double* x_out) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, rp, ci, v);
        std::span<const double> x0s = x0 ? std::span<const double>(x0, n) : std::span<const double>();
        SolveReport rep = sstep_gmres(a, std::span<const double>(b, n), x0s, make_cfg(cfg));
        fill_report(rep, report);
        if (x_out) std::memcpy(x_out, rep.solution.data(), n * sizeof(double));
    });
}
int kref_standard_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        const double* b, const double* x0, const kry_solver_config* cfg,
                        kry_report* report, double* x_out) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, rp, ci, v);
        std::span<const double> x0s = x0 ? std::span<const double>(x0, n) : std::span<const double>();
        SolveReport rep = standard_gmres(a, std::span<const double>(b, n), x0s, make_cfg(cfg));
        fill_report(rep, report);
        if (x_out) std::memcpy(x_out, rep.solution.data(), n * sizeof(double));
    });
}

}  // extern "C"
