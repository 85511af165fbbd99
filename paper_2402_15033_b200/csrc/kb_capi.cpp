// extern "C" boundary (include/krylov_b200.h).  Every entry point binds the
// context's device, runs the C++ implementation and converts kb::Error into
// a status code; nothing throws across the ABI.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>

#include "kb_ctx.hpp"
#include "kb_dense.hpp"
#include "kb_gmres.hpp"
#include "kb_operator.hpp"
#include "kb_ortho.hpp"
#include "kb_store.hpp"

using kb::i64;

struct kry_ctx {
    std::unique_ptr<kb::Ctx> c;
    kb::DevBuf up0, up1, up2;  // staging for host-view entry points
    kb::Workspace ws;          // solver workspace reused across solves (destroyed before c)
};
struct kry_operator {
    std::unique_ptr<kb::Operator> op;
    kry_ctx* owner;
};
struct kry_store {
    std::unique_ptr<kb::Store> st;
    kry_ctx* owner;
    kb::DevBuf upload;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f, int64_t* aux = nullptr) {
    try {
        f();
        return KRY_OK;
    } catch (const kb::Error& e) {
        g_last_error = e.what();
        if (aux) *aux = e.aux;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return KRY_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return KRY_INTERNAL;
    }
}

kb::Ctx& C(kry_ctx* ctx) {
    if (!ctx || !ctx->c) kb::fail(KRY_INVALID_ARGUMENT, "null context");
    kb::bind_device(*ctx->c);
    return *ctx->c;
}

size_t mat_bytes(i64 ld, i64 cols) { return static_cast<size_t>(ld) * static_cast<size_t>(cols) * 8; }

// Host n×k (ld == n) → device buffer with ld = device_ld(n).
double* upload(kb::Ctx& c, kb::DevBuf& buf, const double* h, i64 n, i64 k) {
    const i64 ld = kb::device_ld(n);
    buf.ensure(std::max<size_t>(mat_bytes(ld, k), 8));
    if (k > 0 && h)
        KB_CUDA(cudaMemcpy2DAsync(buf.p, ld * 8, h, n * 8, n * 8, k, cudaMemcpyHostToDevice, c.stream));
    return buf.p;
}

void download(kb::Ctx& c, double* h, const double* d, i64 ld, i64 n, i64 k) {
    if (k > 0 && h)
        KB_CUDA(cudaMemcpy2DAsync(h, n * 8, d, ld * 8, n * 8, k, cudaMemcpyDeviceToHost, c.stream));
}

void put_mat(const kb::Mat& m, double* out) {
    if (out && !m.a.empty()) std::memcpy(out, m.a.data(), m.a.size() * 8);
}
void put_upper(const kb::Upper& u, double* out) {
    if (out && !u.a.empty()) std::memcpy(out, u.a.data(), u.a.size() * 8);
}

void fill_outcome(const kb::Outcome& o, kry_append_outcome* out) {
    if (!out) return;
    out->committed = o.committed;
    out->truncated = o.truncated ? 1 : 0;
    out->breakdown = o.breakdown ? 1 : 0;
    out->pivot = o.pivot;
    out->kappa_estimate = o.kappa_estimate;
}

void fill_report(const kb::Report& r, kry_report* out) {
    if (!out) return;
    out->status = r.status;
    out->breakdown = r.breakdown ? 1 : 0;
    out->iterations = r.iterations;
    out->restarts = r.restarts;
    out->initial_residual = r.initial_residual;
    out->final_relative_residual = r.final_relative_residual;
    out->breakdown_kappa = r.breakdown_kappa;
    out->reduces = r.sync.reduces;
    out->reduces_per_iteration = r.reduces_per_iteration;
    out->wall_seconds = r.wall_seconds;
    out->n_cycle_residuals = static_cast<int64_t>(r.cycle_residuals.size());
    for (int64_t i = 0; i < out->n_cycle_residuals && i < out->cycle_residuals_cap; ++i)
        out->cycle_residuals[i] = r.cycle_residuals[i];
    out->n_per_block = static_cast<int64_t>(r.sync.per_block.size());
    for (int64_t i = 0; i < out->n_per_block && i < out->per_block_cap; ++i) out->per_block[i] = r.sync.per_block[i];
    out->n_per_big_panel = static_cast<int64_t>(r.sync.per_big_panel.size());
    for (int64_t i = 0; i < out->n_per_big_panel && i < out->per_big_panel_cap; ++i)
        out->per_big_panel[i] = r.sync.per_big_panel[i];
    out->mpk_bytes = r.mpk_bytes;
    out->ortho_bytes = r.ortho_bytes;
}

struct Snapshot {
    std::array<double, kb::PH_COUNT> sec;
    int64_t launches, allreduces, gram_launches, update_launches, fused_launches;
    double gram_bytes, update_bytes, fused_bytes;
    explicit Snapshot(const kb::Ctx& c)
        : sec(c.seconds),
          launches(c.launches),
          allreduces(c.allreduces),
          gram_launches(c.gram_launches),
          update_launches(c.update_launches),
          gram_bytes(c.gram_bytes),
          update_bytes(c.update_bytes),
          fused_bytes(c.fused_bytes) {
        fused_launches = c.fused_launches;
    }
};

void fill_telemetry(const kb::Ctx& c, const Snapshot& s0, kry_report* out) {
    if (!out) return;
    out->mpk_seconds = c.seconds[kb::PH_MPK] - s0.sec[kb::PH_MPK];
    out->ortho_seconds = c.seconds[kb::PH_ORTHO] - s0.sec[kb::PH_ORTHO];
    out->gram_kernel_seconds = c.seconds[kb::PH_GRAM] - s0.sec[kb::PH_GRAM];
    out->update_kernel_seconds = c.seconds[kb::PH_UPDATE] - s0.sec[kb::PH_UPDATE];
    out->restart_seconds = c.seconds[kb::PH_RESTART] - s0.sec[kb::PH_RESTART];
    out->gpu_launches = c.launches - s0.launches;
    out->allreduces = c.allreduces - s0.allreduces;
    out->gram_launches = c.gram_launches - s0.gram_launches;
    out->update_launches = c.update_launches - s0.update_launches;
    out->gram_bytes = c.gram_bytes - s0.gram_bytes;
    out->update_bytes = c.update_bytes - s0.update_bytes;
    out->fused_kernel_seconds = c.seconds[kb::PH_FUSED] - s0.sec[kb::PH_FUSED];
    out->fused_bytes = c.fused_bytes - s0.fused_bytes;
    out->fused_launches = c.fused_launches - s0.fused_launches;
}

// bcgs_pip on host views; returns the PipOut and writes q.
kb::PipOut pip_host(kry_ctx* ctx, i64 n, const double* qp, i64 c0, const double* v, i64 w, double* q,
                    int64_t* reduces) {
    kb::Ctx& c = C(ctx);
    kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "bcgs_pip shapes");
    const i64 ld = kb::device_ld(n);
    const double* dqp = upload(c, ctx->up0, qp, n, c0);
    const double* dv = upload(c, ctx->up1, v, n, w);
    ctx->up2.ensure(mat_bytes(ld, w));
    i64 red = 0;
    kb::PipOut o = kb::bcgs_pip_partial_device(c, n, dqp, ld, c0, dv, ld, w, ctx->up2.p, ld, red);
    if (reduces) *reduces += red;
    if (o.bad_pivot == 0) download(c, q, ctx->up2.p, ld, n, w);
    c.sync();
    return o;
}

}  // namespace

extern "C" {

int kry_abi_version(void) { return KRY_ABI_VERSION; }
const char* kry_last_error(void) { return g_last_error.c_str(); }

const char* kry_status_name(int s) {
    switch (s) {
        case KRY_OK: return "ok";
        case KRY_DIMENSION_MISMATCH: return "dimension_mismatch";
        case KRY_NOT_POSITIVE_DEFINITE: return "not_positive_definite";
        case KRY_SINGULAR_FACTOR: return "singular_factor";
        case KRY_SINGULAR_R: return "singular_r";
        case KRY_INVALID_ARGUMENT: return "invalid_argument";
        case KRY_UNSUPPORTED: return "unsupported";
        case KRY_CUDA_ERROR: return "cuda_error";
        case KRY_NCCL_ERROR: return "nccl_error";
        case KRY_NO_DEVICE: return "no_device";
        default: return "internal";
    }
}

void kry_solver_config_default(kry_solver_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->restart_len = 60;
    cfg->step = 5;
    cfg->big_step = 0;
    cfg->scheme_kind = KRY_ORTHO_BCGS_PIP2;
    cfg->scheme_big_panel_size = 0;
    cfg->rel_tol = 1e-6;
    cfg->max_iters = 500000;
}

int kry_device_count(int* count) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (count) *count = n;
    if (n == 0) {
        g_last_error = "no CUDA device visible";
        return KRY_NO_DEVICE;
    }
    return KRY_OK;
}

int kry_nccl_unique_id_size(void) { return static_cast<int>(sizeof(ncclUniqueId)); }

int kry_nccl_get_unique_id(void* out) {
    return guarded([&] {
        ncclUniqueId id;
        ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) kb::fail(KRY_NCCL_ERROR, ncclGetErrorString(r));
        std::memcpy(out, &id, sizeof(id));
    });
}

int kry_ctx_create(int device, int nranks, int rank, const void* nccl_id, kry_ctx** out) {
    return guarded([&] {
        if (!out) kb::fail(KRY_INVALID_ARGUMENT, "null output");
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks) kb::fail(KRY_INVALID_ARGUMENT, "bad rank layout");
        auto* k = new kry_ctx;
        try {
            k->c = std::make_unique<kb::Ctx>(device, nranks, rank, nccl_id);
        } catch (...) {
            delete k;
            throw;
        }
        *out = k;
    });
}

int kry_ctx_destroy(kry_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        if (ctx->c) kb::bind_device(*ctx->c);
        ctx->ws.store.reset();
        delete ctx;
    });
}

int kry_ctx_synchronize(kry_ctx* ctx) { return guarded([&] { C(ctx).sync(); }); }
int kry_ctx_set_timing(kry_ctx* ctx, int enabled) { return guarded([&] { C(ctx).timing = enabled != 0; }); }
int kry_ctx_launch_count(kry_ctx* ctx, int64_t* launches) {
    return guarded([&] { *launches = C(ctx).launches; });
}
int kry_ctx_rank(kry_ctx* ctx, int* rank, int* nranks) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        if (rank) *rank = c.rank;
        if (nranks) *nranks = c.nranks;
    });
}

int kry_ctx_stream(kry_ctx* ctx, void** stream) {
    return guarded([&] { *stream = static_cast<void*>(C(ctx).stream); });
}

// ---- operators -------------------------------------------------------------
int kry_operator_create_csr(kry_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t n_local,
                            const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                            kry_operator** out) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        auto* o = new kry_operator;
        o->owner = ctx;
        try {
            o->op.reset(kb::make_csr(c, n_global, row_begin, n_local, row_ptr, col_idx, vals));
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

int kry_operator_create_laplace2d(kry_ctx* ctx, int64_t nx, int64_t ny, kry_operator** out) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        auto* o = new kry_operator;
        o->owner = ctx;
        try {
            o->op.reset(kb::make_laplace(c, 2, nx, ny, 1));
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

int kry_operator_create_laplace3d(kry_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, kry_operator** out) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        auto* o = new kry_operator;
        o->owner = ctx;
        try {
            o->op.reset(kb::make_laplace(c, 3, nx, ny, nz));
        } catch (...) {
            delete o;
            throw;
        }
        *out = o;
    });
}

int kry_laplace_partition(int dims, int64_t nx, int64_t ny, int64_t nz, int nranks, int rank, int64_t* row_begin,
                          int64_t* n_local, int64_t* halo) {
    return guarded([&] {
        if (dims != 2 && dims != 3) kb::fail(KRY_INVALID_ARGUMENT, "dims must be 2 or 3");
        i64 rb = 0, nl = 0, h = 0;
        kb::laplace_partition(dims, nx, ny, dims == 2 ? 1 : nz, nranks, rank, rb, nl, h);
        *row_begin = rb;
        *n_local = nl;
        *halo = h;
    });
}

int kry_operator_destroy(kry_operator* op) {
    return guarded([&] {
        if (!op) return;
        if (op->owner && op->owner->c) kb::bind_device(*op->owner->c);
        delete op;
    });
}

int kry_operator_rows(const kry_operator* op, int64_t* n_global, int64_t* row_begin, int64_t* n_local) {
    return guarded([&] {
        if (n_global) *n_global = op->op->n_global;
        if (row_begin) *row_begin = op->op->row_begin;
        if (n_local) *n_local = op->op->nloc;
    });
}

int kry_operator_nnz(const kry_operator* op, int64_t* nnz_local) {
    return guarded([&] { *nnz_local = op->op->nnz_local; });
}

int kry_operator_jacobi(kry_operator* op) {
    return guarded([&] { op->op->set_jacobi(); });
}

int kry_operator_is_jacobi(const kry_operator* op, int* enabled) {
    return guarded([&] { *enabled = op->op->jacobi ? 1 : 0; });
}

int kry_gen_random_sparse(int64_t n_global, int64_t row_begin, int64_t n_local, int64_t per_row, uint64_t seed,
                          double diag_factor, int jacobi, int64_t* row_ptr, int64_t* col_idx, double* vals) {
    return guarded([&] {
        kb::gen_random_sparse(n_global, row_begin, n_local, per_row, seed, diag_factor, jacobi != 0, row_ptr,
                              col_idx, vals);
    });
}

int kry_spmv_device(kry_ctx* ctx, kry_operator* op, const double* d_x, double* d_y) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        op->op->apply(d_x, d_y);
        c.sync();
    });
}

int kry_spmv(kry_ctx* ctx, kry_operator* op, const double* x, double* y) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        const i64 n = op->op->nloc;
        double* dx = upload(c, ctx->up0, x, n, 1);
        ctx->up1.ensure(static_cast<size_t>(kb::device_ld(n)) * 8);
        op->op->apply(dx, ctx->up1.p);
        download(c, y, ctx->up1.p, n, n, 1);
        c.sync();
    });
}

int kry_mpk(kry_ctx* ctx, kry_operator* op, const double* start, int64_t s, double* v) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        kb::dim_check(s >= 0, "mpk step count");
        const i64 n = op->op->nloc, ld = kb::device_ld(n);
        ctx->up0.ensure(mat_bytes(ld, s + 1));
        KB_CUDA(cudaMemcpyAsync(ctx->up0.p, start, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, c.stream));
        if (s == 0 || !op->op->mpk(ctx->up0.p, ctx->up0.p + ld, ld, static_cast<int>(s)))
            for (i64 k = 0; k < s; ++k) op->op->apply(ctx->up0.p + k * ld, ctx->up0.p + (k + 1) * ld);
        download(c, v, ctx->up0.p, ld, n, s + 1);
        c.sync();
    });
}

// ---- block orthogonalization --------------------------------------------------
int kry_gram(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
             double* r_col, double* g) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "gram shapes");
        const i64 ld = kb::device_ld(n);
        const double* dqp = upload(c, ctx->up0, q_prev, n, c0);
        const double* dv = upload(c, ctx->up1, v, n, w);
        kb::Mat rc, gg;
        kb::gram_device(c, n, dqp, ld, c0, dv, ld, w, rc, gg);
        put_mat(rc, r_col);
        put_mat(gg, g);
    });
}

int kry_gram_full(kry_ctx* ctx, int64_t n, const double* q, int64_t k, double* g) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        kb::dim_check(n >= 1 && k >= 1, "gram shapes");
        const i64 ld = kb::device_ld(n);
        const double* dq = upload(c, ctx->up1, q, n, k);
        kb::Mat rc, gg;
        kb::gram_device(c, n, nullptr, ld, 0, dq, ld, k, rc, gg);
        put_mat(gg, g);
    });
}

int kry_bcgs_pip_partial(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v,
                         int64_t w, double* q, double* r_col, double* r_chol, int64_t* bad_pivot,
                         int64_t* reduces) {
    return guarded([&] {
        kb::PipOut o = pip_host(ctx, n, q_prev, c0, v, w, q, reduces);
        put_mat(o.r_col, r_col);
        put_upper(o.r_jj, r_chol);
        if (bad_pivot) *bad_pivot = o.bad_pivot;
    });
}

int kry_bcgs_pip(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                 double* q, double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    if (pivot) *pivot = 0;
    return guarded(
        [&] {
            kb::PipOut o = pip_host(ctx, n, q_prev, c0, v, w, q, reduces);
            if (o.bad_pivot != 0)
                kb::fail(KRY_NOT_POSITIVE_DEFINITE,
                         "matrix not positive definite at pivot " + std::to_string(o.bad_pivot), o.bad_pivot);
            put_mat(o.r_col, r_col);
            put_upper(o.r_jj, r_jj);
        },
        pivot);
}

int kry_bcgs_pip2(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                  double* q, double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    if (pivot) *pivot = 0;
    return guarded(
        [&] {
            kb::Ctx& c = C(ctx);
            kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "bcgs_pip2 shapes");
            const i64 ld = kb::device_ld(n);
            const double* dqp = upload(c, ctx->up0, q_prev, n, c0);
            const double* dv = upload(c, ctx->up1, v, n, w);
            ctx->up2.ensure(mat_bytes(ld, w));
            i64 red = 0;
            auto throw_if = [&](const kb::PipOut& o) {
                if (o.bad_pivot != 0)
                    kb::fail(KRY_NOT_POSITIVE_DEFINITE,
                             "matrix not positive definite at pivot " + std::to_string(o.bad_pivot), o.bad_pivot);
            };
            kb::PipOut first = kb::bcgs_pip_partial_device(c, n, dqp, ld, c0, dv, ld, w, ctx->up2.p, ld, red);
            if (reduces) *reduces += red;
            red = 0;
            throw_if(first);
            kb::PipOut second =
                kb::bcgs_pip_partial_device(c, n, dqp, ld, c0, ctx->up2.p, ld, w, ctx->up2.p, ld, red);
            if (reduces) *reduces += red;
            throw_if(second);
            kb::Mat rc = first.r_col;
            if (rc.rows > 0) {
                kb::Mat r1(w, w);
                for (i64 j = 0; j < w; ++j)
                    for (i64 i = 0; i <= j; ++i) r1(i, j) = first.r_jj(i, j);
                kb::Mat corr = kb::mat_mul_nn(second.r_col, r1);
                for (i64 j = 0; j < rc.cols; ++j)
                    for (i64 i = 0; i < rc.rows; ++i) rc(i, j) += corr(i, j);
            }
            download(c, q, ctx->up2.p, ld, n, w);
            c.sync();
            put_mat(rc, r_col);
            put_upper(kb::tri_mul(second.r_jj, first.r_jj), r_jj);
        },
        pivot);
}

int kry_cholqr(kry_ctx* ctx, int64_t n, const double* v, int64_t w, double* q, double* r, int64_t* pivot,
               int64_t* reduces) {
    // cholqr (block_ortho.hpp:49-54) == bcgs_pip with an empty prefix.
    return kry_bcgs_pip(ctx, n, nullptr, 0, v, w, q, nullptr, r, pivot, reduces);
}

// BCGS2 pieces on the device (block_ortho.hpp:57-137).
int kry_cholqr2(kry_ctx* ctx, int64_t n, const double* v, int64_t w, double* q, double* r, int64_t* pivot,
                int64_t* reduces) {
    if (pivot) *pivot = 0;
    return guarded(
        [&] {
            kb::Ctx& c = C(ctx);
            kb::dim_check(n >= 1 && w >= 1, "cholqr2 shapes");
            const i64 ld = kb::device_ld(n);
            const double* dv = upload(c, ctx->up1, v, n, w);
            ctx->up2.ensure(mat_bytes(ld, w));
            i64 red = 0;
            double bytes = 0.0;
            try {
                kb::Upper r1 = kb::cholqr_device(c, n, dv, ld, w, ctx->up2.p, ld, red, bytes);
                kb::Upper r2 = kb::cholqr_device(c, n, ctx->up2.p, ld, w, ctx->up2.p, ld, red, bytes);
                if (reduces) *reduces += red;
                download(c, q, ctx->up2.p, ld, n, w);
                c.sync();
                put_upper(kb::tri_mul(r2, r1), r);
            } catch (const kb::CholFail& f) {
                if (reduces) *reduces += red;
                kb::fail(KRY_NOT_POSITIVE_DEFINITE, "matrix not positive definite at pivot " + std::to_string(f.pivot),
                         f.pivot);
            }
        },
        pivot);
}

int kry_bcgs_project(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                     double* vhat, double* r_block, int64_t* reduces) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "bcgs_project shapes");
        const i64 ld = kb::device_ld(n);
        const double* dqp = upload(c, ctx->up0, q_prev, n, c0);
        const double* dv = upload(c, ctx->up1, v, n, w);
        ctx->up2.ensure(mat_bytes(ld, w));
        i64 red = 0;
        double bytes = 0.0;
        kb::Mat rb = kb::project_device(c, n, dqp, ld, c0, dv, ld, w, ctx->up2.p, ld, red, bytes);
        if (reduces) *reduces += red;
        download(c, vhat, ctx->up2.p, ld, n, w);
        c.sync();
        put_mat(rb, r_block);
    });
}

int kry_bcgs2(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
              int32_t intra_kind, double* q, double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces) {
    if (pivot) *pivot = 0;
    return guarded(
        [&] {
            kb::Ctx& c = C(ctx);
            kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "bcgs2 shapes");
            if (intra_kind != 0 && intra_kind != 1) kb::fail(KRY_INVALID_ARGUMENT, "bcgs2: unknown intra kind");
            if (intra_kind == 0 && w > 1)
                kb::fail(KRY_UNSUPPORTED, "BCGS2 with a Householder intra step is not on the device path");
            const i64 ld = kb::device_ld(n);
            const double* dqp = upload(c, ctx->up0, q_prev, n, c0);
            const double* dv = upload(c, ctx->up1, v, n, w);
            ctx->up2.ensure(mat_bytes(ld, 3 * w));  // out | s0 | s1
            double* out = ctx->up2.p;
            i64 red = 0;
            double bytes = 0.0;
            try {
                kb::Bcgs2Out o = kb::bcgs2_device(c, n, dqp, ld, c0, dv, ld, w, out + ld * w, out + 2 * ld * w, ld,
                                                  out, ld, red, bytes);
                if (reduces) *reduces += red;
                download(c, q, out, ld, n, w);
                c.sync();
                put_mat(o.r_col, r_col);
                put_upper(o.r_jj, r_jj);
            } catch (const kb::CholFail& f) {
                if (reduces) *reduces += red;
                kb::fail(KRY_NOT_POSITIVE_DEFINITE, "matrix not positive definite at pivot " + std::to_string(f.pivot),
                         f.pivot);
            }
        },
        pivot);
}

int kry_bcgs_pip_device(kry_ctx* ctx, int64_t n, const double* d_q_prev, int64_t ldq, int64_t c0,
                        const double* d_v, int64_t ldv, int64_t w, double* d_out, int64_t ldo, double* r_col,
                        double* r_jj, int64_t* pivot, int64_t* reduces) {
    if (pivot) *pivot = 0;
    return guarded(
        [&] {
            kb::Ctx& c = C(ctx);
            kb::dim_check(n >= 1 && w >= 1 && c0 >= 0, "bcgs_pip shapes");
            auto aligned = [](const void* p, i64 ld) {
                return p == nullptr || ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld & 1) == 0);
            };
            if (!aligned(d_q_prev, ldq) || !aligned(d_v, ldv) || !aligned(d_out, ldo))
                kb::fail(KRY_INVALID_ARGUMENT, "device operands need 16-byte aligned columns (even ld)");
            i64 red = 0;
            kb::PipOut o = kb::bcgs_pip_partial_device(c, n, d_q_prev, ldq, c0, d_v, ldv, w, d_out, ldo, red);
            if (reduces) *reduces += red;
            c.sync();
            if (o.bad_pivot != 0)
                kb::fail(KRY_NOT_POSITIVE_DEFINITE,
                         "matrix not positive definite at pivot " + std::to_string(o.bad_pivot), o.bad_pivot);
            put_mat(o.r_col, r_col);
            put_upper(o.r_jj, r_jj);
        },
        pivot);
}

int kry_try_cholesky(int64_t k, const double* s, double* r, int64_t* pivot) {
    return guarded([&] {
        kb::Mat sm(k, k);
        std::memcpy(sm.a.data(), s, static_cast<size_t>(k * k) * 8);
        kb::Upper rr;
        *pivot = kb::try_cholesky(sm, rr);
        put_upper(rr, r);
    });
}

int kry_hessenberg_lsq(int64_t k, const double* h, double gamma, double* y, double* implicit_residual,
                       int64_t* valid_cols) {
    return guarded([&] {
        kb::Mat hm(k + 1, k);
        std::memcpy(hm.a.data(), h, static_cast<size_t>((k + 1) * k) * 8);
        kb::Lsq l = kb::solve_hessenberg_lsq(hm, gamma);
        for (size_t i = 0; i < l.y.size(); ++i) y[i] = l.y[i];
        *implicit_residual = l.implicit_residual;
        *valid_cols = l.valid_cols;
    });
}

// ---- basis store ---------------------------------------------------------------
int kry_store_create(kry_ctx* ctx, int64_t n, int64_t m, int64_t panel_size, int64_t big_panel_size,
                     kry_store** out) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        kb::dim_check(n >= 1 && m >= 1, "store shape");
        auto* s = new kry_store;
        s->owner = ctx;
        try {
            s->st = std::make_unique<kb::Store>(c, n, m, panel_size, big_panel_size);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

int kry_store_destroy(kry_store* st) {
    return guarded([&] {
        if (!st) return;
        if (st->owner && st->owner->c) kb::bind_device(*st->owner->c);
        delete st;
    });
}

int kry_store_reset(kry_store* st) {
    return guarded([&] {
        C(st->owner);
        st->st->reset();
        st->st->zero_q();
    });
}

int kry_store_seed_unit_column(kry_store* st, const double* v) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        double* dv = upload(c, st->upload, v, st->st->rows(), 1);
        st->st->seed_unit_column(dv);
        c.sync();
    });
}

int kry_store_append_block(kry_store* st, const double* v, int64_t w, int overlap, int32_t scheme_kind,
                           int64_t big_panel_size, kry_append_outcome* out, int64_t* reduces_delta) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        kb::dim_check(w >= 1, "block width");
        double* dv = upload(c, st->upload, v, st->st->rows(), w);
        kb::Sync sync;
        kb::Outcome o = st->st->append_block(dv, kb::device_ld(st->st->rows()), w, overlap != 0, scheme_kind,
                                             big_panel_size, sync);
        c.sync();
        fill_outcome(o, out);
        if (reduces_delta) *reduces_delta = sync.reduces;
    });
}

int kry_store_preprocess_block(kry_store* st, const double* v, int64_t w, int overlap, kry_append_outcome* out,
                               int64_t* reduces_delta) {
    return kry_store_append_block(st, v, w, overlap, KRY_ORTHO_TWO_STAGE, st ? st->st->big_panel_size() : 0, out,
                                  reduces_delta);
}

int kry_store_finalize_big_panel(kry_store* st, kry_append_outcome* out, int64_t* reduces_delta) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        kb::Sync sync;
        kb::Outcome o = st->st->finalize_big_panel(sync);
        c.sync();
        fill_outcome(o, out);
        if (reduces_delta) *reduces_delta = sync.reduces;
    });
}

int kry_store_mpk(kry_store* st, kry_operator* op, const double* start, int64_t c0, int64_t s) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        kb::dim_check(op->op->nloc == st->st->rows(), "operator rows");
        kb::dim_check(c0 >= 0 && c0 + s + 1 <= st->st->capacity(), "basis store capacity exceeded");
        if (start)
            KB_CUDA(cudaMemcpyAsync(st->st->col(c0), start, static_cast<size_t>(st->st->rows()) * 8,
                                    cudaMemcpyHostToDevice, c.stream));
        st->st->mpk(*op->op, c0, s);
        c.sync();
    });
}

int kry_store_append_inplace(kry_store* st, int64_t w, int overlap, int32_t scheme_kind, int64_t big_panel_size,
                             kry_append_outcome* out, int64_t* reduces_delta) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        kb::Store& s = *st->st;
        if (overlap && s.filled() == 0) kb::fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: basis store capacity exceeded");
        const i64 c0 = overlap ? s.filled() - 1 : s.filled();
        kb::dim_check(c0 + w <= s.capacity(), "basis store capacity exceeded");
        kb::Sync sync;
        kb::Outcome o = s.append_block(s.col(c0), s.ld(), w, overlap != 0, scheme_kind, big_panel_size, sync);
        c.sync();
        fill_outcome(o, out);
        if (reduces_delta) *reduces_delta = sync.reduces;
    });
}

int kry_store_get_info(kry_store* st, kry_store_info* info) {
    return guarded([&] {
        const kb::Store& s = *st->st;
        std::memset(info, 0, sizeof(*info));
        info->rows = s.rows();
        info->capacity = s.capacity();
        info->filled = s.filled();
        info->finalized = s.finalized_count();
        info->big_panel_start = s.big_panel_start();
        info->panel_size = s.panel_size();
        info->big_panel_size = s.big_panel_size();
        info->seam_valid = s.has_seam_column();
        info->big_panel_open = s.big_panel_open();
        info->big_panel_full = s.big_panel_full();
        info->n_records = static_cast<int64_t>(s.block_records().size());
        info->n_panel_states = static_cast<int64_t>(s.panel_states().size());
        info->ld = s.ld();
    });
}

int kry_store_coefficients(kry_store* st, double* r) {
    return guarded([&] { put_upper(st->st->coefficients(), r); });
}

int kry_store_columns(kry_store* st, int64_t first, int64_t count, double* out) {
    return guarded([&] {
        kb::Ctx& c = C(st->owner);
        kb::Store& s = *st->st;
        kb::dim_check(first >= 0 && count >= 0 && first + count <= s.capacity(), "column range");
        download(c, out, s.col(first), s.ld(), s.rows(), count);
        c.sync();
    });
}

int kry_store_column(kry_store* st, int64_t j, double* out) { return kry_store_columns(st, j, 1, out); }

int kry_store_panel_states(kry_store* st, int32_t* states) {
    return guarded([&] {
        const auto& ps = st->st->panel_states();
        for (size_t i = 0; i < ps.size(); ++i) states[i] = ps[i];
    });
}

int kry_store_block_record(kry_store* st, int64_t index, int64_t* c0, int64_t* width, int32_t* overlap,
                           double* carried, double* carried_diag) {
    return guarded([&] {
        const auto& recs = st->st->block_records();
        kb::dim_check(index >= 0 && index < static_cast<int64_t>(recs.size()), "record index");
        const kb::BlockRecord& r = recs[index];
        *c0 = r.c0;
        *width = r.width;
        *overlap = r.overlap ? 1 : 0;
        if (carried)
            for (size_t i = 0; i < r.carried.size(); ++i) carried[i] = r.carried[i];
        *carried_diag = r.carried_diag;
    });
}

int kry_store_check_guards(kry_store* st) {
    return guarded([&] { st->st->check_guards(); });
}

int kry_store_device_ptr(kry_store* st, double** d_q, int64_t* ld) {
    return guarded([&] {
        *d_q = st->st->col(0);
        *ld = st->st->ld();
    });
}

int kry_store_hessenberg(kry_store* st, int64_t k, double* h, int64_t* singular_column) {
    return guarded(
        [&] {
            kb::Mat hm = kb::assemble_hessenberg(st->st->coefficients(), k, st->st->block_records());
            put_mat(hm, h);
        },
        singular_column);
}

// ---- solver ----------------------------------------------------------------------
static int solve_common(kry_ctx* ctx, kry_operator* op, const double* b, const double* x0,
                        const kry_solver_config* cfg, kry_report* report, double* x_out, bool device,
                        bool standard) {
    return guarded([&] {
        kb::Ctx& c = C(ctx);
        if (!op || !cfg) kb::fail(KRY_INVALID_ARGUMENT, "null operator or config");
        const i64 n = op->op->nloc;
        Snapshot snap(c);
        kb::Report rep;
        if (device) {
            rep = kb::gmres(c, *op->op, b, x0, *cfg, standard, x_out, &ctx->ws);
        } else {
            double* db = upload(c, ctx->up0, b, n, 1);
            double* dx0 = x0 ? upload(c, ctx->up1, x0, n, 1) : nullptr;
            // the solution streams to x_out while the last update is computed
            rep = kb::gmres(c, *op->op, db, dx0, *cfg, standard, nullptr, &ctx->ws, x_out);
            c.sync();
        }
        fill_report(rep, report);
        fill_telemetry(c, snap, report);
    });
}

int kry_sstep_gmres(kry_ctx* ctx, kry_operator* op, const double* b, const double* x0, const kry_solver_config* cfg,
                    kry_report* report, double* x_out) {
    return solve_common(ctx, op, b, x0, cfg, report, x_out, false, false);
}

int kry_standard_gmres(kry_ctx* ctx, kry_operator* op, const double* b, const double* x0,
                       const kry_solver_config* cfg, kry_report* report, double* x_out) {
    return solve_common(ctx, op, b, x0, cfg, report, x_out, false, true);
}

int kry_sstep_gmres_device(kry_ctx* ctx, kry_operator* op, const double* d_b, const double* d_x0,
                           const kry_solver_config* cfg, kry_report* report, double* d_x_out) {
    return solve_common(ctx, op, d_b, d_x0, cfg, report, d_x_out, true, false);
}

int kry_standard_gmres_device(kry_ctx* ctx, kry_operator* op, const double* d_b, const double* d_x0,
                              const kry_solver_config* cfg, kry_report* report, double* d_x_out) {
    return solve_common(ctx, op, d_b, d_x0, cfg, report, d_x_out, true, true);
}

}  // extern "C"
