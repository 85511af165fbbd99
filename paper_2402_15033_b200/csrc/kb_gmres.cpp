#include "kb_gmres.hpp"

#include <cstdio>

#include <chrono>
#include <cmath>
#include <limits>
#include <cstdlib>
#include <string>
#include <utility>

namespace kb {

void validate_config(const kry_solver_config& c) {
    // SolverConfig::validate (gmres.hpp:28-35)
    if (c.restart_len <= 0 || c.step <= 0 || c.restart_len % c.step != 0)
        fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: step size must divide the restart length");
    const i64 shat = c.big_step == 0 ? c.restart_len : c.big_step;
    if (shat < c.step || shat > c.restart_len || shat % c.step != 0)
        fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: second step size must be a multiple of s in [s, m]");
    if (!(c.rel_tol > 0.0)) fail(KRY_INVALID_ARGUMENT, "rel_tol must be positive");
}

namespace {

struct Vec {
    DevBuf buf;
    double* p() const { return buf.p; }
};

}  // namespace

Workspace::~Workspace() {
    for (cudaEvent_t e : chunk_ev)
        if (e) cudaEventDestroy(e);
    if (copy_done) cudaEventDestroy(copy_done);
    if (copy_stream) cudaStreamDestroy(copy_stream);
}

namespace {
struct L2Window {
    Ctx& ctx;
    bool set = false;
    size_t prev_limit = 0;
    L2Window(Ctx& c, const double* q, i64 ld) : ctx(c) {
        const char* e = std::getenv("KRY_L2_PERSIST");
        if (e && std::atoi(e) == 0) return;
        int dev = 0, maxwin = 0, maxpersist = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        const size_t col = static_cast<size_t>(ld) * 8;
        const size_t cap = std::min<size_t>(static_cast<size_t>(maxpersist), static_cast<size_t>(maxwin));
        if (cap == 0 || 2 * col > cap) return;  // fewer than two columns would fit: no gain
        const size_t bytes = cap / col * col;
        if (cudaDeviceGetLimit(&prev_limit, cudaLimitPersistingL2CacheSize) != cudaSuccess ||
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = const_cast<double*>(q);
        v.accessPolicyWindow.num_bytes = bytes;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        if (cudaStreamSetAttribute(ctx.stream, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        set = true;
    }
    ~L2Window() {
        if (!set) return;
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(ctx.stream, cudaStreamAttributeAccessPolicyWindow, &v);
        cudaCtxResetPersistingL2Cache();
        // give the set-aside back: later solves (and other work) get the whole L2
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_limit);
    }
};
}  // namespace

Report gmres(Ctx& ctx, Operator& op, const double* d_b_in, const double* d_x0, const kry_solver_config& cfg_in,
             bool standard_mode, double* d_x_out, Workspace* ws, double* h_x_out) {
    kry_solver_config cfg = cfg_in;
    if (standard_mode) {  // standard_gmres (gmres.hpp:404-411)
        cfg.step = 1;
        cfg.big_step = 0;
        cfg.scheme_kind = KRY_ORTHO_BCGS2_CHOLQR2;
        cfg.scheme_big_panel_size = 0;
    }
    validate_config(cfg);
    const auto t_start = std::chrono::steady_clock::now();
    const auto prof_t0 = t_start;
    const int64_t prof_syncs0 = ctx.sync_count, prof_launch0 = ctx.launches;
    const double prof_wait0 = ctx.sync_wait_s;
    const i64 n = op.nloc;
    const i64 m = cfg.restart_len;
    const i64 s = standard_mode ? 1 : cfg.step;
    const bool two_stage = (cfg.scheme_kind == KRY_ORTHO_TWO_STAGE) && !standard_mode;
    const i64 shat = two_stage ? (cfg.big_step == 0 ? m : cfg.big_step) : s;

    Report rep;
    const size_t vbytes = static_cast<size_t>(device_ld(n)) * 8;
    Workspace local;
    Workspace& W = ws ? *ws : local;
    if (W.n != n || W.m != m || W.s != s || W.shat != shat) {
        W.store.reset();
        W.n = n;
        W.m = m;
        W.s = s;
        W.shat = shat;
    }
    DevBuf &x = W.x, &xn = W.xn, &r = W.r, &rn = W.rn;
    // Left Jacobi: the operator is D⁻¹A, the system D⁻¹A x = D⁻¹b.
    const double* d_b = op.scaled_rhs(d_b_in, W.bj);
    x.ensure(vbytes);
    xn.ensure(vbytes);
    r.ensure(vbytes);
    rn.ensure(vbytes);
    if (d_x0)
        KB_CUDA(cudaMemcpyAsync(x.p, d_x0, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    else
        KB_CUDA(cudaMemsetAsync(x.p, 0, vbytes, ctx.stream));

    // r = b − A·x and ‖r‖ in one fused pass (K9).  The norm of the current
    // r is cached: the reference recomputes norm2(r) on the same vector.
    auto residual = [&](const double* xv, double* rv) -> double {
        cudaEvent_t t0 = ctx.begin_phase();
        const int cnt = op.apply(xv, rv, d_b);
        const double sq = ctx.finalize_scalar(op.partials.p, cnt);
        ctx.end_phase(PH_RESTART, t0);
        return std::sqrt(sq);
    };
    double r_norm = residual(x.p, r.p);
    const double r0 = r_norm;
    rep.initial_residual = r0;
    // Host output: h_x_out holds x once copy_done has fired, when host_x_ok.
    bool host_x_ok = false;
    if (h_x_out && !W.copy_stream) {
        KB_CUDA(cudaStreamCreateWithFlags(&W.copy_stream, cudaStreamNonBlocking));
        for (cudaEvent_t& e : W.chunk_ev) KB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        KB_CUDA(cudaEventCreateWithFlags(&W.copy_done, cudaEventDisableTiming));
    }
    // Every exit (including an exception from SingularR, NCCL or CUDA) waits
    // for the chunked solution copies: the ABI must not return while DMA is
    // still writing the caller's buffer.
    struct CopyGuard {
        cudaStream_t s;
        ~CopyGuard() {
            if (s) cudaStreamSynchronize(s);
        }
    } copy_guard{h_x_out ? W.copy_stream : nullptr};
    auto finish = [&]() {
        if (d_x_out)
            KB_CUDA(cudaMemcpyAsync(d_x_out, x.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, ctx.stream));
        if (h_x_out) {
            if (host_x_ok) {
                KB_CUDA(cudaStreamWaitEvent(ctx.stream, W.copy_done, 0));
            } else {  // no (accepted) update streamed out: download x now
                KB_CUDA(cudaStreamWaitEvent(ctx.stream, W.copy_done, 0));  // (an in-flight copy of a rejected update)
                KB_CUDA(cudaMemcpyAsync(h_x_out, x.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx.stream));
            }
        }
        ctx.sync();
        ctx.resolve_timers();
        rep.wall_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    };
    if (r0 == 0.0) {
        rep.status = KRY_STATUS_CONVERGED;
        finish();
        return rep;
    }

    {
        const char* e = std::getenv("KRY_GUARD");
        const bool want_guard = e && std::atoi(e) == 1;
        if (W.store && W.store->guarded() != want_guard) W.store.reset();
    }
    if (!W.store) W.store = std::make_unique<Store>(ctx, n, m, s, shat);
    Store& store = *W.store;
    // Small grids: the basis prefix is re-read by every block's Gram and
    // update (twice per block), and at 512² the whole store (128 MB) is about
    // the size of L2 — an LRU sweep over it misses almost every line.  Pin
    // the leading columns in L2 with a persisting access-policy window on the
    // solver stream (KRY_L2_PERSIST=0 disables); released on every exit.
    L2Window l2win(ctx, store.col(0), store.ld());
    store.ortho_bytes = 0.0;
    const int scheme = cfg.scheme_kind;

    auto usable_cols = [&]() -> i64 {
        i64 k = store.filled() == 0 ? 0 : store.filled() - 1;
        if (store.has_seam_column()) ++k;
        const Upper& rr = store.coefficients();
        for (i64 j = 0; j < k; ++j)
            if (rr(j, j) == 0.0) return j;
        return k;
    };

    struct Check {
        bool implicit_crossed = false;
        bool applied = false;
        double explicit_rel = std::numeric_limits<double>::infinity();
    };

    // gmres.hpp:247-269
    // The unforced check after a cycle's last block and the forced one that
    // follows it see the same store: the host H / LSQ of the first is reused.
    double lsq_seconds = 0.0;  // host H assembly + LSQ (KRY_HOST_PROFILE)
    struct LsqCache {
        i64 reduces = -1, filled = -1;
        double gamma = 0.0;
        Lsq lsq;
        std::vector<double> ycoef;
    } cache;
    auto check_and_update = [&](double gamma, bool force) -> Check {
        Check res;
        const i64 k = usable_cols();
        if (k == 0) return res;
        if (!(cache.reduces == rep.sync.reduces && cache.filled == store.filled() && cache.gamma == gamma)) {
            const auto th = std::chrono::steady_clock::now();
            Mat h = assemble_hessenberg(store.coefficients(), k, store.block_records());
            cache.lsq = solve_hessenberg_lsq(h, gamma);
            if (ctx.host_profile)
                lsq_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - th).count();
            // A deferred last-panel finalize: the same x update over the stored
            // (preprocessed) columns with transformed coefficients.
            if (!store.deferred_coefficients(cache.lsq.y, cache.ycoef)) cache.ycoef = cache.lsq.y;
            cache.reduces = rep.sync.reduces;
            cache.filled = store.filled();
            cache.gamma = gamma;
        }
        const Lsq& lsq = cache.lsq;
        const std::vector<double>& ycoef = cache.ycoef;
        res.implicit_crossed = lsq.implicit_residual <= cfg.rel_tol * r0;
        if (!res.implicit_crossed && !force) return res;
        NvtxRange nv("kry.solution_update");

        cudaEvent_t t0 = ctx.begin_phase();
        // x_new = x + Q·y in row chunks; with a host output each chunk is
        // copied out on the side stream as soon as it is written
        const int nchunk = h_x_out ? 8 : 1;  // ≤ chunk_ev
        if (h_x_out) KB_CUDA(cudaStreamWaitEvent(ctx.stream, W.copy_done, 0));  // xn may still be going out
        for (int ch = 0; ch < nchunk; ++ch) {
            const i64 r0c = n * ch / nchunk, r1c = n * (ch + 1) / nchunk;
            const double* src = x.p + r0c;
            if (lsq.valid_cols == 0)
                KB_CUDA(cudaMemcpyAsync(xn.p + r0c, src, static_cast<size_t>(r1c - r0c) * 8, cudaMemcpyDeviceToDevice,
                                        ctx.stream));
            for (i64 l0 = 0; l0 < lsq.valid_cols; l0 += 64) {
                Coef64 y{};
                const int cnt = static_cast<int>(std::min<i64>(64, lsq.valid_cols - l0));
                for (int i = 0; i < cnt; ++i) y.v[i] = ycoef[l0 + i];
                launch_xupdate(ctx.stream, r1c - r0c, src, store.col(l0) + r0c, store.ld(), cnt, y, xn.p + r0c,
                               ctx.launches);
                src = xn.p + r0c;
            }
            if (h_x_out && r1c > r0c) {
                KB_CUDA(cudaEventRecord(W.chunk_ev[ch], ctx.stream));
                KB_CUDA(cudaStreamWaitEvent(W.copy_stream, W.chunk_ev[ch], 0));
                KB_CUDA(cudaMemcpyAsync(h_x_out + r0c, xn.p + r0c, static_cast<size_t>(r1c - r0c) * 8,
                                        cudaMemcpyDeviceToHost, W.copy_stream));
            }
        }
        if (h_x_out) KB_CUDA(cudaEventRecord(W.copy_done, W.copy_stream));
        rep.mpk_bytes += 0;  // the residual's SpMV is restart-loop traffic
        ctx.end_phase(PH_RESTART, t0);
        const double rnv = residual(xn.p, rn.p);
        res.explicit_rel = rnv / r0;
        if (rnv <= gamma * (1.0 + 1e-12)) {
            std::swap(x.p, xn.p);
            std::swap(r.p, rn.p);
            r_norm = rnv;
            res.applied = true;
            host_x_ok = h_x_out != nullptr;  // the copy going out is x
        } else {
            host_x_ok = false;  // the host got the rejected update
        }
        return res;
    };

    // Speculative queues replayed as CUDA graphs (one rank, no phase timing:
    // the recorded launches hold no events).  Opt-in (KRY_GRAPHS=1): at 512²
    // the cycle is bound by the kernels' own latencies, not by the host's
    // launch rate — 0.0838 vs 0.0835 s two-stage, 0.1275 vs 0.1277 s PIP2
    // (DESIGN.md §5), so the direct launches stay the default.
    const bool use_graphs = [] {
        const char* e = std::getenv("KRY_GRAPHS");
        return e && std::atoi(e) == 1;
    }() && ctx.nranks == 1 && !ctx.timing;
    if (use_graphs) {
        const char* fm = std::getenv("KRY_FUSED_MPK");
        const std::string sig = std::to_string(reinterpret_cast<uintptr_t>(&op)) + "/" +
                                std::to_string(op.geom.jacobi) + "/" + std::to_string(op.jacobi) + "/" +
                                (fm ? fm : "-") + "/" + std::to_string(cfg.scheme_kind) + "/" +
                                std::to_string(s) + "/" + std::to_string(shat);
        if (sig != W.graphs.sig) {
            W.graphs.clear();
            W.graphs.sig = sig;
        }
    }
    // body() enqueues a launch sequence (and does its host bookkeeping).
    // First time for `key`: record it (stream capture) and replay the graph;
    // later: run body() with the launches suppressed and replay the graph —
    // valid while no device buffer was reallocated since the recording.
    auto recorded = [&](uint64_t key, auto&& body) {
        if (!use_graphs) {
            body();
            return;
        }
        for (auto& e : W.graphs.entries) {
            if (e.key != key || e.gen != devbuf_generation()) continue;
            launches_suppressed() = true;
            try {
                body();
            } catch (...) {
                launches_suppressed() = false;
                throw;
            }
            launches_suppressed() = false;
            if (e.gen != devbuf_generation()) fail(KRY_INTERNAL, "graph replay: a device buffer moved");
            KB_CUDA(cudaGraphLaunch(e.exec, ctx.stream));
            return;
        }
        KB_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeRelaxed));
        try {
            body();
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(ctx.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        KB_CUDA(cudaStreamEndCapture(ctx.stream, &g));
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        KB_CUDA(ie);
        for (auto it = W.graphs.entries.begin(); it != W.graphs.entries.end();)
            if (it->key == key) {
                cudaGraphExecDestroy(it->exec);
                it = W.graphs.entries.erase(it);
            } else {
                ++it;
            }
        W.graphs.entries.push_back({key, devbuf_generation(), exec});
        KB_CUDA(cudaGraphLaunch(exec, ctx.stream));
    };

    // read per solve (tests switch them between solves)
    const bool speculate_default = [] {  // KRY_SPECULATE=0: every block waits for its factorisation
        const char* e = std::getenv("KRY_SPECULATE");
        return !(e && std::string(e) == "0");
    }();
    const bool defer_last = [] {
        const char* e = std::getenv("KRY_DEFER_FINALIZE");
        return !(e && std::string(e) == "0");
    }();
    bool done = false;
    int stagnation_strikes = 0;
    const i64 blocks = m / s;

    while (!done) {
        const double gamma = r_norm;
        if (gamma / r0 <= cfg.rel_tol) {
            rep.status = KRY_STATUS_CONVERGED;
            break;
        }
        if (rep.iterations >= cfg.max_iters) {
            rep.status = KRY_STATUS_MAX_ITERS;
            break;
        }
        NvtxRange nv_cycle("kry.cycle");
        store.reset();
        {
            cudaEvent_t t0 = ctx.begin_phase();
            launch_scale_div(ctx.stream, n, r.p, gamma, store.col(0), ctx.launches);  // v1 = r/γ (K10)
            ctx.end_phase(PH_RESTART, t0);
        }
        if (standard_mode) store.seed_unit_column(store.col(0));

        bool updated_this_cycle = false;
        bool speculate = speculate_default && two_stage && store.can_speculate(s + 1);
        // one-stage BCGS-PIP2: the rest of the cycle is queued without host
        // waits (both passes factorised on the device) and replayed block by
        // block, so the per-block convergence check keeps its place
        bool spec_pip2 = speculate_default && !two_stage && !standard_mode && scheme == KRY_ORTHO_BCGS_PIP2 &&
                         store.can_speculate_pip2(s + 1);
        // standard GMRES: the columns of the cycle are queued the same way
        // (four BCGS2 passes each, device coefficients) while the prefix
        // fits one Gram group, and replayed column by column
        bool spec_std = speculate_default && standard_mode && store.can_speculate_std(store.filled());
        bool skip_mpk = false;  // a speculative block being redone: its raw columns are in place
        for (i64 j = 0; j < blocks && !done; ++j) {
            Outcome oc;
            if (speculate) {
                // Queue the rest of the big panel without waiting: device
                // factorisation + gated updates (Store::preprocess_speculative),
                // then one sync replays the bookkeeping.  A failed block is
                // redone on the synchronous path below, which handles the
                // truncation / breakdown exactly as the reference.
                // 2-D stencil on one rank: block j's update, block j+1's MPK
                // and Gram in one pass (K6, k_fused.cu); the MPK is then part
                // of the BlkOrtho phase.
                NvtxRange nv("kry.speculative_panel");
                const i64 j0 = j;
                i64 jj = j;
                const bool fuse = store.can_fuse(op, s);
                auto queue_panel = [&] {
                    jj = j0;
                    for (;;) {
                        if (fuse) {
                            cudaEvent_t t1 = ctx.begin_phase();
                            if (jj == j0)
                                store.spec_fused_first(op, s, jj != 0);
                            else
                                store.spec_fused_next(op, s);
                            ctx.end_phase(PH_ORTHO, t1);
                            rep.mpk_bytes += 8.0 * op.nloc * (s + 1.0);
                        } else {
                            const i64 c0 = (jj == 0) ? 0 : store.spec_filled() - 1;
                            cudaEvent_t t0 = ctx.begin_phase();
                            rep.mpk_bytes += store.mpk(op, c0, s) ? 8.0 * op.nloc * (s + 1.0) : s * op.bytes_per_apply();
                            ctx.end_phase(PH_MPK, t0);
                            cudaEvent_t t1 = ctx.begin_phase();
                            store.preprocess_speculative(s + 1, jj != 0);
                            ctx.end_phase(PH_ORTHO, t1);
                        }
                        ++jj;
                        if (store.spec_panel_full() || jj == blocks) break;
                    }
                    store.spec_flush();
                };
                if (fuse)
                    queue_panel();
                else
                    recorded((uint64_t(1) << 60) | (uint64_t(j0) << 30) | uint64_t(store.filled()), queue_panel);
                cudaEvent_t t1 = ctx.begin_phase();
                const i64 f = store.resolve_speculative(rep.sync);
                ctx.end_phase(PH_ORTHO, t1);
                rep.iterations += s * (f < 0 ? jj - j0 : f);
                if (f >= 0) {
                    speculate = false;
                    skip_mpk = true;
                    j = j0 + f - 1;  // ++j: the failed block, synchronously
                    continue;
                }
                j = jj - 1;  // the panel's last block: finalize / check below
                oc.committed = s + 1;
            } else if (spec_pip2) {
                if (!store.spec_has_next()) {
                    NvtxRange nv("kry.speculative_pip2_cycle");
                    recorded((uint64_t(2) << 60) | (uint64_t(j) << 30) | uint64_t(store.filled()), [&] {
                        for (i64 jj = j; jj < blocks; ++jj) {
                            const i64 c0 = (jj == 0) ? 0 : store.spec_filled() - 1;
                            cudaEvent_t t0 = ctx.begin_phase();
                            rep.mpk_bytes +=
                                store.mpk(op, c0, s) ? 8.0 * op.nloc * (s + 1.0) : s * op.bytes_per_apply();
                            ctx.end_phase(PH_MPK, t0);
                            cudaEvent_t t1 = ctx.begin_phase();
                            store.preprocess_speculative_pip2(s + 1, jj != 0);
                            ctx.end_phase(PH_ORTHO, t1);
                        }
                    });
                    cudaEvent_t t1 = ctx.begin_phase();
                    store.spec_fetch();
                    ctx.end_phase(PH_ORTHO, t1);
                }
                if (store.spec_commit_next(rep.sync) != 1) {
                    // the factorisation failed (or the queue is off): redo this
                    // block on the synchronous path, raw columns in place
                    store.spec_drop();
                    spec_pip2 = false;
                    skip_mpk = true;
                    --j;
                    continue;
                }
                oc.committed = s + 1;
            } else if (spec_std) {
                if (!store.spec_has_next()) {
                    NvtxRange nv("kry.speculative_standard_cycle");
                    i64 queued = 0;
                    recorded((uint64_t(3) << 60) | (uint64_t(j) << 30) | uint64_t(store.filled()), [&] {
                        queued = 0;
                        for (i64 jj = j; jj < blocks; ++jj) {
                            const i64 f = store.spec_filled();
                            if (!store.can_speculate_std(f)) break;
                            cudaEvent_t t0 = ctx.begin_phase();
                            op.apply(store.col(f - 1), store.col(f));
                            ctx.end_phase(PH_MPK, t0);
                            rep.mpk_bytes += op.bytes_per_apply();
                            cudaEvent_t t1 = ctx.begin_phase();
                            store.preprocess_speculative_std();
                            ctx.end_phase(PH_ORTHO, t1);
                            ++queued;
                        }
                    });
                    if (queued == 0) {  // the prefix outgrew one Gram group: synchronous from here
                        spec_std = false;
                        --j;
                        continue;
                    }
                    cudaEvent_t t1 = ctx.begin_phase();
                    store.spec_fetch();
                    ctx.end_phase(PH_ORTHO, t1);
                }
                if (store.spec_commit_next(rep.sync) != 1) {
                    // a failed CholQR (or the queue is off): redo this column
                    // on the synchronous path, its raw SpMV output in place
                    store.spec_drop();
                    spec_std = false;
                    skip_mpk = true;
                    --j;
                    continue;
                }
                oc.committed = 1;
            } else if (standard_mode) {
                const i64 f = store.filled();
                if (!skip_mpk) {
                    cudaEvent_t t0 = ctx.begin_phase();
                    op.apply(store.col(f - 1), store.col(f));
                    ctx.end_phase(PH_MPK, t0);
                    rep.mpk_bytes += op.bytes_per_apply();
                }
                skip_mpk = false;
                cudaEvent_t t1 = ctx.begin_phase();
                oc = store.append_block(store.col(f), store.ld(), 1, false, scheme, 0, rep.sync);
                ctx.end_phase(PH_ORTHO, t1);
            } else {
                NvtxRange nv("kry.block");
                const i64 c0 = (j == 0) ? 0 : store.filled() - 1;
                if (!skip_mpk) {
                    cudaEvent_t t0 = ctx.begin_phase();
                    // fused MPK: one read of the start + s writes; else s SpMVs
                    rep.mpk_bytes += store.mpk(op, c0, s) ? 8.0 * op.nloc * (s + 1.0) : s * op.bytes_per_apply();
                    ctx.end_phase(PH_MPK, t0);
                }
                skip_mpk = false;
                cudaEvent_t t1 = ctx.begin_phase();
                if (two_stage)
                    oc = store.preprocess_block(store.col(c0), store.ld(), s + 1, j != 0, rep.sync);
                else
                    oc = store.append_block(store.col(c0), store.ld(), s + 1, j != 0, scheme,
                                            cfg.scheme_big_panel_size, rep.sync);
                ctx.end_phase(PH_ORTHO, t1);
            }
            if (!speculate) rep.iterations += s;  // (the speculative branch counted its blocks)

            if (oc.breakdown || oc.truncated) {
                rep.breakdown = true;
                rep.breakdown_kappa = oc.kappa_estimate;
                if (two_stage && store.big_panel_open()) {
                    cudaEvent_t t1 = ctx.begin_phase();
                    store.finalize_big_panel(rep.sync, defer_last);
                    ctx.end_phase(PH_ORTHO, t1);
                }
                Check res = check_and_update(gamma, true);
                updated_this_cycle = true;
                rep.status = (res.explicit_rel <= cfg.rel_tol) ? KRY_STATUS_CONVERGED : KRY_STATUS_ORTHO_BREAKDOWN;
                done = true;
                break;
            }

            if (two_stage) {
                const bool last_block = (j + 1 == blocks);
                if (store.big_panel_full() || last_block) {
                    NvtxRange nv("kry.finalize_big_panel");
                    cudaEvent_t t1 = ctx.begin_phase();
                    // The cycle's last panel is only read by the solution update:
                    // defer its (15.6 GB at 4000²) rewrite into the y coefficients.
                    Outcome fin = store.finalize_big_panel(rep.sync, defer_last && last_block);
                    ctx.end_phase(PH_ORTHO, t1);
                    if (fin.breakdown) {
                        rep.breakdown = true;
                        rep.breakdown_kappa = fin.kappa_estimate;
                        Check res = check_and_update(gamma, true);
                        updated_this_cycle = true;
                        rep.status =
                            (res.explicit_rel <= cfg.rel_tol) ? KRY_STATUS_CONVERGED : KRY_STATUS_ORTHO_BREAKDOWN;
                        done = true;
                        break;
                    }
                } else {
                    continue;  // convergence is only observable per big panel
                }
            }

            Check res = check_and_update(gamma, false);
            if (res.implicit_crossed) {
                updated_this_cycle = true;
                if (res.explicit_rel <= cfg.rel_tol) {
                    rep.status = KRY_STATUS_CONVERGED;
                    done = true;
                } else {
                    break;  // implicit check was optimistic: restart from the update
                }
            }
        }

        store.spec_drop();  // speculative PIP2 blocks past an early end of the cycle
        if (!updated_this_cycle) check_and_update(gamma, true);
        const double rnorm = r_norm;
        rep.cycle_residuals.push_back(rnorm / r0);
        if (done) break;
        ++rep.restarts;
        if (rnorm / r0 <= cfg.rel_tol) {
            rep.status = KRY_STATUS_CONVERGED;
            break;
        }
        if (rnorm > 0.99 * gamma) {
            if (++stagnation_strikes >= 2) {
                rep.status = KRY_STATUS_STAGNATION;
                break;
            }
        } else {
            stagnation_strikes = 0;
        }
    }

    rep.final_relative_residual = r_norm / r0;
    if (rep.iterations > 0)
        rep.reduces_per_iteration = static_cast<double>(rep.sync.reduces) / static_cast<double>(rep.iterations);
    rep.ortho_bytes = store.ortho_bytes;
    finish();
    store.check_guards();  // KRY_GUARD debug builds of the basis: no kernel wrote outside it
    if (ctx.host_profile) {
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - prof_t0).count();
        std::fprintf(stderr,
                     "[kry host profile] wall %.6f s, blocked in %lld syncs %.6f s, launches %lld, cycles %lld, "
                     "H+LSQ %.6f s\n",
                     wall, static_cast<long long>(ctx.sync_count - prof_syncs0), ctx.sync_wait_s - prof_wait0,
                     static_cast<long long>(ctx.launches - prof_launch0), static_cast<long long>(rep.restarts + 1),
                     lsq_seconds);
    }
    return rep;
}

}  // namespace kb
