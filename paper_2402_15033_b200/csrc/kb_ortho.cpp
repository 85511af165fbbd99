#include "kb_ortho.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "kb_kernels.hpp"

namespace kb {

namespace {

std::vector<std::pair<i64, i64>> groups_for(i64 c0, i64 w) {
    if (c0 == 0) {
        if (round_up(w, 8) > 64)
            fail(KRY_UNSUPPORTED, "block width above 64 columns is not supported on the device path");
        return {{0, 0}};
    }
    return prefix_groups(c0, w);
}

}  // namespace

void gram_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                 Mat& r_col, Mat& g, i64 x_first, i64 x_count, Mat* gx) {
    dim_check(w >= 1, "gram of empty matrix");
    if (round_up(w, 8) > 64) {
        // V wider than one 64-slot pass (a finalize panel ŝ + 1 > 64, e.g.
        // m = 120, ŝ = 120): V = [V1 V2], V1 64 columns — PᵀV1 and V1ᵀV1,
        // then V1ᵀV2 and V2ᵀV2 (V1 as the prefix), then PᵀV2 (recursive in V2).
        const i64 w1 = 64, w2 = w - w1;
        const double* V2 = V + w1 * ldv;
        Mat rc1, g11, r12, g22, rc2, gtmp;
        gram_device(ctx, n, P, ldp, c0, V, ldv, w1, rc1, g11);
        gram_device(ctx, n, V, ldv, w1, V2, ldv, w2, r12, g22);
        if (c0 > 0) gram_device(ctx, n, P, ldp, c0, V2, ldv, w2, rc2, gtmp);
        r_col = Mat(c0, w);
        g = Mat(w, w);
        for (i64 j = 0; j < w; ++j)
            for (i64 l = 0; l < c0; ++l) r_col(l, j) = j < w1 ? rc1(l, j) : rc2(l, j - w1);
        for (i64 j = 0; j < w1; ++j)
            for (i64 i = 0; i < w1; ++i) g(i, j) = g11(i, j);
        for (i64 j = 0; j < w2; ++j) {
            for (i64 i = 0; i < w1; ++i) g(i, w1 + j) = g(w1 + j, i) = r12(i, j);
            for (i64 i = 0; i < w2; ++i) g(w1 + i, w1 + j) = g22(i, j);
        }
        if (gx) *gx = Mat();
        return;
    }
    // Launch plan: one pass per (V column range, prefix group).  A Gram pass
    // holds at most 64 column slots, so a prefix is split into groups that
    // fit beside V; a V wider than 56 columns with a prefix (a finalize of
    // ŝ+1 > 56 columns after an earlier panel, e.g. m = 120, ŝ = 60) runs
    // VᵀV alone and PᵀV in 32-column halves of V.
    struct Pass {
        i64 vj0, wv, start, cp;
        bool vv;
    };
    std::vector<Pass> plain, split;
    if (c0 == 0 || round_up(w, 8) + 8 <= 64) {
        const auto groups = groups_for(c0, w);
        for (size_t gi = 0; gi < groups.size(); ++gi)
            plain.push_back({0, w, groups[gi].first, groups[gi].second, gi == 0});
    }
    if (c0 > 0 && round_up(w, 8) > 32) {
        groups_for(0, w);  // width check
        split.push_back({0, w, 0, 0, true});
        for (i64 vj0 = 0; vj0 < w; vj0 += 32) {
            const i64 wv = std::min<i64>(32, w - vj0);
            for (const auto& grp : prefix_groups(c0, wv)) split.push_back({vj0, wv, grp.first, grp.second, false});
        }
    }
    // columns streamed from HBM by a plan: each pass reads its V range and its prefix group
    auto cost = [](const std::vector<Pass>& ps) {
        i64 c = 0;
        for (const Pass& q : ps) c += q.wv + q.cp;
        return c;
    };
    const std::vector<Pass>& passes = (split.empty() || (!plain.empty() && cost(plain) <= cost(split))) ? plain : split;
    const bool want_x = gx && x_count > 0 && passes.size() == 1 && round_up(w, 8) == 8 && x_first >= 0 &&
                        x_first + x_count <= c0;
    if (gx) *gx = Mat();
    ctx.gram_partials.ensure(static_cast<size_t>(gram_scratch_doubles(w)) * 8);
    ctx.gram_packed.ensure((passes.size() + 1) * 64 * 64 * 8);
    std::vector<std::vector<int>> tiles(passes.size());

    cudaEvent_t t0 = ctx.begin_phase();
    size_t offset = 0;
    for (size_t pi = 0; pi < passes.size(); ++pi) {
        const Pass& ps = passes[pi];
        launch_gram_pass(ctx.stream, n, ps.cp > 0 ? P + ps.start * ldp : nullptr, ldp, ps.cp, V + ps.vj0 * ldv, ldv,
                         ps.wv, ps.vv, ctx.gram_partials.p, ctx.gram_packed.p + offset, tiles[pi], ctx.launches,
                         want_x ? x_first : -1, want_x ? x_count : 0);
        offset += tiles[pi].size() * 64;
    }
    ctx.end_phase(PH_GRAM, t0);
    ctx.gram_bytes += 8.0 * n * (c0 + w);
    ctx.gram_launches += 1;
    ctx.allreduce_sum(ctx.gram_packed.p, offset);
    ctx.h_packed.ensure(std::max<size_t>(offset, 1) * 8);
    KB_CUDA(cudaMemcpyAsync(ctx.h_packed.p, ctx.gram_packed.p, offset * 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();

    // Unpack: tile (jb, ib) entry e = m + 8·nn ↦ slot row 8ib+m, V column 8jb+nn.
    r_col = Mat(c0, w);
    g = Mat(w, w);
    if (want_x) *gx = Mat(c0, x_count);
    const double* h = ctx.h_packed.p;
    size_t off = 0;
    for (size_t pi = 0; pi < passes.size(); ++pi) {
        const Pass& ps = passes[pi];
        const i64 wslots = round_up(ps.wv, 8);
        for (int id : tiles[pi]) {
            if (id >= 64) {  // extra P×P tile: rows slot block ib, columns slot block xb
                const int xb = (id - 64) / 8, ib = (id - 64) % 8;
                for (int e = 0; e < 64; ++e) {
                    const i64 a = 8 * ib + (e & 7) - wslots, b = 8 * xb + (e >> 3) - wslots - x_first;
                    if (a >= 0 && a < ps.cp && b >= 0 && b < x_count) (*gx)(a, b) = h[off + e];
                }
                off += 64;
                continue;
            }
            const int jb = id / 8, ib = id % 8;
            for (int e = 0; e < 64; ++e) {
                const i64 mrow = 8 * ib + (e & 7), jl = 8 * jb + (e >> 3);
                const double val = h[off + e];
                if (jl >= ps.wv) continue;
                const i64 j = ps.vj0 + jl;
                if (mrow < wslots) {
                    if (ps.vv && mrow <= jl) g(mrow, j) = val;  // VᵀV from the pass that carries it
                } else {
                    const i64 l = mrow - wslots;
                    if (l < ps.cp) r_col(ps.start + l, j) = val;
                }
            }
            off += 64;
        }
    }
    for (i64 j = 0; j < w; ++j)
        for (i64 i = 0; i < j; ++i) g(j, i) = g(i, j);
}

void update_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                   const Mat& r_col, const Upper& r_jj, double* out, i64 ldo, bool triangular) {
    if (triangular)
        for (i64 j = 0; j < w; ++j)
            if (r_jj(j, j) == 0.0) fail(KRY_SINGULAR_FACTOR, "triangular factor has a zero diagonal entry");
    if (round_up(w, 8) > 64) {
        // Blocked: Q1 = (V1 − P·R_col1)·R11⁻¹; then V2 − P·R_col2 (stored),
        // and that minus Q1·R12, times R22⁻¹ (Q1 as the prefix).  On the
        // substitution kernels every element receives its terms in the
        // unblocked order (prefix, block-1 columns, block-2 columns, then
        // ×1/r_jj) — one wide substitution, term for term.
        const i64 w1 = 64, w2 = w - w1;
        Mat rc1(c0, w1), rc2(c0, w2), r12(w1, w2);
        Upper r11(w1), r22(w2), none(w2);
        for (i64 l = 0; l < c0; ++l) {
            for (i64 j = 0; j < w1; ++j) rc1(l, j) = r_col(l, j);
            for (i64 j = 0; j < w2; ++j) rc2(l, j) = r_col(l, w1 + j);
        }
        for (i64 j = 0; j < w1; ++j)
            for (i64 i = 0; i <= j; ++i) r11.at(i, j) = r_jj(i, j);
        for (i64 j = 0; j < w2; ++j) {
            for (i64 i = 0; i < w1; ++i) r12(i, j) = r_jj(i, w1 + j);
            for (i64 i = 0; i <= j; ++i) r22.at(i, j) = r_jj(w1 + i, w1 + j);
        }
        const double* V2 = V + w1 * ldv;
        double* out2 = out + w1 * ldo;
        // (each call stages its coefficients through ctx.h_coef / ctx.coef:
        // wait for the previous launch before the next one reuses them)
        update_device(ctx, n, P, ldp, c0, V, ldv, w1, rc1, r11, out, ldo, triangular);
        ctx.sync();
        if (c0 > 0) {
            update_device(ctx, n, P, ldp, c0, V2, ldv, w2, rc2, none, out2, ldo, /*triangular=*/false);
            ctx.sync();
        } else if (out2 != V2) {
            KB_CUDA(cudaMemcpy2DAsync(out2, ldo * 8, V2, ldv * 8, n * 8, w2, cudaMemcpyDeviceToDevice, ctx.stream));
        }
        if (triangular) update_device(ctx, n, out, ldo, w1, out2, ldo, w2, r12, r22, out2, ldo, true);
        return;
    }
    if (triangular && w >= 17 && round_up(w, 8) + round_up(c0, 8) <= 64) {
        // Wide, well-conditioned R_jj (finalize / second pass): substitution
        // as a DMMA GEMM against the explicit inverse (k_tsqr.cu, K5b).
        Upper rinv(w);
        for (i64 j = 0; j < w; ++j) {
            rinv.at(j, j) = 1.0 / r_jj(j, j);
            for (i64 i = j - 1; i >= 0; --i) {
                double s = 0.0;
                for (i64 k = i; k < j; ++k) s += rinv(i, k) * r_jj(k, j);
                rinv.at(i, j) = -s / r_jj(j, j);
            }
        }
        double nr = 0.0, ni = 0.0;
        for (i64 j = 0; j < w; ++j)
            for (i64 i = 0; i <= j; ++i) {
                nr += r_jj(i, j) * r_jj(i, j);
                ni += rinv(i, j) * rinv(i, j);
            }
        if (std::sqrt(nr * ni) <= 4.0 * w) {
            const i64 wslots = round_up(w, 8), nbw = wslots / 8, nb = nbw + round_up(c0, 8) / 8;
            const size_t total = static_cast<size_t>(2 * nb) * nbw * 32;
            ctx.h_coef.ensure(total * 8);
            ctx.coef.ensure(total * 8);
            double* hm = ctx.h_coef.p;
            // M row k: V slot k < wslots → R⁻¹(k, :); P slot → −(R_col·R⁻¹)(k − wslots, :).
            auto mval = [&](i64 k, i64 j) -> double {
                if (j >= w) return 0.0;
                if (k < wslots) return (k < w && k <= j) ? rinv(k, j) : 0.0;
                const i64 l = k - wslots;
                if (l >= c0) return 0.0;
                double s = 0.0;
                for (i64 t = 0; t <= j; ++t) s += r_col(l, t) * rinv(t, j);
                return -s;
            };
            for (i64 kc = 0; kc < 2 * nb; ++kc)
                for (i64 jb = 0; jb < nbw; ++jb)
                    for (int lane = 0; lane < 32; ++lane)
                        hm[(kc * nbw + jb) * 32 + lane] = mval(4 * kc + (lane & 3), 8 * jb + (lane >> 2));
            cudaEvent_t t0 = ctx.begin_phase();
            KB_CUDA(cudaMemcpyAsync(ctx.coef.p, hm, total * 8, cudaMemcpyHostToDevice, ctx.stream));
            launch_update_mma(ctx.stream, n, c0 > 0 ? P : nullptr, ldp, c0, V, ldv, w, ctx.coef.p, out, ldo,
                              ctx.launches);
            ctx.end_phase(PH_UPDATE, t0);
            ctx.update_bytes += 8.0 * n * (c0 + 2.0 * w);
            ctx.update_launches += 1;
            return;
        }
    }
    const int wmax = update_wmax(w);
    const size_t total = static_cast<size_t>(c0 + wmax + 1) * wmax;
    ctx.h_coef.ensure(total * 8);
    ctx.coef.ensure(total * 8);
    double* hc = ctx.h_coef.p;
    std::memset(hc, 0, total * 8);
    // Column slot of j in a coefficient row: natural order, or for the
    // two-threads-per-row kernel (wmax 64) even columns then odd columns.
    auto slot = [wmax](i64 j) -> i64 { return wmax == 64 ? (j & 1) * 32 + (j >> 1) : j; };
    for (i64 l = 0; l < c0; ++l)
        for (i64 j = 0; j < w; ++j) hc[l * wmax + slot(j)] = -r_col(l, j);
    double* nrjj = hc + c0 * wmax;
    double* inv = nrjj + static_cast<size_t>(wmax) * wmax;
    for (i64 j = 0; j < w; ++j) {
        for (i64 l = 0; l < j; ++l) nrjj[l * wmax + slot(j)] = triangular ? -r_jj(l, j) : 0.0;
        inv[slot(j)] = triangular ? 1.0 / r_jj(j, j) : 1.0;
    }
    cudaEvent_t t0 = ctx.begin_phase();
    KB_CUDA(cudaMemcpyAsync(ctx.coef.p, hc, total * 8, cudaMemcpyHostToDevice, ctx.stream));
    launch_update(ctx.stream, n, c0 > 0 ? P : nullptr, ldp, c0, V, ldv, w, ctx.coef.p, triangular, out, ldo,
                  ctx.launches);
    ctx.end_phase(PH_UPDATE, t0);
    ctx.update_bytes += 8.0 * n * (c0 + 2.0 * w);
    ctx.update_launches += 1;
}

PipOut bcgs_pip_partial_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V,
                               i64 ldv, i64 w, double* out, i64 ldo, i64& reduces, bool do_update, i64 x_first,
                               i64 x_count, Mat* gx) {
    reduces += 1;  // fused [Q_prev, V]ᵀV (block_ortho.hpp:155)
    Mat r_col, s;
    gram_device(ctx, n, P, ldp, c0, V, ldv, w, r_col, s, x_first, x_count, gx);
    return pip_from_gram(ctx, n, P, ldp, c0, V, ldv, w, std::move(r_col), std::move(s), out, ldo, do_update);
}

PipOut pip_from_gram(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                     Mat r_col, Mat s, double* out, i64 ldo, bool do_update) {
    PipOut o;
    o.r_col = std::move(r_col);
    if (c0 > 0) {
        // Pythagorean update S = VᵀV − R_colᵀR_col, upper + mirror (block_ortho.hpp:159-166).
        for (i64 j = 0; j < w; ++j)
            for (i64 i = 0; i <= j; ++i) {
                const double c = dot_seq(o.r_col.col(i), o.r_col.col(j), c0);
                s(i, j) -= c;
                if (i != j) s(j, i) = s(i, j);
            }
    }
    o.bad_pivot = try_cholesky(s, o.r_jj);
    if (o.bad_pivot != 0) return o;
    if (do_update) {
        update_device(ctx, n, P, ldp, c0, V, ldv, w, o.r_col, o.r_jj, out, ldo);
    } else {
        for (i64 j = 0; j < w; ++j)  // tri_solve_right's check still applies to a deferred update
            if (o.r_jj(j, j) == 0.0) fail(KRY_SINGULAR_FACTOR, "triangular factor has a zero diagonal entry");
    }
    return o;
}

Upper cholqr_device(Ctx& ctx, i64 n, const double* V, i64 ldv, i64 w, double* out, i64 ldo, i64& reduces,
                    double& bytes) {
    reduces += 1;
    Mat none, g;
    gram_device(ctx, n, nullptr, 0, 0, V, ldv, w, none, g);
    Upper r;
    const i64 piv = try_cholesky(g, r);
    if (piv != 0) throw CholFail{piv};
    update_device(ctx, n, nullptr, 0, 0, V, ldv, w, none, r, out, ldo);
    bytes += 8.0 * n * 3.0 * w;
    return r;
}

Mat project_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                   double* out, i64 ldo, i64& reduces, double& bytes) {
    if (c0 == 0) {
        if (out != V)
            KB_CUDA(cudaMemcpy2DAsync(out, ldo * 8, V, ldv * 8, n * 8, w, cudaMemcpyDeviceToDevice, ctx.stream));
        return Mat(0, w);
    }
    reduces += 1;
    Mat r_block, g;
    gram_device(ctx, n, P, ldp, c0, V, ldv, w, r_block, g);
    Upper ident(w);
    update_device(ctx, n, P, ldp, c0, V, ldv, w, r_block, ident, out, ldo, /*triangular=*/false);
    bytes += 8.0 * n * (2.0 * c0 + 3.0 * w);
    return r_block;
}

Bcgs2Out bcgs2_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                      double* s0, double* s1, i64 lds, double* out, i64 ldo, i64& reduces, double& bytes) {
    const bool single = (w == 1);
    // intra: CholQR (one column) or CholQR2 (R = R₂·R₁), x → dst via mid
    auto intra = [&](const double* x, i64 ldx, double* mid, double* dst, i64 ldd) -> Upper {
        if (single) return cholqr_device(ctx, n, x, ldx, w, dst, ldd, reduces, bytes);
        Upper r1 = cholqr_device(ctx, n, x, ldx, w, mid, lds, reduces, bytes);
        Upper r2 = cholqr_device(ctx, n, mid, lds, w, dst, ldd, reduces, bytes);
        return tri_mul(r2, r1);
    };
    Bcgs2Out o;
    if (c0 == 0) {
        o.r_jj = intra(V, ldv, s0, out, ldo);
        o.r_col = Mat(0, w);
        return o;
    }
    Mat first = project_device(ctx, n, P, ldp, c0, V, ldv, w, s0, lds, reduces, bytes);
    Upper inner = intra(s0, lds, s1, s1, lds);
    Mat second = project_device(ctx, n, P, ldp, c0, s1, lds, w, s1, lds, reduces, bytes);
    Upper outer = cholqr_device(ctx, n, s1, lds, w, out, ldo, reduces, bytes);
    Mat ir(w, w);
    for (i64 j = 0; j < w; ++j)
        for (i64 i = 0; i <= j; ++i) ir(i, j) = inner(i, j);
    Mat corr = mat_mul_nn(second, ir);
    o.r_col = std::move(first);
    for (i64 j = 0; j < o.r_col.cols; ++j)
        for (i64 i = 0; i < o.r_col.rows; ++i) o.r_col(i, j) += corr(i, j);
    o.r_jj = tri_mul(outer, inner);
    return o;
}

}  // namespace kb
