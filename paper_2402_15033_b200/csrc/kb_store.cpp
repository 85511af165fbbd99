#include "kb_store.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kb_kernels.hpp"
#include "kb_ortho.hpp"

namespace kb {

Store::Store(Ctx& ctx, i64 n, i64 m, i64 panel_size, i64 big_panel_size)
    : ctx_(ctx),
      n_(n),
      max_cols_(m + 1),
      panel_size_(panel_size),
      big_panel_size_(big_panel_size == 0 ? m : big_panel_size),
      ld_(device_ld(n)),
      r_(m + 1) {
    // BasisStore ctor checks (basis_store.hpp:51-54).
    if (panel_size_ == 0 || m % panel_size_ != 0)
        fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: panel size must divide the restart length");
    if (big_panel_size_ % panel_size_ != 0 || big_panel_size_ > m)
        fail(KRY_DIMENSION_MISMATCH,
             "dimension mismatch: big panel size must be a multiple of the panel size, <= m");
    pgram_ = Mat(max_cols_, max_cols_);
    pready_.assign(static_cast<size_t>(max_cols_), 0);
    if (const char* e = std::getenv("KRY_FUSED_PANEL_GRAM")) fused_panel_gram_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("KRY_GUARD")) qoff_ = std::atoi(e) == 1 ? 1 : 0;
    q_.ensure(static_cast<size_t>(ld_) * (max_cols_ + 2 * qoff_) * 8);
    zero_q();
}

void Store::zero_q() {
    KB_CUDA(cudaMemsetAsync(q_.p, 0, q_.bytes, ctx_.stream));
    if (guarded()) fill_guards();
}

void Store::fill_guards() {
    const size_t colb = static_cast<size_t>(ld_) * 8;
    KB_CUDA(cudaMemsetAsync(q_.p, 0xFF, colb, ctx_.stream));                           // column −1
    KB_CUDA(cudaMemsetAsync(q_.p + (max_cols_ + 1) * ld_, 0xFF, colb, ctx_.stream));  // column m + 1
    if (ld_ > n_)  // padding rows [n, ld) of every column
        KB_CUDA(cudaMemset2DAsync(col(0) + n_, colb, 0xFF, static_cast<size_t>(ld_ - n_) * 8, max_cols_,
                                  ctx_.stream));
}

void Store::check_guards() {
    if (!guarded()) return;
    std::vector<uint64_t> h(static_cast<size_t>(ld_) * (max_cols_ + 2));
    KB_CUDA(cudaMemcpyAsync(h.data(), q_.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
    for (i64 c = 0; c < max_cols_ + 2; ++c) {
        const bool guard_col = c == 0 || c == max_cols_ + 1;
        for (i64 r = guard_col ? 0 : n_; r < ld_; ++r)
            if (h[static_cast<size_t>(c * ld_ + r)] != ~uint64_t(0))
                fail(KRY_INTERNAL, "KRY_GUARD: basis guard overwritten at column " + std::to_string(c - 1) + ", row " +
                                       std::to_string(r));
    }
}

bool Store::deferred_coefficients(const std::vector<double>& y, std::vector<double>& y_out) const {
    if (!pending_) return false;
    // Q_fin[:, c0+i] = (Q[:, c0:c0+w) − Q[:, 0:c0]·R_col)·R_jj⁻¹ column i; R_jj⁻¹ is
    // upper triangular, so the first p panel columns only involve the first p.
    const i64 k = static_cast<i64>(y.size());
    y_out = y;
    if (k <= pend_c0_) return true;
    const i64 p = std::min(k - pend_c0_, pend_w_);
    std::vector<double> z(static_cast<size_t>(p));
    for (i64 i = p; i-- > 0;) {  // z = R_jj[:p,:p]⁻¹ · y_panel (back substitution)
        double s = y[pend_c0_ + i];
        for (i64 l = i + 1; l < p; ++l) s -= pend_rjj_(i, l) * z[l];
        z[i] = s / pend_rjj_(i, i);
    }
    for (i64 l = 0; l < pend_c0_; ++l) {  // y_pre −= R_col[:, :p]·z
        double s = 0.0;
        for (i64 i = 0; i < p; ++i) s += pend_rcol_(l, i) * z[i];
        y_out[l] = y[l] - s;
    }
    for (i64 i = 0; i < p; ++i) y_out[pend_c0_ + i] = z[i];
    return true;
}

void Store::reset() {
    pending_ = false;
    fpend_.live = false;
    spec_drop();
    std::fill(pready_.begin(), pready_.end(), 0);
    filled_ = 0;
    finalized_ = 0;
    big_panel_start_ = 0;
    seam_valid_ = false;
    states_.clear();
    records_.clear();
    r_ = Upper(max_cols_);
    // The reference also zeroes Q (basis_store.hpp:91).  The solver never
    // reads a column before writing it, so gmres() skips this pass
    // (Store::reset is only used by the C-ABI reset, where it is kept).
}

void Store::seed_unit_column(const double* d_v) {
    if (filled_ != 0) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: seed requires an empty store");
    if (d_v != col(0))
        KB_CUDA(cudaMemcpyAsync(col(0), d_v, static_cast<size_t>(n_) * 8, cudaMemcpyDeviceToDevice, ctx_.stream));
    r_.at(0, 0) = 1.0;
    filled_ = 1;
    finalized_ = 1;
    big_panel_start_ = 1;
}

double* Store::scratch(int which, i64 w) {
    scratch_[which].ensure(static_cast<size_t>(ld_) * round_up(w, 8) * 8);
    return scratch_[which].p;
}

bool Store::can_speculate(i64 w) const {
    // one prefix group (round_up(c0,8) + 8 ≤ 64) for every block of the
    // cycle — the last block's prefix is c0 = capacity − w (s = 1..4 with
    // m = 60 exceed it: c0 = 59 at w = 2) — and the fused panel-Gram
    // bookkeeping this path assumes
    return w >= 1 && w <= 8 && round_up(max_cols_ - w, 8) + 8 <= 64 && fused_panel_gram_;
}

bool Store::spec_panel_full() const {
    const i64 f = spec_filled(), b = spec_.empty() ? big_panel_start_ : spec_bps_;
    return f > b && f - b >= big_panel_size_ + 1;
}

Store::SpecPlan Store::spec_plan(i64 w, bool overlap, bool pieces) {
    const bool first = spec_.empty();
    const i64 filled = first ? filled_ : spec_filled_;
    if (overlap && filled == 0) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: basis store capacity exceeded");
    const i64 c0 = overlap ? filled - 1 : filled;
    if (c0 + w > max_cols_) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: basis store capacity exceeded");
    const i64 maxb = 4 * max_cols_;  // queue capacity in result slots (≤ m blocks per cycle; 2 per PIP2 block, 4 per standard column)
    if (first) {
        spec_bps_ = big_panel_start_;
        spec_xd_ = big_panel_start_;
        while (spec_xd_ < max_cols_ && pready_[static_cast<size_t>(spec_xd_)]) ++spec_xd_;
        spec_slots_.ensure(static_cast<size_t>(maxb) * kSlotDoubles * 8);
        spec_coef_.ensure(static_cast<size_t>(maxb) * 640 * 8);
        spec_skip_.ensure(static_cast<size_t>(maxb) * 4);
        spec_host_.ensure(static_cast<size_t>(maxb) * kSlotDoubles * 8);
    }
    SpecPlan p{c0, static_cast<i64>(spec_.size()), -1, 0};
    // panel-Gram pieces (same rule as run_scheme's first-stage branch): the
    // previous block is a preprocessed block of the open panel unless this
    // is the panel's first block
    const bool prev_in_panel = !first || (!records_.empty() && states_.back() == KRY_PANEL_PREPROCESSED);
    if (pieces && prev_in_panel) {
        const i64 xend = std::min(c0 / 8 * 8, spec_xd_ / 8 * 8 + 16);
        if (xend > spec_xd_) {
            p.xf = spec_xd_;
            p.xc = xend - spec_xd_;
        }
    }
    ctx_.gram_partials.ensure(static_cast<size_t>(gram_scratch_doubles(w)) * 8);
    ctx_.gram_packed.ensure(2 * 64 * 64 * 8);
    return p;
}

// [allreduce] → device factorisation of the packed Gram in ctx_.gram_packed.
PipBlockArgs Store::spec_factor(const SpecPlan& p, i64 w, int mode) {
    PipBlockArgs a{};
    a.mode = mode;
    a.packed = ctx_.gram_packed.p;
    a.nb = static_cast<int>(1 + round_up(p.c0, 8) / 8);
    a.nx = p.xc > 0 ? static_cast<int>((8 + p.xf + p.xc - 1) / 8 - (8 + p.xf) / 8 + 1) : 0;
    a.xb0 = p.xc > 0 ? static_cast<int>((8 + p.xf) / 8) : 0;
    a.x_first = static_cast<int>(p.xf);
    a.x_count = static_cast<int>(p.xc);
    a.c0 = static_cast<int>(p.c0);
    a.w = static_cast<int>(w);
    a.wmax = update_wmax(w);
    a.slot = spec_slots_.p + p.idx * kSlotDoubles;
    a.prev_slot = p.idx > 0 ? spec_slots_.p + (p.idx - 1) * kSlotDoubles : nullptr;
    a.coef = spec_coef_.p + p.idx * 640;
    a.skip = spec_skip_.as<int>() + p.idx;
    ctx_.allreduce_sum(ctx_.gram_packed.p, static_cast<size_t>(a.nb + a.nx * (a.nb - 1)) * 64);
    launch_pip_block(ctx_.stream, a, ctx_.launches);
    return a;
}

void Store::spec_push(const SpecPlan& p, i64 w, bool overlap, const double* raw) {
    spec_.push_back({p.c0, w, overlap, p.xf, p.xc, raw});
    spec_filled_ = p.c0 + w;
    spec_bps_ = std::min(spec_bps_, p.c0);
    if (p.xc > 0) spec_xd_ = p.xf + p.xc;
}

void Store::preprocess_speculative(i64 w, bool overlap) {
    const SpecPlan p = spec_plan(w, overlap);
    const i64 c0 = p.c0;
    // Gram (+ reduce) → allreduce → device factorisation → gated update
    std::vector<int> tiles;
    cudaEvent_t t0 = ctx_.begin_phase();
    launch_gram_pass(ctx_.stream, n_, c0 > 0 ? col(0) : nullptr, ld_, c0, col(c0), ld_, w, true,
                     ctx_.gram_partials.p, ctx_.gram_packed.p, tiles, ctx_.launches, p.xf, p.xc);
    ctx_.end_phase(PH_GRAM, t0);
    ctx_.gram_bytes += 8.0 * n_ * (c0 + w);
    ctx_.gram_launches += 1;
    const PipBlockArgs a = spec_factor(p, w);
    cudaEvent_t t1 = ctx_.begin_phase();
    launch_update(ctx_.stream, n_, c0 > 0 ? col(0) : nullptr, ld_, c0, col(c0), ld_, w, a.coef, true, col(c0), ld_,
                  ctx_.launches, a.skip);
    ctx_.end_phase(PH_UPDATE, t1);
    ctx_.update_bytes += 8.0 * n_ * (c0 + 2.0 * w);
    ctx_.update_launches += 1;
    spec_push(p, w, overlap, nullptr);
}

// ---- fused first stage (K6, k_fused.cu) ------------------------------------
bool Store::can_fuse(const Operator& op, i64 s) {
    // Opt-in (KRY_FUSED_PASS=1): measured slower than the separate kernels
    // on B200 ("fused first-stage pass").
    const bool on = [] {
        const char* e = std::getenv("KRY_FUSED_PASS");
        return e && std::atoi(e) == 1;
    }();
    if (!on || !can_speculate(s + 1) || op.kind != Operator::LAPLACE2D || ctx_.nranks != 1 || op.nloc != n_) return false;
    for (auto& b : fraw_) b.ensure(static_cast<size_t>(ld_) * (s + 1) * 8);
    ctx_.gram_partials.ensure(static_cast<size_t>(std::max(fused_partials_doubles(), gram_scratch_doubles(s + 1))) * 8);
    return fused_pass_supported(op.geom, static_cast<int>(s), s + 1, max_cols_ - (s + 1), ld_, col(0), fraw_[0].p,
                                fraw_[1].p);
}

void Store::spec_fused_first(Operator& op, i64 s, bool overlap) {
    const i64 w = s + 1;
    const SpecPlan p = spec_plan(w, overlap);
    const int buf = 0;
    double* raw = fraw_[buf].p;
    // raw block: column 0 = the start (store column c0), 1..s = A^k·start
    KB_CUDA(cudaMemcpyAsync(raw, col(p.c0), static_cast<size_t>(n_) * 8, cudaMemcpyDeviceToDevice, ctx_.stream));
    cudaEvent_t t0 = ctx_.begin_phase();
    if (!op.mpk(raw, raw + ld_, ld_, static_cast<int>(s)))
        for (i64 k = 0; k < s; ++k) op.apply(raw + k * ld_, raw + (k + 1) * ld_);
    ctx_.end_phase(PH_MPK, t0);
    std::vector<int> tiles;
    cudaEvent_t t1 = ctx_.begin_phase();
    launch_gram_pass(ctx_.stream, n_, p.c0 > 0 ? col(0) : nullptr, ld_, p.c0, raw, ld_, w, true,
                     ctx_.gram_partials.p, ctx_.gram_packed.p, tiles, ctx_.launches, p.xf, p.xc);
    ctx_.end_phase(PH_GRAM, t1);
    ctx_.gram_bytes += 8.0 * n_ * (p.c0 + w);
    ctx_.gram_launches += 1;
    const PipBlockArgs a = spec_factor(p, w);
    fpend_ = {true, p.c0, w, buf, a.coef, a.skip};
    spec_push(p, w, overlap, raw);
}

void Store::spec_fused_next(Operator& op, i64 s) {
    const i64 w = s + 1;
    if (!fpend_.live || fpend_.w != w) fail(KRY_INTERNAL, "fused pass without a pending block");
    const SpecPlan p = spec_plan(w, true);
    const int nbuf = 1 - fpend_.buf;
    FusedPassArgs f{};
    f.Q = col(0);
    f.ld = ld_;
    f.V = fraw_[fpend_.buf].p;
    f.Vn = fraw_[nbuf].p;
    f.c0 = static_cast<int>(fpend_.c0);
    f.w = static_cast<int>(w);
    f.coef = fpend_.coef;
    f.skip = fpend_.skip;
    f.c0n = static_cast<int>(p.c0);
    f.x_first = static_cast<int>(p.xf);
    f.x_count = static_cast<int>(p.xc);
    f.partials = ctx_.gram_partials.p;
    cudaEvent_t t0 = ctx_.begin_phase();
    launch_fused_pass(ctx_.stream, op.geom, static_cast<int>(s), f, ctx_.gram_packed.p, ctx_.launches);
    ctx_.end_phase(PH_FUSED, t0);
    // necessary HBM traffic: prefix + raw block read once, block j and raw block j+1 written
    ctx_.fused_bytes += 8.0 * n_ * (fpend_.c0 + 3.0 * w);
    ctx_.fused_launches += 1;
    const PipBlockArgs a = spec_factor(p, w);
    fpend_ = {true, p.c0, w, nbuf, a.coef, a.skip};
    spec_push(p, w, true, fraw_[nbuf].p);
}

void Store::spec_flush() {
    if (!fpend_.live) return;
    const i64 c0 = fpend_.c0, w = fpend_.w;
    cudaEvent_t t1 = ctx_.begin_phase();
    launch_update(ctx_.stream, n_, c0 > 0 ? col(0) : nullptr, ld_, c0, fraw_[fpend_.buf].p, ld_, w, fpend_.coef, true,
                  col(c0), ld_, ctx_.launches, fpend_.skip);
    ctx_.end_phase(PH_UPDATE, t1);
    ctx_.update_bytes += 8.0 * n_ * (c0 + 2.0 * w);
    ctx_.update_launches += 1;
    fpend_.live = false;
}

i64 Store::resolve_speculative(Sync& sync) {
    if (spec_.empty()) return -1;
    spec_fetch();
    i64 failed = -1;
    for (size_t i = 0; i < spec_.size(); ++i)
        if (spec_commit_next(sync) == 0) {
            failed = static_cast<i64>(i);
            break;
        }
    spec_drop();
    return failed;
}

void Store::spec_fetch() {
    if (spec_.empty()) return;
    const size_t slots = spec_.size() * (spec_.front().pip2 ? 2 : spec_.front().std1 ? 4 : 1);
    KB_CUDA(cudaMemcpyAsync(spec_host_.p, spec_slots_.p, slots * kSlotDoubles * 8, cudaMemcpyDeviceToHost,
                            ctx_.stream));
    ctx_.sync();
    spec_fetched_ = true;
    spec_next_ = 0;
}

void Store::spec_drop() {
    spec_.clear();
    spec_fetched_ = false;
    spec_next_ = 0;
}

namespace {
// R_col and R_jj of one result slot (k_pip.cu layout)
void slot_factors(const double* slot, i64 c0, i64 w, Mat& r_col, Upper& r_jj) {
    r_col = Mat(c0, w);
    r_jj = Upper(w);
    const double* rc = slot + kSlotRcol;
    const double* rj = rc + c0 * w;
    for (i64 j = 0; j < w; ++j) {
        for (i64 l = 0; l < c0; ++l) r_col(l, j) = rc[l + j * c0];
        for (i64 l = 0; l <= j; ++l) r_jj.at(l, j) = rj[l + j * w];
    }
}
}  // namespace

int Store::spec_commit_next(Sync& sync) {
    if (!spec_fetched_ || spec_next_ >= spec_.size()) return -1;
    const size_t i = spec_next_;
    const SpecBlock& b = spec_[i];
    const int per = b.pip2 ? 2 : b.std1 ? 4 : 1;
    const double* slot = spec_host_.p + per * i * kSlotDoubles;
    bool failed = false;
    for (int k = 0; k < per; ++k) failed = failed || slot[k * kSlotDoubles + kSlotStatus] != 0.0;
    if (failed) {
        // fused path: the block's raw columns live outside the store;
        // put them where the synchronous redo expects them
        if (b.raw)
            KB_CUDA(cudaMemcpy2DAsync(col(b.c0), ld_ * 8, b.raw, ld_ * 8, n_ * 8, b.w, cudaMemcpyDeviceToDevice,
                                      ctx_.stream));
        spec_next_ = spec_.size();
        return 0;
    }
    ++spec_next_;
    const i64 before = sync.reduces;
    OrthoRes res;
    if (b.std1) {
        // run_scheme BCGS2 with one column (intra = CholQR): R_col = R₁ +
        // T_col·R_in, R_jj = R_out·R_in — the synchronous path's arithmetic.
        const double* sl[4] = {slot, slot + kSlotDoubles, slot + 2 * kSlotDoubles, slot + 3 * kSlotDoubles};
        Mat first(b.c0, 1), second(b.c0, 1), ir(1, 1);
        Upper inner(1), outer(1);
        for (i64 l = 0; l < b.c0; ++l) {
            first(l, 0) = sl[0][kSlotRcol + l];
            second(l, 0) = sl[2][kSlotRcol + l];
        }
        inner.at(0, 0) = sl[1][kSlotRcol];
        outer.at(0, 0) = sl[3][kSlotRcol];
        ir(0, 0) = inner(0, 0);
        Mat corr = mat_mul_nn(second, ir);
        res.r_col = std::move(first);
        for (i64 l = 0; l < res.r_col.rows; ++l) res.r_col(l, 0) += corr(l, 0);
        res.r_jj = tri_mul(outer, inner);
        sync.add(4);
        ortho_bytes += 2.0 * 8.0 * n_ * (2.0 * b.c0 + 3.0) + 2.0 * 8.0 * n_ * 3.0;
        commit(b.c0, b.overlap, res, 1, KRY_PANEL_FINAL);
    } else if (b.pip2) {
        // run_scheme BcgsPip2 (basis_store.hpp:220-239): R_col = R₁ + T_col·R_jj₁,
        // R_jj = T_jj·R_jj₁ — the synchronous path's arithmetic (run_scheme).
        OrthoRes first, second;
        slot_factors(slot, b.c0, b.w, first.r_col, first.r_jj);
        slot_factors(slot + kSlotDoubles, b.c0, b.w, second.r_col, second.r_jj);
        res.r_col = std::move(first.r_col);
        if (res.r_col.rows > 0) {
            Mat rjj(b.w, b.w);
            for (i64 j = 0; j < b.w; ++j)
                for (i64 l = 0; l <= j; ++l) rjj(l, j) = first.r_jj(l, j);
            Mat corr = mat_mul_nn(second.r_col, rjj);
            for (i64 j = 0; j < res.r_col.cols; ++j)
                for (i64 l = 0; l < res.r_col.rows; ++l) res.r_col(l, j) += corr(l, j);
        }
        res.r_jj = tri_mul(second.r_jj, first.r_jj);
        sync.add(2);
        ortho_bytes += 2.0 * 8.0 * n_ * (2.0 * b.c0 + 3.0 * b.w);
        commit(b.c0, b.overlap, res, b.w, KRY_PANEL_FINAL);
    } else {
        slot_factors(slot, b.c0, b.w, res.r_col, res.r_jj);
        const double* pieces = slot + kSlotPieces;
        for (i64 k = 0; k < b.x_count; ++k) {
            for (i64 l = 0; l < b.c0; ++l) pgram_(l, b.x_first + k) = pieces[l + k * b.c0];
            pready_[static_cast<size_t>(b.x_first + k)] = 1;
        }
        // preprocess_block → append_block bookkeeping (one reduce per block)
        sync.add(1);
        ortho_bytes += 8.0 * n_ * (2.0 * b.c0 + 3.0 * b.w);
        commit(b.c0, b.overlap, res, b.w, KRY_PANEL_PREPROCESSED);
    }
    sync.per_block.push_back(sync.reduces - before);
    return 1;
}

bool Store::can_speculate_pip2(i64 w) const {
    // the device factorisation handles c0 ≤ 64, w ≤ 8, and every block's
    // prefix must fit one 64-slot Gram group (as can_speculate)
    return w >= 1 && w <= 8 && round_up(max_cols_ - w, 8) + 8 <= 64;
}

void Store::preprocess_speculative_pip2(i64 w, bool overlap) {
    const SpecPlan p = spec_plan(w, overlap, /*pieces=*/false);
    const i64 c0 = p.c0, b = static_cast<i64>(spec_.size());
    double* s0 = scratch(0, w);
    for (int pass = 0; pass < 2; ++pass) {
        // pass 1: V (store columns) → scratch; pass 2: scratch → store columns
        const double* V = pass == 0 ? col(c0) : s0;
        double* out = pass == 0 ? s0 : col(c0);
        SpecPlan q = p;
        q.idx = 2 * b + pass;
        std::vector<int> tiles;
        cudaEvent_t t0 = ctx_.begin_phase();
        launch_gram_pass(ctx_.stream, n_, c0 > 0 ? col(0) : nullptr, ld_, c0, V, ld_, w, true, ctx_.gram_partials.p,
                         ctx_.gram_packed.p, tiles, ctx_.launches, -1, 0);
        ctx_.end_phase(PH_GRAM, t0);
        ctx_.gram_bytes += 8.0 * n_ * (c0 + w);
        ctx_.gram_launches += 1;
        const PipBlockArgs a = spec_factor(q, w);
        cudaEvent_t t1 = ctx_.begin_phase();
        launch_update(ctx_.stream, n_, c0 > 0 ? col(0) : nullptr, ld_, c0, V, ld_, w, a.coef, true, out, ld_,
                      ctx_.launches, a.skip);
        ctx_.end_phase(PH_UPDATE, t1);
        ctx_.update_bytes += 8.0 * n_ * (c0 + 2.0 * w);
        ctx_.update_launches += 1;
    }
    spec_push(p, w, overlap, nullptr);
    spec_.back().pip2 = true;
}

bool Store::can_speculate_std(i64 c0) const {
    // one prefix group for the projection Grams (round_up(c0, 8) + 8 ≤ 64)
    return c0 >= 1 && c0 + 1 <= max_cols_ && round_up(c0, 8) + 8 <= 64;
}

void Store::preprocess_speculative_std() {
    const i64 w = 1;
    const SpecPlan p = spec_plan(w, false, /*pieces=*/false);
    const i64 c0 = p.c0, b = static_cast<i64>(spec_.size());
    double* s0 = scratch(0, w);
    double* s1 = scratch(1, w);
    // bcgs2 (block_ortho.hpp:102-137) on one column: project V → s0, CholQR
    // s0 → s1, project s1 → s0, CholQR s0 → the store column.  Only the last
    // pass writes the store, so a failure anywhere leaves V raw there.
    struct Pass {
        const double* v;
        double* out;
        bool project;
    };
    const Pass passes[4] = {{col(c0), s0, true}, {s0, s1, false}, {s1, s0, true}, {s0, col(c0), false}};
    for (int k = 0; k < 4; ++k) {
        const Pass& ps = passes[k];
        const i64 pc0 = ps.project ? c0 : 0;
        SpecPlan q = p;
        q.c0 = pc0;
        q.idx = 4 * b + k;
        std::vector<int> tiles;
        cudaEvent_t t0 = ctx_.begin_phase();
        launch_gram_pass(ctx_.stream, n_, pc0 > 0 ? col(0) : nullptr, ld_, pc0, ps.v, ld_, w, true,
                         ctx_.gram_partials.p, ctx_.gram_packed.p, tiles, ctx_.launches, -1, 0);
        ctx_.end_phase(PH_GRAM, t0);
        ctx_.gram_bytes += 8.0 * n_ * (pc0 + w);
        ctx_.gram_launches += 1;
        const PipBlockArgs a = spec_factor(q, w, ps.project ? 1 : 0);
        cudaEvent_t t1 = ctx_.begin_phase();
        launch_update(ctx_.stream, n_, pc0 > 0 ? col(0) : nullptr, ld_, pc0, ps.v, ld_, w, a.coef, !ps.project, ps.out,
                      ld_, ctx_.launches, a.skip);
        ctx_.end_phase(PH_UPDATE, t1);
        ctx_.update_bytes += 8.0 * n_ * (pc0 + 2.0 * w);
        ctx_.update_launches += 1;
    }
    spec_push(p, w, false, nullptr);
    spec_.back().std1 = true;
}

bool Store::mpk(Operator& op, i64 c0, i64 s) {
    dim_check(c0 + s + 1 <= max_cols_, "basis store capacity exceeded");
    if (op.mpk(col(c0), col(c0 + 1), ld_, static_cast<int>(s))) return true;
    for (i64 k = 0; k < s; ++k) op.apply(col(c0 + k), col(c0 + k + 1));
    return false;
}

Outcome Store::append_block(const double* V, i64 ldv, i64 w, bool overlap, int kind, i64, Sync& sync) {
    const i64 before = sync.reduces;
    Outcome out = append_impl(V, ldv, w, overlap, kind, sync);
    sync.per_block.push_back(sync.reduces - before);
    return out;
}

Outcome Store::preprocess_block(const double* V, i64 ldv, i64 w, bool overlap, Sync& sync) {
    return append_block(V, ldv, w, overlap, KRY_ORTHO_TWO_STAGE, big_panel_size_, sync);
}

Outcome Store::append_impl(const double* V, i64 ldv, i64 w, bool overlap, int kind, Sync& sync) {
    Outcome out;
    i64 width = w;
    if (overlap && filled_ == 0) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: basis store capacity exceeded");
    const i64 c0 = overlap ? filled_ - 1 : filled_;
    if (c0 + width > max_cols_) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: basis store capacity exceeded");

    // basis_store.hpp:178-208: first-pass pivot failure truncates and retries.
    while (width >= 1) {
        i64 bad = 0;
        try {
            OrthoRes res = run_scheme(c0, V, ldv, width, kind, sync);
            commit(c0, overlap, res, width, kind == KRY_ORTHO_TWO_STAGE ? KRY_PANEL_PREPROCESSED : KRY_PANEL_FINAL);
            out.committed = width;
            if (out.truncated) record_seam(V + width * ldv, sync);
            return out;
        } catch (const FirstPassFailure& e) {
            bad = e.pivot;
        } catch (const SecondPassBreakdown& e) {
            out.breakdown = true;
            out.truncated = false;
            out.pivot = e.pivot;
            out.kappa_estimate = diagnostic_kappa(c0, V, ldv, width);
            return out;
        }
        out.truncated = true;
        out.pivot = bad;
        if (bad <= 1) break;
        width = std::min(width, bad - 1);
    }
    out.breakdown = true;
    out.truncated = false;
    out.kappa_estimate = diagnostic_kappa(c0, V, ldv, w);
    return out;
}

Store::OrthoRes Store::pip(i64 c0, const double* V, i64 ldv, i64 w, double* out, i64 ldo, Sync& sync,
                           bool first_pass, bool do_update, i64 x_first, i64 x_count) {
    i64 red = 0;
    Mat gx;
    PipOut o = bcgs_pip_partial_device(ctx_, n_, col(0), ld_, c0, V, ldv, w, out, ldo, red, do_update, x_first,
                                       x_count, x_count > 0 ? &gx : nullptr);
    sync.add(red);
    if (gx.rows > 0) {  // panel Gram pieces for the previous block's (now final) columns
        for (i64 b = 0; b < gx.cols; ++b) {
            for (i64 a = 0; a < gx.rows; ++a) pgram_(a, x_first + b) = gx(a, b);
            pready_[static_cast<size_t>(x_first + b)] = 1;
        }
    }
    // algorithmic bytes actually moved: Gram reads c0+w; the update reads c0+w and writes w
    ortho_bytes += do_update ? 8.0 * n_ * (2.0 * c0 + 3.0 * w) : 8.0 * n_ * (c0 + w);
    if (o.bad_pivot != 0) {
        if (first_pass) throw FirstPassFailure{o.bad_pivot};
        throw SecondPassBreakdown{o.bad_pivot};
    }
    return OrthoRes{std::move(o.r_col), std::move(o.r_jj)};
}

namespace {
// the device helpers count reduces in an i64; the store's SyncCounter adds them
Upper cholqr_dev(Ctx& ctx, i64 n, const double* V, i64 ldv, i64 w, double* out, i64 ldo, Sync& sync, double& bytes) {
    i64 red = 0;
    struct Add {
        Sync& s;
        i64& r;
        ~Add() { s.add(r); }
    } add{sync, red};
    return cholqr_device(ctx, n, V, ldv, w, out, ldo, red, bytes);
}
Mat project_dev(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w, double* out,
                i64 ldo, Sync& sync, double& bytes) {
    i64 red = 0;
    Mat r = project_device(ctx, n, P, ldp, c0, V, ldv, w, out, ldo, red, bytes);
    sync.add(red);
    return r;
}
}  // namespace

Store::OrthoRes Store::run_scheme(i64 c0, const double* V, i64 ldv, i64 w, int kind, Sync& sync) {
    switch (kind) {
        case KRY_ORTHO_TWO_STAGE: {  // single first-stage pass
            // The previous block's columns are final now: let this Gram also
            // produce their products with every earlier column (panel Gram).
            // Only whole 8-column slot blocks are requested (one, at most two
            // per Gram): a partial block costs a full block of DMMA work, and
            // the extra tiles stay hidden under the HBM stream only while
            // they are few.
            i64 xf = -1, xc = 0;
            if (fused_panel_gram_ && !records_.empty() && states_.back() == KRY_PANEL_PREPROCESSED) {
                i64 xd = big_panel_start_;
                while (xd < c0 && pready_[static_cast<size_t>(xd)]) ++xd;
                const i64 xend = std::min(c0 / 8 * 8, xd / 8 * 8 + 16);
                if (xend > xd) {
                    xf = xd;
                    xc = xend - xd;
                }
            }
            return pip(c0, V, ldv, w, col(c0), ld_, sync, true, true, xf, xc);
        }
        case KRY_ORTHO_BCGS_PIP2: {
            double* s0 = scratch(0, w);
            OrthoRes first = pip(c0, V, ldv, w, s0, ld_, sync, true);
            OrthoRes second = pip(c0, s0, ld_, w, col(c0), ld_, sync, false);
            OrthoRes out;
            out.r_col = std::move(first.r_col);
            if (out.r_col.rows > 0) {
                Mat rjj(w, w);
                for (i64 j = 0; j < w; ++j)
                    for (i64 i = 0; i <= j; ++i) rjj(i, j) = first.r_jj(i, j);
                Mat corr = mat_mul_nn(second.r_col, rjj);
                for (i64 j = 0; j < out.r_col.cols; ++j)
                    for (i64 i = 0; i < out.r_col.rows; ++i) out.r_col(i, j) += corr(i, j);
            }
            out.r_jj = tri_mul(second.r_jj, first.r_jj);
            return out;
        }
        case KRY_ORTHO_BCGS2_HHQR:
        case KRY_ORTHO_BCGS2_CHOLQR2: {
            // bcgs2 (block_ortho.hpp:102-137) / run_scheme (basis_store.hpp:240-280).
            const bool single = (w == 1);
            if (kind == KRY_ORTHO_BCGS2_HHQR && !single)
                fail(KRY_UNSUPPORTED, "BCGS2 with a Householder intra step is not on the device path");
            double* s0 = scratch(0, w);
            double* s1 = scratch(1, w);
            // intra: CholQR (single column) or CholQR2; input x → output dst.
            // The first CholQR of CholQR2 writes `mid`, only the second writes
            // dst: V may alias dst (the solver feeds blocks in place), and a
            // failure of the second pass must leave V raw for the retry and
            // record_seam (append_impl, basis_store.hpp:169-209).
            auto intra = [&](const double* x, i64 ldx, double* mid, double* dst) -> Upper {
                if (single) return cholqr_dev(ctx_, n_, x, ldx, w, dst, ld_, sync, ortho_bytes);
                Upper r1 = cholqr_dev(ctx_, n_, x, ldx, w, mid, ld_, sync, ortho_bytes);
                Upper r2 = cholqr_dev(ctx_, n_, mid, ld_, w, dst, ld_, sync, ortho_bytes);
                return tri_mul(r2, r1);
            };
            OrthoRes out;
            if (c0 == 0) {
                try {
                    out.r_jj = intra(V, ldv, s0, col(c0));
                } catch (const CholFail& f) {
                    throw FirstPassFailure{f.pivot};
                }
                out.r_col = Mat(0, w);
                return out;
            }
            Mat first_block;
            Upper inner_r;
            try {
                first_block = project_dev(ctx_, n_, col(0), ld_, c0, V, ldv, w, s0, ld_, sync, ortho_bytes);
                inner_r = intra(s0, ld_, s1, s1);
            } catch (const CholFail& f) {
                throw FirstPassFailure{f.pivot};
            }
            try {
                Mat second_block =
                    project_dev(ctx_, n_, col(0), ld_, c0, s1, ld_, w, s1, ld_, sync, ortho_bytes);
                Upper outer_r = cholqr_dev(ctx_, n_, s1, ld_, w, col(c0), ld_, sync, ortho_bytes);
                Mat ir(w, w);
                for (i64 j = 0; j < w; ++j)
                    for (i64 i = 0; i <= j; ++i) ir(i, j) = inner_r(i, j);
                Mat corr = mat_mul_nn(second_block, ir);
                out.r_col = std::move(first_block);
                for (i64 j = 0; j < out.r_col.cols; ++j)
                    for (i64 i = 0; i < out.r_col.rows; ++i) out.r_col(i, j) += corr(i, j);
                out.r_jj = tri_mul(outer_r, inner_r);
                return out;
            } catch (const CholFail& f) {
                throw SecondPassBreakdown{f.pivot};
            }
        }
    }
    fail(KRY_INVALID_ARGUMENT, "unknown orthogonalization scheme");
}

void Store::commit(i64 c0, bool overlap, const OrthoRes& res, i64 w, int state) {
    // basis_store.hpp:285-327 (the q copy is unnecessary: run_scheme already
    // wrote the block into columns [c0, c0+w)).
    BlockRecord rec;
    rec.c0 = c0;
    rec.width = w;
    rec.overlap = overlap;
    const i64 rc = res.r_col.rows;
    if (overlap) {
        const double rho = r_(c0, c0);
        if (rc > 0) rec.carried.assign(res.r_col.col(0), res.r_col.col(0) + c0);
        rec.carried_diag = res.r_jj(0, 0);
        for (i64 i = 0; i < c0; ++i) r_.at(i, c0) += rho * res.r_col(i, 0);
        r_.at(c0, c0) = rho * res.r_jj(0, 0);
        for (i64 j = 1; j < w; ++j) {
            for (i64 i = 0; i < c0; ++i) r_.at(i, c0 + j) = res.r_col(i, j);
            for (i64 i = 0; i <= j; ++i) r_.at(c0 + i, c0 + j) = res.r_jj(i, j);
        }
    } else {
        for (i64 j = 0; j < w; ++j) {
            for (i64 i = 0; i < c0; ++i) r_.at(i, c0 + j) = (rc > 0) ? res.r_col(i, j) : 0.0;
            for (i64 i = 0; i <= j; ++i) r_.at(c0 + i, c0 + j) = res.r_jj(i, j);
        }
    }
    filled_ = c0 + w;
    seam_valid_ = false;
    if (state == KRY_PANEL_FINAL) {
        finalized_ = filled_;
        big_panel_start_ = filled_;
    } else {
        big_panel_start_ = std::min(big_panel_start_, c0);
        finalized_ = std::min(finalized_, c0);
    }
    states_.push_back(state);
    records_.push_back(std::move(rec));
}

Outcome Store::finalize_big_panel(Sync& sync, bool deferred) {
    const i64 before = sync.reduces;
    Outcome out;
    if (!big_panel_open()) return out;
    if (pending_) fail(KRY_INTERNAL, "a deferred finalize is still pending");
    const i64 c0 = big_panel_start_;
    const i64 w = filled_ - c0;
    OrthoRes res;
    try {
        Mat rc, g;
        if (fused_finalize_gram(c0, w, rc, g)) {
            sync.add(1);  // the last block's Gram: the panel's one reduce
            PipOut o = pip_from_gram(ctx_, n_, col(0), ld_, c0, col(c0), ld_, w, std::move(rc), std::move(g),
                                     col(c0), ld_, !deferred);
            // Same algorithmic bytes as the unfused finalize:
            // the Gram's reads of Q[:, 0:c_last) happened in the first stage.
            ortho_bytes += !deferred ? 8.0 * n_ * (2.0 * c0 + 3.0 * w) : 8.0 * n_ * (c0 + w);
            if (o.bad_pivot != 0) throw FirstPassFailure{o.bad_pivot};
            res = OrthoRes{std::move(o.r_col), std::move(o.r_jj)};
        } else {
            res = pip(c0, col(c0), ld_, w, col(c0), ld_, sync, true, /*do_update=*/!deferred);
        }
        std::fill(pready_.begin() + c0, pready_.end(), 0);
        if (deferred) {
            pending_ = true;
            pend_c0_ = c0;
            pend_w_ = w;
            pend_rcol_ = res.r_col;
            pend_rjj_ = res.r_jj;
        }
    } catch (const FirstPassFailure& e) {
        out.breakdown = true;
        out.pivot = e.pivot;
        out.kappa_estimate = diagnostic_kappa(c0, col(c0), ld_, w);
        sync.per_big_panel.push_back(sync.reduces - before);
        return out;
    }
    for (i64 c = c0; c < filled_; ++c) combine_column(c, c0, w, res);
    for (BlockRecord& rec : records_)
        if (rec.c0 >= c0) combine_record(rec, c0, w, res);
    finalized_ = filled_;
    big_panel_start_ = filled_;
    for (int& st : states_)
        if (st == KRY_PANEL_PREPROCESSED) st = KRY_PANEL_FINAL;
    out.committed = w;
    sync.per_big_panel.push_back(sync.reduces - before);
    return out;
}

bool Store::fused_finalize_gram(i64 c0, i64 w, Mat& r_col, Mat& g) {
    // The finalize Gram [Q_fin, P]ᵀP of the panel P = Q[:, c0:c0+w) from the
    // pieces the first-stage Grams already produced (the panel's leading
    // whole 8-column blocks) plus one narrow Gram of the trailing columns
    // against everything before them: the same numbers, but a ≤16-wide Gram
    // that streams at HBM speed instead of the compute-bound (w+1)-wide one.
    // Falls back (false) when no piece is there.
    if (!fused_panel_gram_) return false;
    i64 c_last = c0;  // first panel column without its products
    while (c_last < filled_ && pready_[static_cast<size_t>(c_last)]) ++c_last;
    const i64 wl = filled_ - c_last;
    if (c_last == c0 || wl < 1 || wl > 16) return false;
    Mat rc2, g2;
    gram_device(ctx_, n_, col(0), ld_, c_last, col(c_last), ld_, wl, rc2, g2);
    r_col = Mat(c0, w);
    g = Mat(w, w);
    for (i64 j = 0; j < w; ++j) {
        const i64 b = c0 + j;
        if (b < c_last) {
            for (i64 a = 0; a < c0; ++a) r_col(a, j) = pgram_(a, b);
            for (i64 i = 0; i <= j; ++i) g(i, j) = pgram_(c0 + i, b);
        } else {
            const i64 jj = b - c_last;
            for (i64 a = 0; a < c0; ++a) r_col(a, j) = rc2(a, jj);
            for (i64 i = 0; i <= j; ++i) {
                const i64 row = c0 + i;
                g(i, j) = row < c_last ? rc2(row, jj) : g2(row - c_last, jj);
            }
        }
    }
    for (i64 j = 0; j < w; ++j)
        for (i64 i = 0; i < j; ++i) g(j, i) = g(i, j);
    return true;
}

void Store::combine_column(i64 c, i64 c0, i64 w, const OrthoRes& res) {
    // basis_store.hpp:331-345
    std::vector<double> part(static_cast<size_t>(w), 0.0);
    const i64 top = std::min(c, c0 + w - 1);
    for (i64 i = c0; i <= top; ++i) part[i - c0] = r_(i, c);
    for (i64 i = 0; i < c0; ++i) {
        double s = 0.0;
        for (i64 l = 0; l < w; ++l) s += res.r_col(i, l) * part[l];
        r_.at(i, c) += s;
    }
    for (i64 i = 0; i < w && c0 + i <= c; ++i) {
        double s = 0.0;
        for (i64 l = i; l < w; ++l) s += res.r_jj(i, l) * part[l];
        r_.at(c0 + i, c) = s;
    }
}

void Store::combine_record(BlockRecord& rec, i64 c0, i64 w, const OrthoRes& res) {
    // basis_store.hpp:347-369.  Divergence: a
    // non-overlap record with c0 > 0 has no carried column; the reference
    // dereferences an empty vector there.  It is skipped (the solver never
    // produces one: only block 0 is non-overlap and it has c0 = 0).
    if (!rec.overlap && rec.c0 > 0) return;
    std::vector<double> full(static_cast<size_t>(rec.c0 + 1), 0.0);
    for (i64 i = 0; i < rec.c0; ++i) full[i] = rec.carried[i];
    full[rec.c0] = rec.carried_diag;
    std::vector<double> part(static_cast<size_t>(w), 0.0);
    const i64 top = std::min(rec.c0, c0 + w - 1);
    for (i64 i = c0; i <= top; ++i) part[i - c0] = full[i];
    for (i64 i = 0; i < c0; ++i) {
        double s = 0.0;
        for (i64 l = 0; l < w; ++l) s += res.r_col(i, l) * part[l];
        full[i] += s;
    }
    for (i64 i = 0; i < w && c0 + i <= rec.c0; ++i) {
        double s = 0.0;
        for (i64 l = i; l < w; ++l) s += res.r_jj(i, l) * part[l];
        full[c0 + i] = s;
    }
    for (i64 i = 0; i < rec.c0; ++i) rec.carried[i] = full[i];
    rec.carried_diag = full[rec.c0];
}

void Store::record_seam(const double* dropped, Sync& sync) {
    // basis_store.hpp:374-381: coefficients of the first dropped raw vector.
    if (filled_ >= max_cols_) return;
    sync.add(1);
    Mat rc, g;
    gram_device(ctx_, n_, col(0), ld_, filled_, dropped, ld_, 1, rc, g);
    for (i64 i = 0; i < filled_; ++i) r_.at(i, filled_) = rc(i, 0);
    r_.at(filled_, filled_) = 0.0;
    seam_valid_ = true;
}

double Store::diagnostic_kappa(i64 c0, const double* V, i64 ldv, i64 w) {
    // basis_store.hpp:383-387 → accumulated_cond on host copies.  The
    // diagnostic needs every row, so a multi-rank run reports 0.
    if (c0 + w > 512 || ctx_.nranks > 1) return 0.0;
    Mat q(n_, c0), x(n_, w);
    if (c0 > 0)
        KB_CUDA(cudaMemcpy2DAsync(q.a.data(), n_ * 8, col(0), ld_ * 8, n_ * 8, c0, cudaMemcpyDeviceToHost,
                                  ctx_.stream));
    KB_CUDA(cudaMemcpy2DAsync(x.a.data(), n_ * 8, V, ldv * 8, n_ * 8, w, cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
    return accumulated_cond(q, x);
}

}  // namespace kb
