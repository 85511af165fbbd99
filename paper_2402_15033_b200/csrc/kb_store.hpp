// Device-resident basis store (krylov::BasisStore, basis_store.hpp:42-401).
//
// Q lives in HBM as one column-major n×(m+1) allocation (ld padded for TMA);
// the MPK writes each block straight into its columns and BCGS-PIP rewrites
// them in place, so a block never round-trips through a separate buffer.  R,
// the block records and the panel state machine are host-side and follow
// the reference operation for operation (they are O(m²) and replicated per
// rank).
#pragma once

#include <vector>

#include "kb_ctx.hpp"
#include "kb_dense.hpp"
#include "kb_operator.hpp"

namespace kb {

struct Sync {  // SyncCounter (block_ortho.hpp:15-21)
    i64 reduces = 0;
    std::vector<i64> per_block, per_big_panel;
    void add(i64 k = 1) { reduces += k; }
};

struct Outcome {  // AppendOutcome (basis_store.hpp:16-22)
    i64 committed = 0;
    bool truncated = false;
    bool breakdown = false;
    i64 pivot = 0;
    double kappa_estimate = 0.0;
};

class Store {
public:
    Store(Ctx& ctx, i64 n, i64 m, i64 panel_size, i64 big_panel_size);

    i64 rows() const { return n_; }
    i64 capacity() const { return max_cols_; }
    i64 filled() const { return filled_; }
    i64 finalized_count() const { return finalized_; }
    i64 big_panel_start() const { return big_panel_start_; }
    i64 panel_size() const { return panel_size_; }
    i64 big_panel_size() const { return big_panel_size_; }
    bool big_panel_open() const { return filled_ > big_panel_start_; }
    bool big_panel_full() const { return big_panel_open() && filled_ - big_panel_start_ >= big_panel_size_ + 1; }
    bool has_seam_column() const { return seam_valid_; }
    const Upper& coefficients() const { return r_; }
    const std::vector<int>& panel_states() const { return states_; }
    const std::vector<BlockRecord>& block_records() const { return records_; }
    double* col(i64 j) { return q_.p + (j + qoff_) * ld_; }
    const double* col(i64 j) const { return q_.p + (j + qoff_) * ld_; }
    // KRY_GUARD=1 (debug, read at construction): the basis is allocated with a
    // guard column on each side, and the guard columns and every column's
    // padding rows [n, ld) hold an all-ones NaN pattern that no kernel may
    // write (and none may read without poisoning its result) — an
    // out-of-bounds check of every kernel that touches the store, for a pool
    // where compute-sanitizer is unavailable.  check_guards() fails loudly.
    bool guarded() const { return qoff_ != 0; }
    void check_guards();
    i64 ld() const { return ld_; }
    Ctx& ctx() { return ctx_; }

    void reset();
    void zero_q();
    void seed_unit_column(const double* d_v);
    // V (device, n×w, leading dimension ldv) may be the store's own columns
    // [c0, c0+w) (in-place path used by the solver's MPK) or a caller buffer.
    Outcome append_block(const double* V, i64 ldv, i64 w, bool overlap, int kind, i64 big_panel,
                         Sync& sync);
    Outcome preprocess_block(const double* V, i64 ldv, i64 w, bool overlap, Sync& sync);
    // `deferred`: leave Q[:, c0:filled) as the preprocessed panel and keep the
    // finalize transform (R_col, R_jj) pending — valid only when nothing but
    // the solution update reads the panel afterwards (the cycle's last panel).
    Outcome finalize_big_panel(Sync& sync, bool deferred = false);
    // Pending deferred finalize: x += Q_fin[:, 0:k]·y becomes the same
    // update over the stored columns with y' = (y_pre − R_col·z, z),
    // z = R_jj⁻¹·y_panel.  Returns false when nothing is pending.
    bool deferred_coefficients(const std::vector<double>& y, std::vector<double>& y_out) const;
    // ---- speculative first stage (two-stage scheme; k_pip.cu) -------------
    // preprocess_speculative() queues Gram → [allreduce] → device
    // factorisation → flag-gated update for the block in store columns
    // [c0, c0+w) (c0 from the *predicted* fill: every queued block assumed
    // committed at full width) without waiting for the GPU.
    // resolve_speculative() copies the result slots back (one sync) and
    // replays the host bookkeeping block by block exactly as
    // preprocess_block() would; it returns the queue index of the first block
    // whose factorisation failed (its raw columns are intact: the caller
    // redoes it on the synchronous path) or −1.
    bool can_speculate(i64 w) const;
    void preprocess_speculative(i64 w, bool overlap);
    // Fused first stage (K6, 2-D stencil, one rank): the queue's first block
    // runs MPK → Gram → factorisation into a raw buffer outside the store
    // and leaves its update pending; every later block is one fused pass
    // (pending update → MPK → Gram, k_fused.cu) + factorisation;
    // spec_flush() runs the last pending update (before resolve).
    bool can_fuse(const Operator& op, i64 s);
    void spec_fused_first(Operator& op, i64 s, bool overlap);
    void spec_fused_next(Operator& op, i64 s);
    void spec_flush();
    i64 resolve_speculative(Sync& sync);
    // ---- speculative one-stage BCGS-PIP2 (run_scheme BcgsPip2,
    // basis_store.hpp:220-239) -------------------------------------------
    // preprocess_speculative_pip2() queues both passes of a block (Gram →
    // [allreduce] → device factorisation → gated update, twice: V → scratch
    // → store columns) without waiting.  The one-stage solver checks
    // convergence after every block, so the queue is replayed one block at
    // a time: spec_fetch() copies the result slots back (one sync),
    // spec_commit_next() replays the next block's bookkeeping exactly as
    // append_block() would (R = composed passes, 2 reduces) and returns 1,
    // or 0 when that block's factorisation failed (its raw columns are
    // intact for the synchronous redo), or −1 when the queue is exhausted;
    // spec_drop() discards what is left (the cycle ended early).
    bool can_speculate_pip2(i64 w) const;
    void preprocess_speculative_pip2(i64 w, bool overlap);
    // ---- speculative standard GMRES (s = 1: BCGS2 with one column,
    // block_ortho.hpp:102-137) -------------------------------------------
    // preprocess_speculative_std() queues the four passes of the column in
    // store column c0 = spec_filled() (project → CholQR → project → CholQR:
    // Gram → [allreduce] → device coefficients → gated update, V → scratch →
    // scratch → scratch → store column) without waiting; replayed one column
    // at a time by spec_commit_next() (R composed as run_scheme's BCGS2, 4
    // reduces).  can_speculate_std(c0): the prefix fits one Gram group.
    bool can_speculate_std(i64 c0) const;
    void preprocess_speculative_std();
    void spec_fetch();
    int spec_commit_next(Sync& sync);
    bool spec_has_next() const { return spec_fetched_ && spec_next_ < spec_.size(); }
    void spec_drop();
    i64 spec_filled() const { return spec_.empty() ? filled_ : spec_filled_; }
    bool spec_panel_full() const;
    // MPK into the store: column c0 holds the start; columns c0+1..c0+s.
    // Returns true when the fused one-pass kernel ran.
    bool mpk(Operator& op, i64 c0, i64 s);

    // Telemetry: algorithmic BlkOrtho bytes for this rank.
    double ortho_bytes = 0.0;

private:
    struct OrthoRes {
        Mat r_col;
        Upper r_jj;
    };
    struct SecondPassBreakdown {
        i64 pivot;
    };
    struct FirstPassFailure {
        i64 pivot;
    };

    Outcome append_impl(const double* V, i64 ldv, i64 w, bool overlap, int kind, Sync& sync);
    // Writes the orthonormal block into store columns [c0, c0+w).
    OrthoRes run_scheme(i64 c0, const double* V, i64 ldv, i64 w, int kind, Sync& sync);
    OrthoRes pip(i64 c0, const double* V, i64 ldv, i64 w, double* out, i64 ldo, Sync& sync, bool first_pass,
                 bool do_update = true, i64 x_first = -1, i64 x_count = 0);
    // Panel Gram pieces accumulated by the first-stage Grams (fused finalize):
    // pgram_(a, b) = q_aᵀq_b for the preprocessed column b (pready_[b]) and a < b.
    bool fused_panel_gram_ = true;
    Mat pgram_;
    std::vector<char> pready_;
    bool fused_finalize_gram(i64 c0, i64 w, Mat& r_col, Mat& g);
    struct SpecBlock {
        i64 c0, w;
        bool overlap;
        i64 x_first, x_count;
        const double* raw;  // raw block outside the store (fused path) or nullptr
        bool pip2 = false;  // one-stage BCGS-PIP2: result slots 2i (pass 1) and 2i + 1 (pass 2)
        bool std1 = false;  // standard GMRES column: result slots 4i … 4i + 3 (the four BCGS2 passes)
    };
    struct SpecPlan {
        i64 c0, idx, xf, xc;
    };
    SpecPlan spec_plan(i64 w, bool overlap, bool pieces = true);
    PipBlockArgs spec_factor(const SpecPlan& p, i64 w, int mode = 0);
    void spec_push(const SpecPlan& p, i64 w, bool overlap, const double* raw);
    struct FusedPending {
        bool live = false;
        i64 c0 = 0, w = 0;
        int buf = 0;
        double* coef = nullptr;
        int* skip = nullptr;
    };
    FusedPending fpend_;
    DevBuf fraw_[2];  // raw blocks of the fused path (double-buffered)
    std::vector<SpecBlock> spec_;
    size_t spec_next_ = 0;      // next queued block to replay (after spec_fetch)
    bool spec_fetched_ = false;
    i64 spec_filled_ = 0, spec_bps_ = 0, spec_xd_ = 0;
    DevBuf spec_slots_, spec_coef_, spec_skip_;
    HostBuf spec_host_;
    bool pending_ = false;  // deferred finalize transform below applies to Q[:, pend_c0_:pend_c0_+pend_w_)
    i64 pend_c0_ = 0, pend_w_ = 0;
    Mat pend_rcol_;
    Upper pend_rjj_;
    void commit(i64 c0, bool overlap, const OrthoRes& res, i64 w, int state);
    void combine_column(i64 col, i64 c0, i64 w, const OrthoRes& res);
    void combine_record(BlockRecord& rec, i64 c0, i64 w, const OrthoRes& res);
    void record_seam(const double* dropped, Sync& sync);
    double diagnostic_kappa(i64 c0, const double* V, i64 ldv, i64 w);
    double* scratch(int which, i64 w);

    Ctx& ctx_;
    i64 n_, max_cols_, panel_size_, big_panel_size_;
    i64 filled_ = 0, finalized_ = 0, big_panel_start_ = 0;
    bool seam_valid_ = false;
    DevBuf q_;
    i64 qoff_ = 0;  // 1 with guard columns (KRY_GUARD)
    void fill_guards();
    i64 ld_;
    Upper r_;
    std::vector<int> states_;
    std::vector<BlockRecord> records_;
    DevBuf scratch_[2];
};

}  // namespace kb
