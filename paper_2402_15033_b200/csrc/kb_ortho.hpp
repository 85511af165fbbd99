// Device BCGS-PIP (block_ortho.hpp:152-189): fused Gram on the GPU → one
// allreduce of the (c0+w)×w Gram → Pythagorean Cholesky on the host
// (replicated per rank) → fused update kernel, in place over the store.
#pragma once

#include "kb_ctx.hpp"
#include "kb_dense.hpp"

namespace kb {

struct PipOut {
    Mat r_col;       // c0 × w
    Upper r_jj;      // w × w (partial factor on failure)
    i64 bad_pivot = 0;
};

// R_col = Pᵀ V (c0×w) and G = VᵀV (w×w, upper computed and mirrored, as
// gram(), dense_kernels.hpp:95-105), summed over ranks.
void gram_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                 Mat& r_col, Mat& g, i64 x_first = -1, i64 x_count = 0, Mat* gx = nullptr);
// Optional extra output (first-stage shapes): gx = P[:, 0:c0]ᵀ·P[:, x_first:x_first+x_count]
// (c0 × x_count), from the same launch and the same allreduce.

// The part of bcgs_pip_partial after the Gram: Pythagorean update, Cholesky,
// (update).  r_col / g as returned by gram_device.
PipOut pip_from_gram(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                     Mat r_col, Mat g, double* out, i64 ldo, bool do_update);

// out = (V − P·R_col)·R_jj⁻¹ (block_ortho.hpp:171-176 + tri_solve_right).
void update_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                   const Mat& r_col, const Upper& r_jj, double* out, i64 ldo, bool triangular = true);

// bcgs_pip_partial: adds 1 to `reduces`; writes the block to `out` only when
// the Pythagorean Cholesky succeeds (bad_pivot == 0).
PipOut bcgs_pip_partial_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V,
                               i64 ldv, i64 w, double* out, i64 ldo, i64& reduces, bool do_update = true,
                               i64 x_first = -1, i64 x_count = 0, Mat* gx = nullptr);

}  // namespace kb
