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

// CholQR (block_ortho.hpp:49-54) on the device: adds its one reduce to
// `reduces` (also when it fails), writes Q = V·R⁻¹ to `out`; a Cholesky
// failure throws CholFail{pivot} (callers map it to the reference's
// first / second-pass semantics or to NotPositiveDefinite).
struct CholFail {
    i64 pivot;
};
Upper cholqr_device(Ctx& ctx, i64 n, const double* V, i64 ldv, i64 w, double* out, i64 ldo, i64& reduces,
                    double& bytes);

// bcgs_project (block_ortho.hpp:70-87): R_block = PᵀV (one reduce when
// c0 > 0), out = V − P·R_block (out may alias V).
Mat project_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                   double* out, i64 ldo, i64& reduces, double& bytes);

// bcgs2 (block_ortho.hpp:102-137) with the CholQR2 intra step (CholQR on a
// single column): project, intra, re-project, CholQR; R_col = T_col·R_in +
// R_col, R_jj = R_out·R_in.  Scratch s0 / s1: n × w each (ld lds).  Throws
// CholFail.  The HHQR intra step is not on the device path.
struct Bcgs2Out {
    Mat r_col;
    Upper r_jj;
};
Bcgs2Out bcgs2_device(Ctx& ctx, i64 n, const double* P, i64 ldp, i64 c0, const double* V, i64 ldv, i64 w,
                      double* s0, double* s1, i64 lds, double* out, i64 ldo, i64& reduces, double& bytes);

}  // namespace kb
