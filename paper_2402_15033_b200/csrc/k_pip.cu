// Device-side BCGS-PIP factorisation for speculative first-stage blocks.
//
// The host path (kb_ortho.cpp pip_from_gram) waits for every Gram, runs the
// Pythagorean update and try_cholesky on the CPU and sends the update
// coefficients back — one host round trip per block.  For the two-stage
// first stage the outcome is almost always "committed at full width", so the
// solver can queue a whole big panel of blocks without waiting: this kernel
// (one CTA per block) does the same arithmetic on the device, in the same
// operation order with no contraction (bit-identical to the host), writes the
// update coefficients for K5 and a result slot the host replays later
// (Store::resolve_speculative).  A failed Cholesky — or any failure earlier in
// the chain — sets the block's skip flag, so its update never overwrites the
// raw block and the host can redo it on the synchronous path.
#include <cuda_runtime.h>

#include "kb_common.hpp"
#include "kb_device.hpp"
#include "kb_kernels.hpp"

namespace kb {

namespace {

constexpr int kPipThreads = 256;
constexpr int kPipMaxC0 = 64, kPipMaxW = 8;

__global__ void __launch_bounds__(kPipThreads) pip_block_kernel(const PipBlockArgs a) {
    KB_PDL_WAIT();
    __shared__ double rc[kPipMaxC0 * kPipMaxW];  // R_col, column-major c0 × w
    __shared__ double s[kPipMaxW * kPipMaxW];    // G, then S = G − R_colᵀR_col
    __shared__ double r[kPipMaxW * kPipMaxW];    // R_jj (upper), column-major
    __shared__ int bad;
    const int c0 = a.c0, w = a.w, tid = threadIdx.x;
    // 1. unpack the packed Gram tiles: the nb regular tiles (slot block t:
    //    rows 8t + m, V column nn) then the extra prefix × prefix tiles.  One
    //    flat loop over all entries so the L2 loads are independent.
    double* pieces = a.slot + kSlotPieces;
    const int nreg = a.nb * 64, ntot = nreg + a.nx * (a.nb - 1) * 64;
    // all loads first (≤ 22 tiles · 64 / 256 threads = 6 per thread), so the
    // L2 round trips overlap instead of serialising behind the scatter
    constexpr int kPer = (22 * 64 + kPipThreads - 1) / kPipThreads;
    double vals[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int idx = tid + u * kPipThreads;
        vals[u] = idx < ntot ? a.packed[idx] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int idx = tid + u * kPipThreads;
        if (idx >= ntot) break;
        const double v = vals[u];
        const int e = idx & 63;
        if (idx < nreg) {
            const int mrow = 8 * (idx >> 6) + (e & 7), j = e >> 3;
            if (j >= w) continue;
            if (mrow < 8) {
                if (mrow < w) s[mrow + j * kPipMaxW] = v;  // upper and lower: mirrored below
            } else if (mrow - 8 < c0) {
                rc[(mrow - 8) + j * c0] = v;
            }
        } else {
            const int xt = (idx - nreg) >> 6, k = xt / (a.nb - 1), ib = 1 + xt % (a.nb - 1);
            const int ar = 8 * ib + (e & 7) - 8, bc = 8 * (a.xb0 + k) + (e >> 3) - 8 - a.x_first;
            if (ar >= 0 && ar < c0 && bc >= 0 && bc < a.x_count) pieces[ar + bc * c0] = v;
        }
    }
    __syncthreads();
    // mirror the upper triangle of VᵀV (gram(), dense_kernels.hpp:95-105)
    for (int idx = tid; idx < w * w; idx += kPipThreads) {
        const int i = idx % w, j = idx / w;
        if (i > j) s[i + j * kPipMaxW] = s[j + i * kPipMaxW];
    }
    __syncthreads();
    if (a.mode == 1) {
        // bcgs_project (block_ortho.hpp:70-87): R_block = Q_prevᵀV as it is,
        // update V − Q_prev·R_block (K5 coefficients −R_col, no intra factor:
        // the host path's update_device(…, triangular = false)); the chain
        // status passes through (an earlier failure skips this update too).
        const int piv = (a.prev_slot && a.prev_slot[kSlotStatus] != 0.0) ? -1 : 0;
        if (tid == 0) {
            a.slot[kSlotStatus] = static_cast<double>(piv);
            *a.skip = piv != 0 ? 1 : 0;
        }
        double* rcol_out = a.slot + kSlotRcol;
        for (int idx = tid; idx < c0 * w; idx += kPipThreads) rcol_out[idx] = rc[idx];
        if (piv != 0) return;
        const int wm = a.wmax;
        for (int idx = tid; idx < (c0 + wm + 1) * wm; idx += kPipThreads) {
            const int row = idx / wm, j = idx % wm;
            double v = 0.0;
            if (row < c0) {
                if (j < w) v = -rc[row + j * c0];
            } else if (row == c0 + wm) {
                if (j < w) v = 1.0;
            }
            a.coef[idx] = v;
        }
        return;
    }
    // 2. Pythagorean update, one (i ≤ j) entry per thread, dot in index
    //    order (block_ortho.hpp:159-166 via dot_seq).
    for (int idx = tid; idx < w * w; idx += kPipThreads) {
        const int i = idx % w, j = idx / w;
        if (i > j || c0 == 0) continue;
        double c = 0.0;
        for (int l = 0; l < c0; ++l) c = __dadd_rn(c, __dmul_rn(rc[l + i * c0], rc[l + j * c0]));
        s[i + j * kPipMaxW] = __dsub_rn(s[i + j * kPipMaxW], c);
    }
    __syncthreads();
    for (int idx = tid; idx < w * w; idx += kPipThreads) {
        const int i = idx % w, j = idx / w;
        if (i > j) s[i + j * kPipMaxW] = s[j + i * kPipMaxW];
    }
    __syncthreads();
    // 3. try_cholesky (dense_kernels.hpp:111-127), row by row on one warp.
    //    Every entry keeps the reference's exact operation sequence
    //    (r_ij = (s_ij − Σ_{k<i} r_ki·r_kj in k order) / r_ii, the diagonal
    //    likewise then sqrt), so the factor is bit-identical; only independent
    //    entries run concurrently: the critical path is w sqrt + w divisions
    //    instead of w sqrt + w(w−1)/2 divisions.  The first non-positive
    //    diagonal is the reference's pivot (row i's diagonal needs exactly the
    //    columns < i the reference has finished when it reaches column i).
    if (tid < 32) {
        int piv = 0;
        if (a.prev_slot && a.prev_slot[kSlotStatus] != 0.0) piv = -1;  // an earlier block failed
        for (int i = 0; i < w && piv == 0; ++i) {
            double d = s[i + i * kPipMaxW];  // every lane: same value, no broadcast
            for (int k = 0; k < i; ++k) d = __dsub_rn(d, __dmul_rn(r[k + i * kPipMaxW], r[k + i * kPipMaxW]));
            if (!(d > 0.0)) {
                piv = i + 1;
                break;
            }
            const double rii = __dsqrt_rn(d);
            const int j = tid;
            if (j == i) r[i + i * kPipMaxW] = rii;
            if (j > i && j < w) {
                double acc = s[i + j * kPipMaxW];
                for (int k = 0; k < i; ++k)
                    acc = __dsub_rn(acc, __dmul_rn(r[k + i * kPipMaxW], r[k + j * kPipMaxW]));
                r[i + j * kPipMaxW] = __ddiv_rn(acc, rii);
            }
            __syncwarp();
        }
        if (tid == 0) {
            bad = piv;
            a.slot[kSlotStatus] = static_cast<double>(piv);
            *a.skip = piv != 0 ? 1 : 0;
        }
    }
    __syncthreads();
    // 4. result slot (host replay) and the K5 coefficients
    //    (update_device layout: −R_col[c0][wmax], −R_jj[wmax][wmax], 1/r_jj).
    double* rcol_out = a.slot + kSlotRcol;
    double* rjj_out = rcol_out + c0 * w;
    for (int idx = tid; idx < c0 * w; idx += kPipThreads) rcol_out[idx] = rc[idx];
    for (int idx = tid; idx < w * w; idx += kPipThreads) {
        const int i = idx % w, j = idx / w;
        rjj_out[idx] = (i <= j && bad == 0) ? r[i + j * kPipMaxW] : 0.0;
    }
    if (bad != 0) return;
    const int wm = a.wmax;
    double* nrc = a.coef;
    double* nrjj = nrc + c0 * wm;
    double* inv = nrjj + wm * wm;
    for (int idx = tid; idx < (c0 + wm + 1) * wm; idx += kPipThreads) {
        const int row = idx / wm, j = idx % wm;
        double v = 0.0;
        if (row < c0) {
            if (j < w) v = -rc[row + j * c0];
        } else if (row < c0 + wm) {
            const int l = row - c0;
            if (j < w && l < j) v = -r[l + j * kPipMaxW];
        } else {
            if (j < w) v = __drcp_rn(r[j + j * kPipMaxW]);
        }
        nrc[idx] = v;
    }
}

}  // namespace

void launch_pip_block(cudaStream_t stream, const PipBlockArgs& a, int64_t& launches) {
    if (a.c0 > kPipMaxC0 || a.w > kPipMaxW || a.w < 1) fail(KRY_INTERNAL, "speculative block shape");
    launch_pdl(pip_block_kernel, 1, kPipThreads, 0, stream, a);
    KB_LAUNCHED();
    launches += 1;
}

}  // namespace kb
