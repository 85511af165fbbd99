// Tall-skinny BlkOrtho kernels for sm_100a (K3 fused Gram, K5/K5t/K5b updates).
//
// The Gram and the TMA updates stream row tiles of [V | P] (V = the block
// being orthogonalized, w ≤ 64 columns; P = prefix basis columns) from HBM
// into shared memory with 2-D TMA loads (cp.async.bulk.tensor, mbarrier
// complete_tx) through a multi-stage ring driven by one producer warp, and
// consume them with 4–8 compute warps.  Every byte is read from HBM once per
// launch.
//
//  * gram_kernel<NBW, NB, NX>: G = [V | P]ᵀ·V on the DMMA pipe (mma.m8n8k4
//    f64).  The Gram is the reduction over rows, so rows are the MMA k
//    dimension and an 8×8 output tile is spread over the 32 lanes (2 doubles
//    per lane): the whole (c0+w)×w output (≤ 36 tiles, upper triangle only
//    for VᵀV, which is what gram() computes, dense_kernels.hpp:95-105) stays
//    in registers for the launch.  A fragment for column block b is the same
//    for the A and the B operand, so one conflict-free LDS per block per four
//    rows feeds every tile of that block.  NX extra tiles return panel-Gram
//    pieces (kb_store.cpp).  Per-CTA partials are reduced by
//    gram_reduce_kernel in a fixed order (deterministic, no float atomics).
//  * update_tma_kernel (K5t) / update_kernel (K5): Q = (V − P·R_col)·R_jj⁻¹
//    row-locally in the order of bcgs_pip_partial's update + tri_solve_right
//    (block_ortho.hpp:171-176, dense_kernels.hpp:139-154): vhat_j = V_j −
//    Σ_l R_col(l,j)·p_l (l ascending), x_j = vhat_j − Σ_{l<j} R(l,j)·x_l,
//    x_j *= 1/R(j,j).  K5t streams P through a TMA ring in 16-column chunks,
//    K5 loads it directly; both write the block in place over the store.
//  * update_pair_kernel (w 33..64) and update_mma_kernel (K5b, a DMMA GEMM
//    against the explicit inverse for well-conditioned wide R).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "kb_common.hpp"
#include "kb_device.hpp"
#include "kb_kernels.hpp"

namespace kb {

namespace {

using namespace dev;

// Consumer warps per CTA: 8 while the accumulators are small, 4 for the
// widest Gram shapes (≥ 30 register-resident tiles) to stay spill-free.
__host__ __device__ constexpr int consumer_warps(int nbw) { return nbw >= 5 ? 4 : 8; }
constexpr int kSmemBudget = 200 * 1024;

struct TsParams {
    i64 n;          // rows
    i64 ntiles;     // ceil(n / tr)
    int tr;         // rows per tile
    int w;          // V columns
    int wslots;     // round_up(w, 8)
    int cp;         // P columns in this pass
    int cpslots;    // round_up(cp, 8)
    int stages;
    int vv;         // gram: compute the VᵀV tiles in this pass
    int consumers;  // consumer warps (empty-barrier arrival count)
    int xb0;        // gram: first extra P slot block (NX > 0)
    unsigned tx_bytes;
};

// Shared ring set-up common to both kernels.  Returns the stage base.
__device__ __forceinline__ double* ring_setup(unsigned char* smem, const TsParams& p,
                                              uint64_t*& full, uint64_t*& empty) {
    const int slots = p.wslots + p.cpslots;
    const size_t stage_doubles = static_cast<size_t>(slots) * p.tr;
    double* ring = reinterpret_cast<double*>(smem);
    full = reinterpret_cast<uint64_t*>(smem + stage_doubles * 8 * p.stages);
    empty = full + p.stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.consumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // Zero the padding slots (never written by TMA) of every stage.
    const int padv = p.wslots - p.w, padp = p.cpslots - p.cp;
    if (padv + padp > 0) {
        for (int s = 0; s < p.stages; ++s) {
            double* st = ring + s * stage_doubles;
            for (int idx = threadIdx.x; idx < (padv + padp) * p.tr; idx += blockDim.x) {
                const int slot_i = idx / p.tr, r = idx % p.tr;
                const int slot = slot_i < padv ? p.w + slot_i : p.wslots + p.cp + (slot_i - padv);
                st[static_cast<size_t>(slot) * p.tr + r] = 0.0;
            }
        }
    }
    __syncthreads();
    return ring;
}

// Producer loop (one elected lane of the producer warp).  Stage index and
// use count advance incrementally (no integer division per tile).
__device__ __forceinline__ void ring_produce(const CUtensorMap* map_v, const CUtensorMap* map_p,
                                            const TsParams& p, double* ring, uint64_t* full,
                                            uint64_t* empty) {
    const size_t stage_doubles = static_cast<size_t>(p.wslots + p.cpslots) * p.tr;
    int s = 0, use = 0;
    for (i64 tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        double* st = ring + s * stage_doubles;
        mbar_expect_tx(&full[s], p.tx_bytes);
        const int row0 = static_cast<int>(tile * p.tr);
        tma_load_2d(st, map_v, row0, 0, &full[s]);
        if (p.cp > 0) tma_load_2d(st + static_cast<size_t>(p.wslots) * p.tr, map_p, row0, 0, &full[s]);
        if (++s == p.stages) {
            s = 0;
            ++use;
        }
    }
}

// Tiles of the Gram, in (jb, ib) order: jb < NBW indexes the V column blocks
// (output columns), ib < NB the [V | P] column blocks (output rows); the
// VᵀV part keeps only ib ≤ jb (gram() computes the upper triangle).
__host__ __device__ constexpr bool tile_valid(int nbw, int jb, int ib) { return ib >= nbw || ib <= jb; }
__host__ __device__ constexpr int tile_pos(int nbw, int nb, int jb, int ib) {
    int t = 0;
    for (int j = 0; j < nbw; ++j)
        for (int i = 0; i < nb; ++i) {
            if (!tile_valid(nbw, j, i)) continue;
            if (j == jb && i == ib) return t;
            ++t;
        }
    return -1;
}
__host__ __device__ constexpr int tile_count(int nbw, int nb) {
    int t = 0;
    for (int j = 0; j < nbw; ++j)
        for (int i = 0; i < nb; ++i) t += tile_valid(nbw, j, i) ? 1 : 0;
    return t;
}

// ---------------------------------------------------------------------------
// K3: fused Gram  G = [V | P]ᵀ V  on DMMA (mma.m8n8k4.f64).
//   Blocks of 8 columns: b < NBW are V blocks, NBW ≤ b < NB are P blocks.
//   Rows are the MMA k dimension: each 4-row chunk contributes one DMMA per
//   tile; a lane's fragment for block b is X[r0 + lane%4][8b + lane/4]
//   for both operands, so one LDS per block feeds every tile of the block.
//   The smem column stride tr ≡ 4 (mod 16) makes those loads conflict-free.
// ---------------------------------------------------------------------------
// NX > 0 (first-stage shapes only): additionally accumulate P_blocksᵀ·X for
// the NX 8-column P blocks starting at block p.xb0 — the just-preprocessed
// columns of the previous block, which the two-stage finalize needs
// (Store::pgram_).  They ride on data this launch streams anyway.
template <int NBW, int NB, int NX = 0, int CW = consumer_warps(NBW)>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    gram_kernel(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_p,
                const TsParams p, double* __restrict__ partials) {
    KB_PDL_WAIT();
    constexpr int T = tile_count(NBW, NB) + NX * (NB - NBW);
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full, *empty;
    double* ring = ring_setup(smem, p, full, empty);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t stage_doubles = static_cast<size_t>(p.wslots + p.cpslots) * p.tr;

    if (warp == CW) {
        if (lane == 0) ring_produce(&map_v, &map_p, p, ring, full, empty);
        return;
    }

    double acc[NBW][NB][2];
#pragma unroll
    for (int jb = 0; jb < NBW; ++jb)
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) acc[jb][ib][0] = acc[jb][ib][1] = 0.0;
    double accx[NX > 0 ? NX : 1][NB][2];
#pragma unroll
    for (int k = 0; k < (NX > 0 ? NX : 1); ++k)
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) accx[k][ib][0] = accx[k][ib][1] = 0.0;
    const int xb0 = p.xb0;

    const int frag_off = (lane >> 2) * p.tr + (lane & 3);
    const int nchunks = p.tr / 4;
    const bool vv = p.vv != 0;
    int s = 0, use = 0, rot = warp;
    for (i64 tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        mbar_wait(&full[s], use & 1);
        const double* st = ring + s * stage_doubles + frag_off;
#pragma unroll 2
        for (int c = rot; c < nchunks; c += CW) {
            const double* base = st + 4 * c;
            double f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = base[static_cast<size_t>(8 * b) * p.tr];
#pragma unroll
            for (int jb = 0; jb < NBW; ++jb)
#pragma unroll
                for (int ib = 0; ib < NB; ++ib) {
                    if (!tile_valid(NBW, jb, ib)) continue;
                    if (ib >= NBW || vv) dmma(acc[jb][ib][0], acc[jb][ib][1], f[ib], f[jb]);
                }
            if constexpr (NX > 0) {
#pragma unroll
                for (int k = 0; k < NX; ++k) {
                    const double fx = base[static_cast<size_t>(8 * (xb0 + k)) * p.tr];
#pragma unroll
                    for (int ib = NBW; ib < NB; ++ib)
                        if (ib <= xb0 + k) dmma(accx[k][ib][0], accx[k][ib][1], f[ib], fx);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        rot = (rot + 1) & (CW - 1);
        if (++s == p.stages) {
            s = 0;
            ++use;
        }
    }

    // Cross-warp reduction in fixed warp order, through the (now idle) ring.
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
    double* scratch = ring;  // [warp][T][64]
    const int e0 = (lane >> 2) + 8 * (2 * (lane & 3));
#pragma unroll
    for (int jb = 0; jb < NBW; ++jb)
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
            if (!tile_valid(NBW, jb, ib)) continue;
            double* t = scratch + (static_cast<size_t>(warp) * T + tile_pos(NBW, NB, jb, ib)) * 64;
            t[e0] = acc[jb][ib][0];
            t[e0 + 8] = acc[jb][ib][1];
        }
    if constexpr (NX > 0) {  // extra tiles after the regular ones, (k, ib) order
#pragma unroll
        for (int k = 0; k < NX; ++k)
#pragma unroll
            for (int ib = NBW; ib < NB; ++ib) {
                double* t = scratch +
                            (static_cast<size_t>(warp) * T + tile_count(NBW, NB) + k * (NB - NBW) + (ib - NBW)) * 64;
                t[e0] = accx[k][ib][0];
                t[e0 + 8] = accx[k][ib][1];
            }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
    constexpr int per_cta = T * 64;
    double* out = partials + static_cast<size_t>(blockIdx.x) * per_cta;
    for (int e = threadIdx.x; e < per_cta; e += CW * 32) {
        double sum = scratch[e];
#pragma unroll
        for (int w = 1; w < CW; ++w) sum += scratch[static_cast<size_t>(w) * per_cta + e];
        out[e] = sum;
    }
}

// One warp per output entry: lanes sum the per-CTA partials with a fixed
// stride, then a fixed xor tree.  Deterministic for a given grid size.
__global__ void gram_reduce_kernel(const double* __restrict__ partials, int grid, int per_cta,
                                   double* __restrict__ packed) {
    KB_PDL_WAIT();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= per_cta) return;
    double s = 0.0;
    for (int c = lane; c < grid; c += 32) s += partials[static_cast<size_t>(c) * per_cta + gw];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) packed[gw] = s;
}

template <int NBW, int NB>
const void* gram_fn(int nbw, int nb) {
    if (nbw == NBW && nb == NB) return reinterpret_cast<const void*>(gram_kernel<NBW, NB>);
    if constexpr (NB < 8) {
        return gram_fn<NBW, NB + 1>(nbw, nb);
    } else if constexpr (NBW < 8) {
        return gram_fn<NBW + 1, NBW + 1>(nbw, nb);
    } else {
        return nullptr;
    }
}

// First-stage Gram (NBW = 1) with NX ∈ {1, 2} extra P-column blocks.
template <int NB>
const void* gram_x_fn(int nb, int nx) {
    if (nb == NB) {
        if (nx == 1) return reinterpret_cast<const void*>(gram_kernel<1, NB, 1>);
        if (nx == 2) return reinterpret_cast<const void*>(gram_kernel<1, NB, 2>);
        return nullptr;
    }
    if constexpr (NB < 8) return gram_x_fn<NB + 1>(nb, nx);
    return nullptr;
}

// ---------------------------------------------------------------------------
// K5: fused update  out = (V − P·R_col)·R_jj⁻¹, row-local (R rows per thread), in place
// over the store (out may alias V; P never aliases out).  Coalesced 512-byte
// warp loads/stores straight from HBM at high occupancy; the coefficients are
// broadcast from shared memory.  Both loops are right-looking so every row
// keeps w independent FMA chains, while each element still receives its
// terms in the reference's order (l ascending, then ×1/R(j,j)).
// coef layout (doubles): nrc[cp][WMAX] = −R_col, nrjj[WMAX][WMAX] = −R_jj(l,j)
// for l < j, inv[WMAX] = 1/R_jj(j,j).
// ---------------------------------------------------------------------------
// R = 2 requires even ld's and 16-byte aligned P/V/out (the store's layout);
// an odd last row is finished by the scalar path.
template <int WMAX, int R>
__global__ void __launch_bounds__(256)
    update_kernel(i64 n, const double* __restrict__ P, i64 ldp, int cp, const double* V, i64 ldv, int w,
                  const double* __restrict__ coef, int triangular, double* out, i64 ldo, const int* skip) {
    KB_PDL_WAIT();
    if (skip && *skip) return;  // speculative block whose factorisation failed (k_pip.cu)
    // Columns w ≤ j < WMAX are identity padding (zero coefficients, inv = 1):
    // the arithmetic below is branch-free and leaves them at zero.
    extern __shared__ __align__(16) double c_sm[];
    // nrc rows zero-padded from cp to cpp = round_up(cp, 12) (the prefix loop
    // runs in whole 12-column groups); then nrjj and inv.
    const int cpp = (cp + 11) / 12 * 12;
    for (int i = threadIdx.x; i < cpp * WMAX; i += blockDim.x) c_sm[i] = i < cp * WMAX ? coef[i] : 0.0;
    for (int i = threadIdx.x; i < (WMAX + 1) * WMAX; i += blockDim.x)
        c_sm[cpp * WMAX + i] = coef[cp * WMAX + i];
    __syncthreads();
    const double* nrc = c_sm;
    const double* nrjj = c_sm + static_cast<size_t>(cpp) * WMAX;
    const double* inv = nrjj + WMAX * WMAX;
    const i64 groups = n / R;
    const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    for (i64 g = tid; g < groups; g += static_cast<i64>(gridDim.x) * blockDim.x)
        update_rows<WMAX, R>(g * R, P, ldp, cp, cpp, V, ldv, w, nrc, nrjj, inv, triangular, out, ldo);
    if (R > 1 && tid < n - groups * R)
        update_rows<WMAX, 1>(groups * R + tid, P, ldp, cp, cpp, V, ldv, w, nrc, nrjj, inv, triangular, out, ldo);
}

// Wide blocks (33 ≤ w ≤ 64, the ŝ+1 finalize panel): two threads per row.
// Thread parity p owns columns j ≡ p (mod 2); each finalized x_k is passed
// to the partner with one shuffle.  Half the accumulators per thread → twice
// the resident warps, which the 64-step substitution chain needs.
// coef layout: nrc[cp][2][32] and nrjj[64][2][32] (column j = 2·jj + parity),
// inv[2][32].
__global__ void __launch_bounds__(256)
    update_pair_kernel(i64 n, const double* __restrict__ P, i64 ldp, int cp, const double* V, i64 ldv, int w,
                       const double* __restrict__ coef, int triangular, double* out, i64 ldo, const int* skip) {
    KB_PDL_WAIT();
    if (skip && *skip) return;
    constexpr int H = 32;
    extern __shared__ __align__(16) double c_sm[];
    const int ncoef = (cp + 64 + 1) * 64;
    for (int i = threadIdx.x; i < ncoef; i += blockDim.x) c_sm[i] = coef[i];
    __syncthreads();
    const int par = threadIdx.x & 1;
    const double* nrc = c_sm + par * H;
    const double* nrjj = c_sm + static_cast<size_t>(cp) * 64 + par * H;
    const double* inv = c_sm + static_cast<size_t>(cp + 64) * 64 + par * H;
    const unsigned lane = threadIdx.x & 31;
    const i64 pairs = static_cast<i64>(gridDim.x) * (blockDim.x / 2);
    // Every thread runs the same trip count (shuffles stay convergent).
    for (i64 base = blockIdx.x * static_cast<i64>(blockDim.x / 2); base < n; base += pairs) {
        const i64 row = base + (threadIdx.x >> 1);
        const bool live = row < n;
        double acc[H];
#pragma unroll
        for (int jj = 0; jj < H; ++jj) {
            const int j = 2 * jj + par;
            acc[jj] = (live && j < w) ? V[row + j * ldv] : 0.0;
        }
        const double* prow = P + (live ? row : 0);
        for (int l = 0; l < cp; ++l) {
            const double pv = __ldg(prow + l * ldp);
            const double2* cr = reinterpret_cast<const double2*>(nrc + l * 64);
#pragma unroll
            for (int jj = 0; jj < H; jj += 2) {
                const double2 c = cr[jj / 2];
                acc[jj] = fma(c.x, pv, acc[jj]);
                acc[jj + 1] = fma(c.y, pv, acc[jj + 1]);
            }
        }
        if (triangular) {
#pragma unroll
            for (int k = 0; k < 64; ++k) {
                const int kk = k >> 1;
                double xk = 0.0;
                if ((k & 1) == par) {
                    acc[kk] *= inv[kk];
                    xk = acc[kk];
                }
                xk = __shfl_sync(0xffffffffu, xk, (lane & ~1u) | static_cast<unsigned>(k & 1));
                // columns j > k owned by this thread: jj from first(j > k, j ≡ par)
                const int first = (k + 1 + ((k + 1 + par) & 1)) >> 1;  // smallest jj with 2jj+par > k
                const double* rk = nrjj + k * 64;
#pragma unroll
                for (int jj = 0; jj < H; ++jj)
                    if (jj >= first) acc[jj] = fma(rk[jj], xk, acc[jj]);
            }
        }
        if (live) {
#pragma unroll
            for (int jj = 0; jj < H; ++jj) {
                const int j = 2 * jj + par;
                if (j < w) out[row + j * ldo] = acc[jj];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K5b: update as a tall-skinny DMMA GEMM,  out = [V | P] · M  with
//   M = [[R_jj⁻¹]; [−R_col·R_jj⁻¹]]  (slots × wslots, R_jj⁻¹ upper triangular).
// Used only when R_jj is well conditioned (κ_F ≤ 4w) — the second-stage
// finalize and second passes, where the panel is already nearly orthonormal
// and R_jj ≈ I — so the explicit inverse loses nothing against substitution
// while the 1830-FMA/row substitution moves onto the DMMA pipe.  [V | P] is
// staged through the same TMA ring as the Gram (rows ≡ 4 mod 16: the A
// fragment loads X[r0 + lane/4][4kc + lane%4] are conflict-free); M lives in
// shared memory in fragment order, mfrag[(kc·NBW + jb)·32 + lane] =
// M[4kc + lane%4][8jb + lane/4].  Chunks are 8 rows (the MMA m dimension);
// the last chunk of a tile overhangs it and its extra rows are discarded.
// ---------------------------------------------------------------------------
template <int NBW, int NB, int CW = 8>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    update_mma_kernel(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_p,
                      const TsParams p, const double* __restrict__ mfrag, double* out, i64 ldo) {
    KB_PDL_WAIT();
    constexpr int KC = 2 * NB;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full, *empty;
    double* ring = ring_setup(smem, p, full, empty);
    const size_t stage_doubles = static_cast<size_t>(p.wslots + p.cpslots) * p.tr;
    double* msm = reinterpret_cast<double*>(smem + stage_doubles * 8 * p.stages + 16 * p.stages + 1024);
    msm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(msm) + 127) & ~uintptr_t(127));
    for (int i = threadIdx.x; i < KC * NBW * 32; i += blockDim.x) msm[i] = mfrag[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == CW) {
        if (lane == 0) ring_produce(&map_v, &map_p, p, ring, full, empty);
        return;
    }
    const int m = lane >> 2, kq = lane & 3;
    const int nchunks = (p.tr + 7) / 8;
    int s = 0, use = 0, rot = warp;
    for (i64 tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        mbar_wait(&full[s], use & 1);
        const double* st = ring + s * stage_doubles;
        for (int c = rot; c < nchunks; c += CW) {
            const int r = 8 * c + m;
            double a[KC];
#pragma unroll
            for (int kc = 0; kc < KC; ++kc) a[kc] = st[static_cast<size_t>(4 * kc + kq) * p.tr + r];
            const i64 row = tile * p.tr + r;
            const bool ok = r < p.tr && row < p.n;
#pragma unroll
            for (int jb = 0; jb < NBW; ++jb) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int kc = 0; kc < KC; ++kc)
                    if (kc < 2 * (jb + 1) || kc >= 2 * NBW) dmma(d0, d1, a[kc], msm[(kc * NBW + jb) * 32 + lane]);
                const int col = 8 * jb + 2 * kq;
                if (ok) {
                    if (col < p.w) out[row + col * ldo] = d0;
                    if (col + 1 < p.w) out[row + (col + 1) * ldo] = d1;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        rot = (rot + 1) & (CW - 1);
        if (++s == p.stages) {
            s = 0;
            ++use;
        }
    }
}

// ---------------------------------------------------------------------------
// K5t: the K5 update (w ≤ 8) with the prefix streamed through a TMA ring in
// 16-column chunks: each 256-row tile arrives as one V box then ⌈cp/16⌉
// prefix boxes (4 KB contiguous per column, like the Gram's loads), one
// producer warp, 8 consumer warps with one row per thread.  The arithmetic
// is K5's, term for term (acc = V; acc += −R_col(l,·)·p_l, l ascending;
// right-looking substitution), so the results are bit-identical to K5.
// ---------------------------------------------------------------------------
constexpr int kTmaRows = 256;

// R = 2: each consumer thread owns two adjacent rows (16-byte shared-memory
// loads, and every coefficient broadcast serves both rows); a tile is R
// 256-row boxes, stored per box as [CC][256].
template <int WMAX, int CC, int ST, int R>
__global__ void __launch_bounds__(9 * 32, 1)
    update_tma_kernel(const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_p,
                      i64 n, int cp, int w, const double* __restrict__ coef, double* out, i64 ldo,
                      const int* skip) {
    KB_PDL_WAIT();
    if (skip && *skip) return;  // speculative block whose factorisation failed (k_pip.cu)
    constexpr int CW = 8, BOX = kTmaRows, TR = BOX * R;
    extern __shared__ __align__(1024) unsigned char smem[];
    double* ring = reinterpret_cast<double*>(smem);                      // [ST][R][CC][BOX]
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + ST * CC * TR);
    uint64_t* empty = full + ST;
    double* c_sm = reinterpret_cast<double*>(empty + ST);                 // coefficients
    const int cpp = (cp + CC - 1) / CC * CC;
    const int nchunk = 1 + cpp / CC;  // V, then the prefix
    for (int i = threadIdx.x; i < cpp * WMAX; i += blockDim.x) c_sm[i] = i < cp * WMAX ? coef[i] : 0.0;
    for (int i = threadIdx.x; i < (WMAX + 1) * WMAX; i += blockDim.x) c_sm[cpp * WMAX + i] = coef[cp * WMAX + i];
    if (threadIdx.x == 0) {
        for (int q = 0; q < ST; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const double* nrc = c_sm;
    const double* nrjj = c_sm + static_cast<size_t>(cpp) * WMAX;
    const double* inv = nrjj + WMAX * WMAX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 ntiles = (n + TR - 1) / TR;
    if (warp == CW) {  // producer
        if (lane != 0) return;
        int q = 0, use = 0;
        for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int row0 = static_cast<int>(tile * TR);
            for (int c = 0; c < nchunk; ++c) {
                if (use > 0) mbar_wait(&empty[q], (use - 1) & 1);
                double* st = ring + static_cast<size_t>(q) * CC * TR;
                const unsigned cols = c == 0 ? static_cast<unsigned>(w) : static_cast<unsigned>(CC);
                mbar_expect_tx(&full[q], cols * TR * 8);
#pragma unroll
                for (int bx = 0; bx < R; ++bx) {
                    if (c == 0)
                        tma_load_2d(st + bx * CC * BOX, &map_v, row0 + bx * BOX, 0, &full[q]);
                    else
                        tma_load_2d(st + bx * CC * BOX, &map_p, row0 + bx * BOX, (c - 1) * CC, &full[q]);
                }
                if (++q == ST) {
                    q = 0;
                    ++use;
                }
            }
        }
        return;
    }
    // this thread's rows R·t … R·t + R − 1 of the tile: box R·t / BOX, row R·t % BOX
    const int t = threadIdx.x;
    const int off = (R * t / BOX) * CC * BOX + (R * t) % BOX;
    int q = 0, use = 0;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        double acc[WMAX][R];
        for (int c = 0; c < nchunk; ++c) {
            mbar_wait(&full[q], use & 1);
            const double* st = ring + static_cast<size_t>(q) * CC * TR + off;
            auto ldr = [&](int col, double (&d)[R]) {
                if constexpr (R == 1) {
                    d[0] = st[col * BOX];
                } else {
#pragma unroll
                    for (int h = 0; h < R; h += 2) {
                        const double2 v2 = *reinterpret_cast<const double2*>(st + col * BOX + h);
                        d[h] = v2.x;
                        d[h + 1] = v2.y;
                    }
                }
            };
            if (c == 0) {
#pragma unroll
                for (int j = 0; j < WMAX; ++j) {
                    double d[R];
                    ldr(j, d);
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[j][r] = j < w ? d[r] : 0.0;
                }
            } else {
                const int l0 = (c - 1) * CC;
#pragma unroll
                for (int u = 0; u < CC; ++u) {
                    double pv[R];
                    ldr(u, pv);
                    const double2* cr = reinterpret_cast<const double2*>(nrc + (l0 + u) * WMAX);
#pragma unroll
                    for (int j = 0; j < WMAX; j += 2) {
                        const double2 cf = cr[j / 2];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            acc[j][r] = fma(cf.x, pv[r], acc[j][r]);
                            acc[j + 1][r] = fma(cf.y, pv[r], acc[j + 1][r]);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q]);
            if (++q == ST) {
                q = 0;
                ++use;
            }
        }
        // right-looking substitution, tri_solve_right's order (as K5)
#pragma unroll
        for (int k = 0; k < WMAX; ++k) {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[k][r] *= inv[k];
            const double* rk = nrjj + k * WMAX;
#pragma unroll
            for (int j = k + 1; j < WMAX; ++j)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[j][r] = fma(rk[j], acc[k][r], acc[j][r]);
        }
        const i64 row = tile * TR + R * t;
        if (R > 1 && row + R - 1 < n) {
#pragma unroll
            for (int j = 0; j < WMAX; ++j)
                if (j < w)
#pragma unroll
                    for (int h = 0; h < R; h += 2)
                        *reinterpret_cast<double2*>(out + row + h + j * ldo) = make_double2(acc[j][h], acc[j][h + 1]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (row + r < n)
#pragma unroll
                    for (int j = 0; j < WMAX; ++j)
                        if (j < w) out[row + r + j * ldo] = acc[j][r];
        }
    }
}

template <int NBW, int NB>
const void* update_mma_fn(int nbw, int nb) {
    if (nbw == NBW && nb == NB) return reinterpret_cast<const void*>(update_mma_kernel<NBW, NB>);
    if constexpr (NB < 8) {
        return update_mma_fn<NBW, NB + 1>(nbw, nb);
    } else if constexpr (NBW < 8) {
        return update_mma_fn<NBW + 1, NBW + 1>(nbw, nb);
    } else {
        return nullptr;
    }
}

// ---------------------------------------------------------------------------
// Host side: tensor maps, geometry, launches.
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) fail(KRY_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap encode_map(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols,
                       bool promote = true);

// Tensor maps are cached by their parameters: the solver re-launches the same
// (store column, shape) combinations every cycle, and an encode costs more
// host time than the launch itself.
CUtensorMap make_map_box(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols,
                         bool promote = true);
CUtensorMap make_map(const double* base, i64 ld, i64 rows, i64 cols, int box_rows) {
    return make_map_box(base, ld, rows, cols, box_rows, 0);
}
CUtensorMap make_map_box(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols, bool promote) {
    struct Key {
        const double* base;
        i64 ld, rows, cols;
        int box;
        bool operator==(const Key& o) const {
            return base == o.base && ld == o.ld && rows == o.rows && cols == o.cols && box == o.box;
        }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            size_t h = std::hash<const void*>()(k.base);
            for (i64 v : {k.ld, k.rows, k.cols, static_cast<i64>(k.box)}) h = h * 1000003u ^ std::hash<i64>()(v);
            return h;
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{base, ld, rows, cols, (box_rows * 1024 + box_cols) * 2 + (promote ? 1 : 0)};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (cache.size() > 4096) cache.clear();
    CUtensorMap m = encode_map(base, ld, rows, cols, box_rows, box_cols, promote);
    cache.emplace(key, m);
    return m;
}

CUtensorMap encode_map(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols, bool promote) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    if (cols <= 0 || base == nullptr) return m;  // unused operand
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld & 1) != 0)
        fail(KRY_INTERNAL, "TMA operand must be 16-byte aligned with an even leading dimension");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_cols > 0 ? box_cols : cols)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE,
                             promote ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(KRY_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

int sm_count() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    });
    return n;
}

// cudaFuncSetAttribute once per kernel and size (it is a host-side call per launch otherwise).
void set_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = done[kernel];
    if (bytes <= have) return;
    KB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    have = bytes;
}

// Largest Gram ring stage.  Taller tiles give longer contiguous runs per
// column (132 rows × 8 B ≈ 1 KB at 64 slots) at the price of fewer stages;
// measured at 4000² (Gram ms per cycle): 36 KB 9.16, 50 KB 8.94, 62 KB
// 8.82, 70 KB 8.77, 80 KB 8.83–9.03, 101 KB 8.82.  KRY_GRAM_STAGE_KB overrides.
size_t gram_stage_bytes() {
    static const size_t b = [] {
        const char* e = std::getenv("KRY_GRAM_STAGE_KB");
        return static_cast<size_t>(e ? std::atoi(e) : 70) * 1024;
    }();
    return b;
}

TsParams geometry(i64 n, int w, int cp, bool gram) {
    // TMA tile coordinates are signed 32-bit (cp.async.bulk.tensor): the row
    // of every tile must be < 2^31.  (2^31 rows × 61 columns would be a 1 TB
    // store, far beyond one GPU, but the limit is checked, not assumed.)
    if (n >= (i64(1) << 31)) fail(KRY_UNSUPPORTED, "more than 2^31 - 1 rows per GPU on the TMA Gram/update path");
    TsParams p{};
    p.n = n;
    p.w = w;
    p.wslots = static_cast<int>(round_up(w, 8));
    p.cp = cp;
    p.cpslots = static_cast<int>(round_up(cp, 8));
    const int slots = p.wslots + p.cpslots;
    if (gram) {
        // rows ≡ 4 (mod 16): the DMMA fragment loads are bank-conflict free.
        static const int cand[] = {244, 196, 132, 68};
        p.tr = 68;
        for (int c : cand)
            if (static_cast<size_t>(c) * slots * 8 <= gram_stage_bytes()) {
                p.tr = c;
                break;
            }
    } else {
        p.tr = 128;  // one row per consumer thread
    }
    const size_t stage_bytes = static_cast<size_t>(slots) * p.tr * 8;
    const int wm = w <= 8 ? 8 : w <= 16 ? 16 : w <= 32 ? 32 : 64;
    const size_t coef_bytes = gram ? 0 : static_cast<size_t>(cp + wm + 1) * wm * 8 + 1024;
    int st = static_cast<int>((kSmemBudget - coef_bytes) / stage_bytes);
    p.stages = std::max(2, std::min(8, st));
    p.ntiles = ceil_div(n, p.tr);
    p.tx_bytes = static_cast<unsigned>(static_cast<size_t>(w + cp) * p.tr * 8);
    return p;
}

size_t ring_bytes(const TsParams& p) {
    return static_cast<size_t>(p.wslots + p.cpslots) * p.tr * 8 * p.stages + 16 * p.stages + 64;
}

}  // namespace

void launch_gram_reduce(cudaStream_t stream, const double* partials, int grid, int per_cta, double* packed) {
    launch_pdl(gram_reduce_kernel, static_cast<unsigned>(ceil_div(static_cast<i64>(per_cta) * 32, 256)), 256, 0, stream,
               partials, grid, per_cta, packed);
    KB_LAUNCHED();
}
void set_kernel_smem(const void* kernel, size_t bytes) { set_smem(kernel, bytes); }
CUtensorMap dev::tensor_map_2d(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols,
                               bool l2_promote) {
    return make_map_box(base, ld, rows, cols, box_rows, box_cols, l2_promote);
}
int device_sms() { return sm_count(); }

// Column groups of the prefix so that round_up(w,8) + round_up(group,8) ≤ 64.
std::vector<std::pair<i64, i64>> prefix_groups(i64 c0, i64 w) {
    std::vector<std::pair<i64, i64>> g;
    const i64 wslots = round_up(w, 8);
    if (wslots > 64) fail(KRY_UNSUPPORTED, "block width above 64 columns is not supported on the device path");
    const i64 room = 64 - wslots;
    if (c0 > 0 && room == 0) fail(KRY_UNSUPPORTED, "block width 57..64 with a non-empty prefix is not supported");
    for (i64 b = 0; b < c0; b += room) g.emplace_back(b, std::min(room, c0 - b));
    return g;
}

i64 gram_scratch_doubles(i64 w) {
    (void)w;
    return static_cast<i64>(sm_count()) * 36 * 64;
}

void launch_gram_pass(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V,
                      i64 ldv, i64 w, bool vv, double* d_partials, double* d_packed,
                      std::vector<int>& tile_ids, int64_t& launches, i64 x_first, i64 x_count) {
    TsParams p = geometry(n, static_cast<int>(w), static_cast<int>(cp), true);
    p.vv = vv ? 1 : 0;
    const int nbw = p.wslots / 8, nb = nbw + p.cpslots / 8;
    tile_ids.clear();
    for (int jb = 0; jb < nbw; ++jb)
        for (int ib = 0; ib < nb; ++ib)
            if (tile_valid(nbw, jb, ib)) tile_ids.push_back(jb * 8 + ib);
    // Extra P-column blocks (prefix columns [x_first, x_first + x_count)):
    // tile id 64 + xb*8 + ib ↦ rows = slot block ib, cols = slot block xb.
    int nx = 0;
    p.xb0 = 0;
    if (x_count > 0) {
        const int s0 = p.wslots + static_cast<int>(x_first), s1 = s0 + static_cast<int>(x_count) - 1;
        p.xb0 = s0 / 8;
        nx = s1 / 8 - p.xb0 + 1;
        if (nbw != 1 || nx > 2 || s1 / 8 >= nb) fail(KRY_INTERNAL, "gram extra-column shape");
        for (int k = 0; k < nx; ++k)
            for (int ib = nbw; ib < nb; ++ib) tile_ids.push_back(64 + (p.xb0 + k) * 8 + ib);
    }
    const int T = static_cast<int>(tile_ids.size());
    CUtensorMap mv = make_map(V, ldv, n, w, p.tr);
    CUtensorMap mp = make_map(P, ldp, n, cp, p.tr);
    const int grid = static_cast<int>(std::min<i64>(sm_count(), std::max<i64>(1, p.ntiles)));
    const int cw = consumer_warps(nbw);
    p.consumers = cw;
    const size_t red_bytes = static_cast<size_t>(cw) * T * 64 * 8;
    const size_t smem = std::max(ring_bytes(p), red_bytes) + 1024;
    const void* fn = nx == 0 ? gram_fn<1, 1>(nbw, nb) : gram_x_fn<1>(nb, nx);
    if (!fn) fail(KRY_UNSUPPORTED, "gram shape");
    set_smem(fn, smem);
    void* args[] = {&mv, &mp, &p, &d_partials};
    launch_pdl_c(fn, dim3(grid), dim3((cw + 1) * 32), smem, stream, args);
    KB_LAUNCHED();
    const int per_cta = T * 64;
    launch_pdl(gram_reduce_kernel, static_cast<unsigned>(ceil_div(per_cta * 32, 256)), 256, 0, stream, d_partials, grid,
               per_cta, d_packed);
    KB_LAUNCHED();
    launches += 2;
}

void launch_update_mma(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V, i64 ldv,
                       i64 w, const double* d_mfrag, double* out, i64 ldo, int64_t& launches) {
    TsParams p = geometry(n, static_cast<int>(w), static_cast<int>(cp), true);
    const int nbw = p.wslots / 8, nb = nbw + p.cpslots / 8;
    if (nb > 8) fail(KRY_INTERNAL, "update_mma shape");
    p.consumers = 8;
    const size_t mbytes = static_cast<size_t>(2 * nb) * nbw * 32 * 8;
    const size_t stage_bytes = static_cast<size_t>(p.wslots + p.cpslots) * p.tr * 8;
    p.stages = std::max(2, std::min(p.stages, static_cast<int>((200 * 1024 - mbytes) / stage_bytes)));
    const size_t smem = ring_bytes(p) + 1024 + 128 + mbytes + 256;
    CUtensorMap mv = make_map(V, ldv, n, w, p.tr);
    CUtensorMap mp = make_map(P, ldp, n, cp, p.tr);
    const int grid = static_cast<int>(std::min<i64>(sm_count(), std::max<i64>(1, p.ntiles)));
    const void* fn = update_mma_fn<1, 1>(nbw, nb);
    if (!fn) fail(KRY_UNSUPPORTED, "update_mma shape");
    set_smem(fn, smem);
    void* args[] = {&mv, &mp, &p, &d_mfrag, &out, &ldo};
    launch_pdl_c(fn, dim3(grid), dim3(9 * 32), smem, stream, args);
    KB_LAUNCHED();
    launches += 1;
}

// K5t for w ≤ 8 when the layout allows TMA (KRY_UPDATE_TMA=0 keeps K5).
static bool launch_update_tma(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V,
                              i64 ldv, i64 w, const double* d_coef, bool triangular, double* out, i64 ldo,
                              int64_t& launches, const int* skip) {
    static const bool on = [] {
        const char* e = std::getenv("KRY_UPDATE_TMA");
        return !(e && std::atoi(e) == 0);
    }();
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    if (!on || !triangular || w > 8 || cp < 1 || !a16(P) || !a16(V) || (ldp & 1) || (ldv & 1) ||
        n >= (i64(1) << 31))
        return false;
    const int wmax = update_wmax(w);
    // Two rows per consumer thread, 16-column chunks, 3 × 64 KB stages.
    // Measured at 4000² (update ms per cycle): one row per thread (6 × 32 KB
    // stages) 9.07, two rows 8.79, four rows with 8-column chunks 8.87;
    // KRY_UPDATE_TMA_ROWS=1 selects the one-row variant (A/B).
    static const int rows = [] {
        const char* e = std::getenv("KRY_UPDATE_TMA_ROWS");
        return e && std::atoi(e) == 1 ? 1 : 2;
    }();
    const int cc = 16;
    const int st = rows == 1 ? 6 : 3;
    const int cpp = static_cast<int>(round_up(cp, cc));
    const size_t smem = static_cast<size_t>(st) * cc * kTmaRows * rows * 8 + 2 * st * 8 +
                        static_cast<size_t>(cpp + wmax + 1) * wmax * 8 + 64;
    if (smem > 227 * 1024) return false;
    CUtensorMap mv = make_map(V, ldv, n, w, kTmaRows);
    CUtensorMap mp = make_map_box(P, ldp, n, cp, kTmaRows, cc);
    const i64 ntiles = ceil_div(n, kTmaRows * rows);
    const int grid = static_cast<int>(std::min<i64>(sm_count(), std::max<i64>(1, ntiles)));
    const void* fn = rows == 2 ? (wmax == 6 ? reinterpret_cast<const void*>(update_tma_kernel<6, 16, 3, 2>)
                                            : reinterpret_cast<const void*>(update_tma_kernel<8, 16, 3, 2>))
                               : (wmax == 6 ? reinterpret_cast<const void*>(update_tma_kernel<6, 16, 6, 1>)
                                            : reinterpret_cast<const void*>(update_tma_kernel<8, 16, 6, 1>));
    set_smem(fn, smem);
    int cpi = static_cast<int>(cp), wi = static_cast<int>(w);
    void* args[] = {&mv, &mp, &n, &cpi, &wi, const_cast<double**>(&d_coef), &out, &ldo, const_cast<int**>(&skip)};
    launch_pdl_c(fn, dim3(grid), dim3(9 * 32), smem, stream, args);
    KB_LAUNCHED();
    launches += 1;
    return true;
}

static int update_rows_setting() {  // KRY_UPDATE_ROWS=1 → one row per thread (A/B)
    static const int r = [] {
        const char* e = std::getenv("KRY_UPDATE_ROWS");
        const int v = e ? std::atoi(e) : 2;
        return v == 1 ? 1 : 2;
    }();
    return r;
}

int update_wmax(i64 w) { return w <= 6 ? 6 : w <= 8 ? 8 : w <= 16 ? 16 : w <= 32 ? 32 : 64; }

void launch_update(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V, i64 ldv,
                   i64 w, const double* d_coef, bool triangular, double* out, i64 ldo, int64_t& launches,
                   const int* skip) {
    if (launch_update_tma(stream, n, P, ldp, cp, V, ldv, w, d_coef, triangular, out, ldo, launches, skip)) return;
    const int wmax = update_wmax(w);
    const size_t smem = static_cast<size_t>(round_up(cp, 12) + wmax + 1) * wmax * 8;
    if (smem > 200 * 1024) fail(KRY_UNSUPPORTED, "update coefficients exceed shared memory");
    // Two rows per thread when the layout allows 16-byte accesses.
    const int rsel = update_rows_setting();
    const bool vec = wmax <= 16 && rsel > 1 && ((ldp | ldv | ldo) & 1) == 0 &&
                     ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(V) |
                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const i64 rows_per_thread = vec ? 2 : 1;
    auto go = [&](auto kernel) {
        set_smem(reinterpret_cast<const void*>(kernel), smem);
        const int per_sm = occupancy(reinterpret_cast<const void*>(kernel), 256, smem);
        const i64 want = ceil_div(n, (wmax == 64 ? 128 : 256) * rows_per_thread);
        const int grid = static_cast<int>(std::max<i64>(1, std::min<i64>(want, static_cast<i64>(sm_count()) * std::max(per_sm, 1))));
        launch_pdl(kernel, grid, 256, smem, stream, n, P, ldp, static_cast<int>(cp), V, ldv, static_cast<int>(w), d_coef,
                                            triangular ? 1 : 0, out, ldo, skip);
    };
    switch (wmax) {
        case 6: vec ? go(update_kernel<6, 2>) : go(update_kernel<6, 1>); break;
        case 8: vec ? go(update_kernel<8, 2>) : go(update_kernel<8, 1>); break;
        case 16: vec ? go(update_kernel<16, 2>) : go(update_kernel<16, 1>); break;
        case 32: go(update_kernel<32, 1>); break;
        default: go(update_pair_kernel); break;  // coefficients in the interleaved layout
    }
    KB_LAUNCHED();
    launches += 1;
}


}  // namespace kb
