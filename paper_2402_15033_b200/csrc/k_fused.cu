// K6: the fused first-stage pass of the speculative two-stage path, 2-D
// 5-point stencil, one rank.  OPT-IN (KRY_FUSED_PASS=1): correct (every
// two-stage 2-D golden passes through it) but slower than the separate
// kernels on B200 — DESIGN.md §5 has the measurements.
//
// Between two first-stage blocks the unfused path streams the basis prefix
// Q[:, 0:c0] twice: once in block j's update (K5t: Q_j = (V_j − P·R_col)·R_jj⁻¹)
// and again in block j+1's Gram (K3: [Q[:, 0:c0'] | V_{j+1}]ᵀ·V_{j+1}), with
// block j+1's MPK (K2f) in between, because V_{j+1} = A^k·q (q = Q_j's last
// column) needs the updated block.  For a stencil every row of V_{j+1} only
// depends on rows of q within s grid lines / columns, so the three steps can
// run in one pass over the rows: K6 updates a window line of block j, feeds
// the new q into the s-level stencil wavefront and, s lines later,
// accumulates the Gram of block j+1 over the same rows.  The prefix then
// crosses HBM once per block instead of twice.
//
// Work decomposition.  The grid is cut into 64-column windows (32 lanes ×
// double2) that output their middle 64 − 2H columns (H = S rounded up to
// even, as K2f); tasks are (window, band) pairs in window-major order, task
// i on CTA i mod grid, bands alternating direction (neighbouring windows
// and band seams are processed at the same time, so the recomputed rows hit
// L2).  A band [y0, y1) runs y1 − y0 + 2S line steps: the update computes
// lines y0 − S … y1 + S − 1 (the 2S lines outside the band and the H halo
// columns are recomputed for the wavefront, never stored), level k of the
// MPK trails the update by k lines, the Gram takes the band's line g at step
// g + 2S.  Roles, synchronised by mbarriers:
//   * one TMA producer warp: window line l of [prefix | raw block j] into a
//     ring slot (kBox rows per column);
//   * kFuU update warps, line tt on warp tt mod kFuU: K5's arithmetic term
//     for term (bit-identical to K5/K5t) from the slot; Q_j goes to the
//     store (core rows), over the raw block in the slot (for the Gram), and
//     q to the next raw block and to a shared ring for the MPK warp;
//   * one MPK warp: levels 1..S of the wavefront, K2f's element order
//     (bit-identical to S spmv calls), stored to the next raw block;
//   * kFuG Gram warps, line g on warp g mod kFuG: K3's DMMA tiles from the
//     slot (prefix and Q_j) and the stored levels, plus the panel-Gram pieces
//     (NX extra tiles); per-CTA partials in K3's packed tile layout.
//   A slot is freed after its line's Gram, S lines after its update, so the
//   ring needs ≥ S + 2 slots (7 × 30 KB at c0 = 50) — the constraint that
//   keeps the pass latency-bound.
//
// Races.  Windows overlap by 2H columns and bands recompute 2S lines, so a
// CTA reads rows another CTA owns.  Both raw blocks therefore live outside
// the store (Store::fraw_, double-buffered): the update reads raw block j
// there and writes the store; the MPK writes raw block j+1 to the other
// buffer.  The prefix Q[:, 0:c0] is read-only in the pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kb_common.hpp"
#include "kb_device.hpp"
#include "kb_kernels.hpp"

namespace kb {

namespace {

using namespace dev;

constexpr int kFuU = 2;   // update warps
constexpr int kFuG = 6;   // Gram warps
constexpr int kFuMpk = kFuU, kFuProd = kFuU + 1, kFuG0 = kFuU + 2;
constexpr int kFuWarps = kFuG0 + kFuG;
constexpr int kFuThreads = kFuWarps * 32;
constexpr int kQR = 2;    // q ring (update → MPK), lines; a multiple of kFuU
constexpr int kGR = 6;    // Gram ring (MPK → Gram), lines; a multiple of kFuG
constexpr int kBox = 68;  // rows per slot column: the 64-row window + 4 (≡ 4 mod 16: conflict-free DMMA fragments)
constexpr int kMaxSlots = 12;

struct FusedMaps {
    CUtensorMap p;  // store columns [0, c0): box kBox × c0
    CUtensorMap v;  // raw block j: box kBox × w
};

// One slot holds window line l: [prefix Q[:, 0:c0] | raw block j] (kBox rows
// each).  The update overwrites the raw block with Q_j in place, and the slot
// stays until the Gram of line l (S lines later) has read [prefix | Q_j] —
// so the prefix crosses HBM once and is never re-read.  Slots live for
// S + 2 lines; a line's full/empty barriers are indexed by line mod 2·nslots
// so every parity wait is at most one phase ahead.
//
// Tile order of gram_kernel<1, NB, NX>: (jb = 0, ib = 0..NB−1), then the
// extra tiles (k, ib = 1..NB−1).
template <int S, int WMAX, int NB, int NX, int CL>
__global__ void __launch_bounds__(kFuThreads, 1)
    fused_pass_kernel(const __grid_constant__ FusedMaps maps, const FusedPassArgs a, int nslots) {
    KB_PDL_WAIT();
    if (a.skip && *a.skip) return;  // block j's factorisation failed: nothing may change (k_pip.cu); grid-uniform
    constexpr int H = (S + 1) & ~1, STEP = 64 - 2 * H;
    static_assert(STEP % 4 == 0, "core columns must split into 4-row DMMA chunks");
    static_assert(WMAX == S + 1, "the raw block is the MPK block");
    static_assert(kQR % kFuU == 0 && kGR % kFuG == 0, "rings must be multiples of the role warps");
    constexpr int T = NB + NX * (NB - 1);
    extern __shared__ __align__(1024) unsigned char smem[];
    const int cp = a.c0;
    // TMA destinations must be 128-byte aligned: the raw block starts at voff
    const int voff = (cp * kBox + 15) / 16 * 16;
    const int slot_doubles = voff + (WMAX * kBox + 15) / 16 * 16;
    double* ring = reinterpret_cast<double*>(smem);  // [nslots][cp + w][kBox]; Gram scratch at the end
    const size_t ring_doubles = max(static_cast<size_t>(nslots) * slot_doubles, static_cast<size_t>(kFuG) * T * 64);
    const int nbar = 2 * nslots;
    uint64_t* lfull = reinterpret_cast<uint64_t*>(ring + ring_doubles);  // [2·kMaxSlots]
    uint64_t* lfree = lfull + 2 * kMaxSlots;                             // [2·kMaxSlots]
    uint64_t* qfull = lfree + 2 * kMaxSlots;  // [CL][kQR]  (CTA 0: one ring per writing CTA)
    uint64_t* qempty = qfull + CL * kQR;      // [kQR]      (this CTA's q slots in CTA 0's ring)
    uint64_t* gready = qempty + kQR;          // [kGR]      (this CTA's Gram lines)
    uint64_t* gempty = gready + kGR;          // [CL][kGR]  (CTA 0: per Gram-owning CTA)
    double2* qring = reinterpret_cast<double2*>(gempty + CL * kGR);  // [CL][kQR][32] (CTA 0)
    double* c_sm = reinterpret_cast<double*>(qring + CL * kQR * 32);  // −R_col [cp][WMAX], −R_jj, 1/r_jj
    for (int i = threadIdx.x; i < (cp + WMAX + 1) * WMAX; i += blockDim.x) c_sm[i] = a.coef[i];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * kMaxSlots; ++i) {
            mbar_init(&lfull[i], 1);
            mbar_init(&lfree[i], 1);
        }
        for (int i = 0; i < CL * kQR; ++i) mbar_init(&qfull[i], 1);
        for (int i = 0; i < kQR; ++i) mbar_init(&qempty[i], 1);
        for (int i = 0; i < kGR; ++i) mbar_init(&gready[i], 1);
        for (int i = 0; i < CL * kGR; ++i) mbar_init(&gempty[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if constexpr (CL > 1) cluster_sync_all();  // peers' barriers initialised before any remote arrive

    // Cross-CTA signalling (CL > 1: the pair shares one window column; CTA 0
    // runs the MPK wavefront over all lines, CTA r the TMA/update/Gram of the
    // line steps t ≡ r (mod CL), each line's slot in its owner's shared memory).
    auto arrive_on = [&](uint64_t* bar, unsigned cta) {
        if constexpr (CL > 1)
            mbar_arrive_cluster(bar, cta);
        else
            mbar_arrive(bar);
    };
    auto wait_on = [&](uint64_t* bar, unsigned parity) {
        if constexpr (CL > 1)
            mbar_wait_cluster(bar, parity);
        else
            mbar_wait(bar, parity);
    };
    const int crank = CL > 1 ? static_cast<int>(cluster_rank()) : 0;
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nx = a.nx, ny = a.ny;
    const i64 ld = a.ld, nx64 = nx;
    // Tasks (window wx, band b) in window-major order, task i on cluster i mod
    // clusters: the clusters of one round cover whole runs of windows at the
    // same band, so neighbouring windows pass the same lines at the same time
    // (the overlapping halo columns hit L2), and bands alternate direction so
    // the 2S lines recomputed at a band seam are the ones the neighbouring band
    // processes at the same moment (both reach the seam at the end).
    auto for_tasks = [&](auto&& body) {
        for (int task = cid; task < a.ntasks; task += ncl) {
            const int wx = task / a.nbands, b = task % a.nbands;
            const int y0 = static_cast<int>(static_cast<i64>(b) * ny / a.nbands);
            const int y1 = static_cast<int>(static_cast<i64>(b + 1) * ny / a.nbands);
            body(wx, y0, y1, (b & 1) != 0);
        }
    };
    // this CTA's line steps of a task: t = crank, crank + CL, …
    auto own_count = [&](int steps) { return steps > crank ? (steps - crank + CL - 1) / CL : 0; };
    // line of update step t; levels trail the update by k lines, the Gram by S
    auto step_line = [&](int y0, int y1, bool down, int t) { return down ? y1 - 1 + S - t : y0 - S + t; };
    // Steps t < S and t ≥ len + S are recomputed lines outside the band: no
    // Gram, the update frees their slot.  In-band line of step t: Gram g = t − S.
    auto slot_of = [&](int tt) { return ring + static_cast<size_t>(tt % nslots) * slot_doubles; };

    if (warp == kFuProd) {
        // ---- TMA producer: window line of [prefix | raw block j] per slot ---
        if (lane == 0) {
            const unsigned tx = static_cast<unsigned>(cp + WMAX) * kBox * 8;
            int ub = 0;
            for_tasks([&](int wx, int y0, int y1, bool down) {
                const int steps = y1 - y0 + 2 * S;
                const int ix0 = wx * STEP - H;
                for (int o = 0, n = own_count(steps); o < n; ++o) {
                    const int t = crank + o * CL, ut = ub + o;
                    if (ut >= nslots) {
                        const int pt = ut - nslots;  // the line this slot held
                        mbar_wait(&lfree[pt % nbar], (pt / nbar) & 1);
                    }
                    // rows outside [0, n) (lines off the grid) are zero-filled by TMA
                    const int row0 = step_line(y0, y1, down, t) * nx + ix0;
                    double* st = slot_of(ut);
                    uint64_t* bar = &lfull[ut % nbar];
                    mbar_expect_tx(bar, tx);
                    if (cp > 0) tma_load_2d(st, &maps.p, row0, 0, bar);
                    tma_load_2d(st + voff, &maps.v, row0, 0, bar);
                }
                ub += own_count(steps);
            });
        }
    } else if (warp < kFuU) {
        // ---- update of block j from the slot (K5's arithmetic, term for term)
        const double* nrc = c_sm;
        const double* nrjj = c_sm + cp * WMAX;
        const double* inv = nrjj + WMAX * WMAX;
        double* outj = a.Q + cp * ld;  // store columns [cp, cp + w)
        int tb = 0;
        for_tasks([&](int wx, int y0, int y1, bool down) {
            const int ix = wx * STEP - H + 2 * lane;
            const bool in_grid = ix >= 0 && ix < nx;
            const bool store_lane = in_grid && lane >= H / 2 && lane < 32 - H / 2;
            const int steps = y1 - y0 + 2 * S, nown = own_count(steps);
            for (int o = ((warp - tb) % kFuU + kFuU) % kFuU; o < nown; o += kFuU) {  // tt ≡ warp (mod kFuU)
                const int t = crank + o * CL, tt = tb + o;
                mbar_wait(&lfull[tt % nbar], (tt / nbar) & 1);
                double* st = slot_of(tt) + 2 * lane;
                double acc[WMAX][2];
#pragma unroll
                for (int j = 0; j < WMAX; ++j) {
                    const double2 v = *reinterpret_cast<const double2*>(st + voff + j * kBox);
                    acc[j][0] = v.x;
                    acc[j][1] = v.y;
                }
#pragma unroll 4
                for (int l = 0; l < cp; ++l) {
                    const double2 pv = *reinterpret_cast<const double2*>(st + l * kBox);
                    const double2* cr = reinterpret_cast<const double2*>(nrc + l * WMAX);
#pragma unroll
                    for (int j = 0; j < WMAX; j += 2) {
                        const double2 c = cr[j / 2];
                        acc[j][0] = fma(c.x, pv.x, acc[j][0]);
                        acc[j][1] = fma(c.x, pv.y, acc[j][1]);
                        acc[j + 1][0] = fma(c.y, pv.x, acc[j + 1][0]);
                        acc[j + 1][1] = fma(c.y, pv.y, acc[j + 1][1]);
                    }
                }
                update_tri<WMAX, 2>(acc, nrjj, inv);
                const int l = step_line(y0, y1, down, t);
                const bool live = in_grid && l >= 0 && l < ny;
                const bool in_band = t >= S && t < steps - S;
                const double2 q = live ? make_double2(acc[WMAX - 1][0], acc[WMAX - 1][1]) : make_double2(0.0, 0.0);
                if (in_band) {
                    // Q_j over the raw block in the slot, for this line's Gram
#pragma unroll
                    for (int j = 0; j < WMAX; ++j)
                        *reinterpret_cast<double2*>(st + voff + j * kBox) = make_double2(acc[j][0], acc[j][1]);
                    if (live && store_lane) {
                        const i64 row = static_cast<i64>(l) * nx64 + ix;
#pragma unroll
                        for (int j = 0; j < WMAX; ++j) RowVec<2>::st(outj + row + j * ld, acc[j]);  // w == WMAX
                        *reinterpret_cast<double2*>(a.Vn + row) = q;  // seam: column 0 of raw block j+1
                    }
                    // the slot is refilled by TMA (async proxy) once the Gram frees it
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                // q to the MPK warp (CTA 0's ring for this CTA's lines)
                const int qs = tt % kQR;
                if (tt >= kQR) mbar_wait(&qempty[qs], ((tt / kQR) - 1) & 1);
                double2* qdst = qring + (crank * kQR + qs) * 32 + lane;
                if constexpr (CL > 1)
                    st_cluster_f64x2(qdst, 0, q);
                else
                    *qdst = q;
                __syncwarp();
                if (lane == 0) {
                    arrive_on(&qfull[crank * kQR + qs], 0);
                    if (!in_band) mbar_arrive(&lfree[tt % nbar]);  // recomputed line: no Gram
                }
            }
            tb += nown;
        });
        asm volatile("bar.sync 2, %0;" ::"n"((kFuU + kFuG) * 32));  // the ring is free for the Gram scratch
    } else if (warp == kFuMpk) {
        // ---- MPK of block j+1 (CTA 0): levels 1..S of the q wavefront --------
        // A[k], B[k], C[k]: level k at lines l − k, l − k − 1, l − k − 2 after step l.
        if (crank == 0) {
            int cq[CL], cg[CL];  // per owning CTA: q lines received, Gram lines signalled
#pragma unroll
            for (int r = 0; r < CL; ++r) cq[r] = cg[r] = 0;
            for_tasks([&](int wx, int y0, int y1, bool down) {
                const int ix = wx * STEP - H + 2 * lane;
                const bool in_grid = ix >= 0 && ix < nx;
                const bool store_lane = in_grid && lane >= H / 2 && lane < 32 - H / 2;
                double2 A[S + 1], B[S + 1], C[S + 1];
#pragma unroll
                for (int k = 0; k <= S; ++k) A[k] = B[k] = C[k] = make_double2(0.0, 0.0);
                const int steps = y1 - y0 + 2 * S;
                for (int t = 0; t < steps; ++t) {
                    // q of step t from its owner's ring
                    const int r = t % CL;
                    int c = 0;
#pragma unroll
                    for (int rr = 0; rr < CL; ++rr)
                        if (rr == r) c = cq[rr]++;
                    const int qs = c % kQR;
                    wait_on(&qfull[r * kQR + qs], (c / kQR) & 1);
                    const double2 in = qring[(r * kQR + qs) * 32 + lane];
                    __syncwarp();
                    if (lane == 0) arrive_on(&qempty[qs], r);
                    const int l = step_line(y0, y1, down, t);
                    C[0] = B[0];
                    B[0] = A[0];
                    A[0] = in;
#pragma unroll
                    for (int k = 1; k <= S; ++k) {
                        // ascending: A = line lk + 1, C = lk − 1; descending: the reverse
                        const double2 dn = down ? A[k - 1] : C[k - 1], cu = B[k - 1], up = down ? C[k - 1] : A[k - 1];
                        const double left = __shfl_up_sync(0xffffffffu, cu.y, 1);
                        const double right = __shfl_down_sync(0xffffffffu, cu.x, 1);
                        // spmv's stored order: row−nx, row−1, row, row+1, row+nx (K2f)
                        double s0 = __dadd_rn(0.0, -dn.x);
                        s0 = __dadd_rn(s0, -left);
                        s0 = __dadd_rn(s0, __dmul_rn(4.0, cu.x));
                        s0 = __dadd_rn(s0, -cu.y);
                        s0 = __dadd_rn(s0, -up.x);
                        double s1 = __dadd_rn(0.0, -dn.y);
                        s1 = __dadd_rn(s1, -cu.x);
                        s1 = __dadd_rn(s1, __dmul_rn(4.0, cu.y));
                        s1 = __dadd_rn(s1, -right);
                        s1 = __dadd_rn(s1, -up.y);
                        const int lk = down ? l + k : l - k;
                        const bool live = in_grid && lk >= 0 && lk < ny;
                        const double2 v = live ? make_double2(s0, s1) : make_double2(0.0, 0.0);
                        C[k] = B[k];
                        B[k] = A[k];
                        A[k] = v;
                        if (store_lane && lk >= y0 && lk < y1)
                            *reinterpret_cast<double2*>(a.Vn + k * ld + static_cast<i64>(lk) * nx64 + ix) = v;
                    }
                    const int g = t - 2 * S;  // the segment's g-th line (l ∓ S) is complete
                    if (g >= 0 && g < y1 - y0) {
                        const int owner = (g + S) % CL;  // the CTA that updated line g holds its slot
                        int cgo = 0;
#pragma unroll
                        for (int rr = 0; rr < CL; ++rr)
                            if (rr == owner) cgo = cg[rr]++;
                        const int gs = cgo % kGR;
                        if (cgo >= kGR) mbar_wait(&gempty[owner * kGR + gs], ((cgo / kGR) - 1) & 1);
                        __syncwarp();
                        if (lane == 0) arrive_on(&gready[gs], owner);
                    }
                }
            });
        }
    } else {
        // ---- Gram of block j+1: [V_{j+1} | Q[:, 0:c0']]ᵀ·V_{j+1} --------------
        const int gw = warp - kFuG0;
        double acc[NB][2];
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) acc[ib][0] = acc[ib][1] = 0.0;
        double accx[NX > 0 ? NX : 1][NB][2];
#pragma unroll
        for (int k = 0; k < (NX > 0 ? NX : 1); ++k)
#pragma unroll
            for (int ib = 0; ib < NB; ++ib) accx[k][ib][0] = accx[k][ib][1] = 0.0;
        const int m = lane >> 2, kq = lane & 3;
        // slot block 0 = [q | levels 1..S | 0 0]: q (Q_j's last column) from the
        // slot, the levels from the next raw block (global, written ≤ 2 lines
        // ago by the MPK warp); blocks b ≥ 1 = prefix columns 8(b−1) + m of
        // [Q[:, 0:c0] | Q_j] < c0n, all from the slot
        const int c0n = a.c0n;
        const double* lev = a.Vn + m * ld;
        const bool lev_on = m >= 1 && m < a.w;
        int gb = 0, tb = 0;  // this CTA's Gram lines / line steps of the previous tasks
        for_tasks([&](int wx, int y0, int y1, bool down) {
            const int len = y1 - y0;
            const int g0 = ((crank - S) % CL + CL) % CL;  // first in-band line whose update step is ours
            const int gown = len > g0 ? (len - g0 + CL - 1) / CL : 0;
            for (int k = ((gw - gb) % kFuG + kFuG) % kFuG; k < gown; k += kFuG) {  // gg ≡ gw (mod kFuG)
                const int g = g0 + k * CL, gg = gb + k, gs = gg % kGR;
                wait_on(&gready[gs], (gg / kGR) & 1);
                const int line = down ? y1 - 1 - g : y0 + g;
                const int tt = tb + (g + S - crank) / CL;  // this CTA's slot of the line's update step
                const double* st = slot_of(tt) + H + kq;  // core rows start at slot row H
                const int cbase = wx * STEP + kq;
                const i64 rbase = static_cast<i64>(line) * nx64 + cbase;
                // the line's level fragments (global) in one batch: one L2 round trip per line
                double lv[STEP / 4];
#pragma unroll
                for (int c = 0; c < STEP / 4; ++c)
                    lv[c] = (lev_on && cbase + 4 * c < nx) ? lev[rbase + 4 * c] : 0.0;
#pragma unroll
                for (int c = 0; c < STEP / 4; ++c) {
                    const bool ok = cbase + 4 * c < nx;
                    double f[NB];
                    f[0] = !ok ? 0.0 : m == 0 ? st[voff + (WMAX - 1) * kBox + 4 * c] : lv[c];
#pragma unroll
                    for (int b = 1; b < NB; ++b) {
                        const int col = 8 * (b - 1) + m;
                        f[b] = (ok && col < c0n) ? st[(col < cp ? col * kBox : voff + (col - cp) * kBox) + 4 * c] : 0.0;
                    }
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) dmma(acc[ib][0], acc[ib][1], f[ib], f[0]);
                    if constexpr (NX > 0) {
#pragma unroll
                        for (int k2 = 0; k2 < NX; ++k2) {
                            const int xb = a.xb0 + k2;
                            double fx = 0.0;
#pragma unroll
                            for (int b = 1; b < NB; ++b)
                                if (b == xb) fx = f[b];
#pragma unroll
                            for (int ib = 1; ib < NB; ++ib)
                                if (ib <= xb) dmma(accx[k2][ib][0], accx[k2][ib][1], f[ib], fx);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    arrive_on(&gempty[crank * kGR + gs], 0);
                    mbar_arrive(&lfree[tt % nbar]);
                }
            }
            gb += gown;
            tb += own_count(len + 2 * S);
        });
        // cross-warp sums in fixed warp order (K3's packed tile layout), through
        // the update ring: free once this CTA's update warps are done (bar 2)
        asm volatile("bar.sync 2, %0;" ::"n"((kFuU + kFuG) * 32));
        double* scratch = ring;
        const int e0 = (lane >> 2) + 8 * (2 * (lane & 3));
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
            double* t = scratch + (static_cast<size_t>(gw) * T + ib) * 64;
            t[e0] = acc[ib][0];
            t[e0 + 8] = acc[ib][1];
        }
        if constexpr (NX > 0) {
#pragma unroll
            for (int k = 0; k < NX; ++k)
#pragma unroll
                for (int ib = 1; ib < NB; ++ib) {
                    double* t = scratch + (static_cast<size_t>(gw) * T + NB + k * (NB - 1) + (ib - 1)) * 64;
                    t[e0] = accx[k][ib][0];
                    t[e0 + 8] = accx[k][ib][1];
                }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFuG * 32));
        constexpr int per_cta = T * 64;
        double* out = a.partials + static_cast<size_t>(blockIdx.x) * per_cta;
        for (int e = gw * 32 + lane; e < per_cta; e += kFuG * 32) {
            double sum = scratch[e];
#pragma unroll
            for (int v = 1; v < kFuG; ++v) sum += scratch[static_cast<size_t>(v) * per_cta + e];
            out[e] = sum;
        }
    }
    // no CTA of a cluster leaves while a peer may still arrive on its barriers
    // or write its q ring
    if constexpr (CL > 1) cluster_sync_all();
}

template <int S, int WMAX, int NB, int CL>
const void* fused_fn_nb(int nb, int nx) {
    if (nb == NB) {
        if (nx == 0) return reinterpret_cast<const void*>(fused_pass_kernel<S, WMAX, NB, 0, CL>);
        if constexpr (NB > 1) {
            if (nx == 1) return reinterpret_cast<const void*>(fused_pass_kernel<S, WMAX, NB, 1, CL>);
            if (nx == 2) return reinterpret_cast<const void*>(fused_pass_kernel<S, WMAX, NB, 2, CL>);
        }
        return nullptr;
    }
    if constexpr (NB < 8) return fused_fn_nb<S, WMAX, NB + 1, CL>(nb, nx);
    return nullptr;
}

constexpr size_t kFuSmem = 225 * 1024;
size_t fused_slot_bytes(i64 c0) { return static_cast<size_t>(round_up(c0 * kBox, 16) + round_up(6 * kBox, 16)) * 8; }
constexpr int kMaxCl = 2;  // cluster size of the paired variant
size_t fused_fixed_smem(i64 c0) {
    return static_cast<size_t>(4 * kMaxSlots + (kMaxCl + 1) * kQR + (kMaxCl + 1) * kGR) * 8 +
           static_cast<size_t>(kMaxCl * kQR) * 32 * 16 + static_cast<size_t>(c0 + 7) * 6 * 8;
}
// KRY_FUSED_CLUSTER=2: a CTA pair (thread-block cluster) per window column,
// the line slots split between the two SMs' shared memory (2× the lines in
// flight), q and the Gram-ready signals crossing the pair through DSMEM and
// cluster-scope mbarriers.  Parity-green but measured far slower than one CTA
// per window (4000²: 88.1 vs 34.6 ms per cycle; 8000²: 342 vs 135 ms): every
// line step now waits on a cross-SM handoff.  Default 1.
int fused_cluster() {
    static const int cl = [] {
        const char* e = std::getenv("KRY_FUSED_CLUSTER");
        return e && std::atoi(e) == 2 ? 2 : 1;
    }();
    return cl;
}

}  // namespace

bool fused_pass_supported(const StencilGeom& g, int s, i64 w, i64 c0n, i64 ld, const double* Q,
                          const double* V, const double* Vn) {
    auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return g.dims == 2 && g.jacobi == 0 && g.line0 == 0 && g.lines == g.ny && (g.nx & 1) == 0 && s == 5 && w == s + 1 &&
           update_wmax(w) == 6 && c0n + w <= 64 && (ld & 1) == 0 && a16(Q) && a16(V) && a16(Vn) &&
           // the widest fused update (prefix c0n − w + 1) still gets S + 2 ring slots
           static_cast<size_t>(s + 2) * fused_slot_bytes(c0n - w + 1) + fused_fixed_smem(c0n - w + 1) <= kFuSmem &&
           g.nx + 64 < (i64(1) << 31) && g.ny < (i64(1) << 30);
}

i64 fused_partials_doubles() { return static_cast<i64>(device_sms()) * (8 + 2 * 7) * 64; }

void launch_fused_pass(cudaStream_t stream, const StencilGeom& g, int s, FusedPassArgs a, double* d_packed,
                       int64_t& launches) {
    const int h = (s + 1) & ~1, step = 64 - 2 * h;
    const int nb = 1 + static_cast<int>(round_up(a.c0n, 8) / 8);
    int nxt = 0;
    if (a.x_count > 0) {
        const int s0 = 8 + a.x_first, s1 = s0 + a.x_count - 1;
        a.xb0 = s0 / 8;
        nxt = s1 / 8 - a.xb0 + 1;
        if (nxt > 2 || s1 / 8 >= nb) fail(KRY_INTERNAL, "fused pass: extra-column shape");
    } else {
        a.xb0 = 0;
    }
    const int CL = fused_cluster();
    const void* fn = s != 5 ? nullptr : CL == 2 ? fused_fn_nb<5, 6, 1, 2>(nb, nxt) : fused_fn_nb<5, 6, 1, 1>(nb, nxt);
    if (!fn) fail(KRY_UNSUPPORTED, "fused pass shape");
    a.nx = static_cast<int>(g.nx);
    a.ny = static_cast<int>(g.ny);
    const i64 nwx = ceil_div(g.nx, step);
    const i64 sms = device_sms() / CL;  // clusters (one window column each)
    // bands per window: minimise rounds × (band + 2S) line steps per cluster
    {
        i64 best = -1, best_cost = 0;
        for (i64 nb = 1; nb <= std::max<i64>(1, g.ny / (4 * s)) && nb <= 4096; ++nb) {
            const i64 tasks = nwx * nb, rounds = ceil_div(tasks, sms);
            const i64 cost = rounds * (ceil_div(g.ny, nb) + 2 * s);
            if (best < 0 || cost < best_cost) {
                best = nb;
                best_cost = cost;
            }
        }
        a.nbands = static_cast<int>(best);
        a.ntasks = static_cast<int>(nwx * best);
    }
    const int T = nb + nxt * (nb - 1);
    FusedMaps maps{};
    // window lines start at arbitrary rows: no 256-byte L2 promotion (it would
    // fetch three 256-byte sectors groups per 512-byte column run)
    if (a.c0 > 0) maps.p = dev::tensor_map_2d(a.Q, a.ld, g.nloc, a.c0, kBox, a.c0, false);
    maps.v = dev::tensor_map_2d(a.V, a.ld, g.nloc, a.w, kBox, a.w, false);
    // ring slots: a line's slot lives from its TMA load until its Gram, S
    // lines after its update, so at least S + 2 (one line of prefetch)
    const size_t slot_bytes = fused_slot_bytes(a.c0);
    const size_t fixed = fused_fixed_smem(a.c0);
    int nslots = static_cast<int>(std::min<size_t>(kMaxSlots, (kFuSmem - fixed) / slot_bytes));
    if (nslots < s + 2) fail(KRY_UNSUPPORTED, "fused pass: shared memory");
    const size_t ring = std::max(static_cast<size_t>(nslots) * slot_bytes, static_cast<size_t>(kFuG) * T * 64 * 8);
    const size_t smem = ring + fixed;
    set_kernel_smem(fn, smem);
    const int grid = CL * static_cast<int>(std::max<i64>(1, std::min<i64>(sms, a.ntasks)));
    if (static_cast<i64>(grid) * T * 64 > fused_partials_doubles()) fail(KRY_INTERNAL, "fused pass partials");
    void* args[] = {&maps, &a, &nslots};
    if (!launches_suppressed()) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kFuThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = CL;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        KB_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    }
    KB_LAUNCHED();
    launch_gram_reduce(stream, a.partials, grid, T * 64, d_packed);
    launches += 2;
}

}  // namespace kb
