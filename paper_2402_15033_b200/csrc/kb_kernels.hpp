// Host-callable launchers for the sm_100a kernels of the hot path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "kb_common.hpp"

namespace kb {

// Resident blocks per SM of a kernel at a block size / dynamic smem (cached:
// the occupancy query costs microseconds of host time per launch).
int occupancy(const void* kernel, int threads, size_t smem);

// ---- k_tsqr.cu : BlkOrtho (K3 Gram, K5 update) ---------------------------
std::vector<std::pair<i64, i64>> prefix_groups(i64 c0, i64 w);
i64 gram_scratch_doubles(i64 w);
// Packed G tiles for one prefix group: tile_ids[t] = jb*8 + ib, 64 entries
// per tile (8×8 column-major), written to d_packed in tile order.
// x_first/x_count (optional, w ≤ 8 only): also return P[:,0:cp]ᵀ·P[:, x_first:x_first+x_count]
// as extra tiles (ids 64 + xb*8 + ib, P-slot coordinates) — the panel Gram
// pieces the two-stage finalize reuses (kb_store.cpp).
void launch_gram_pass(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V,
                      i64 ldv, i64 w, bool vv, double* d_partials, double* d_packed,
                      std::vector<int>& tile_ids, int64_t& launches, i64 x_first = -1, i64 x_count = 0);
int update_wmax(i64 w);
// out = [V | P]·M on DMMA; d_mfrag holds M in fragment order (k_tsqr.cu, K5b).
// Requires round_up(w,8) + round_up(cp,8) ≤ 64.
void launch_update_mma(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V, i64 ldv,
                       i64 w, const double* d_mfrag, double* out, i64 ldo, int64_t& launches);
// out = (V − P·R_col)·R_jj⁻¹ (triangular) or V − P·R_col; out may alias V.
// skip (device flag, optional): the kernel returns without writing when *skip != 0.
void launch_update(cudaStream_t stream, i64 n, const double* P, i64 ldp, i64 cp, const double* V, i64 ldv,
                   i64 w, const double* d_coef, bool triangular, double* out, i64 ldo, int64_t& launches,
                   const int* skip = nullptr);

// Fixed-order sum of per-CTA Gram partials (K3 layout) into packed tiles.
void launch_gram_reduce(cudaStream_t stream, const double* partials, int grid, int per_cta, double* packed);
void set_kernel_smem(const void* kernel, size_t bytes);
int device_sms();

// ---- k_pip.cu : device BCGS-PIP factorisation (speculative first stage) --
// Result slot of one block (doubles): [kSlotStatus] 0 = committed, p > 0 =
// Cholesky pivot p failed, −1 = an earlier block of the chain failed;
// [kSlotRcol …] R_col (c0×w) then R_jj (w×w), column-major; [kSlotPieces …]
// the panel-Gram pieces P[:,0:c0]ᵀ·P[:, x_first:x_first+x_count] (c0×x_count).
constexpr int kSlotStatus = 0, kSlotRcol = 8, kSlotPieces = 8 + 64 * 8 + 64, kSlotDoubles = 2048;
struct PipBlockArgs {
    const double* packed;     // reduced (and allreduced) packed Gram tiles of the block
    int nb;                   // slot blocks: 1 (V) + prefix blocks; regular tiles = nb
    int nx, xb0;              // extra prefix column blocks (panel-Gram pieces)
    int x_first, x_count;
    int c0, w, wmax;          // wmax: K5 column padding (update_wmax)
    double* slot;
    const double* prev_slot;  // the previous speculative block's slot, or nullptr
    double* coef;             // K5 coefficients for this block's update
    int* skip;                // K5 skip flag: set when this block (or an earlier one) failed
    int mode;                 // 0: BCGS-PIP factorisation; 1: bcgs_project (coefficients −R_col only)
};
void launch_pip_block(cudaStream_t stream, const PipBlockArgs& a, int64_t& launches);

// ---- k_ops.cu : operators (K1/K2), restart-loop vectors (K8-K10) ---------
struct StencilGeom {
    int dims;        // 2 or 3
    i64 nx, ny, nz;  // grid
    i64 row_begin;   // first global row owned
    i64 nloc;        // rows owned
    i64 halo;        // halo length (nx for 2D, nx*ny for 3D)
    // derived on the host (kernel-uniform, no device division):
    i64 lines;       // owned grid lines (nloc / nx)
    i64 line0;       // global index of the first owned line
    i64 z0;          // first owned plane (3D)
    i64 nzl;         // owned planes (3D)
    // Jacobi-scaled operator D⁻¹A (kry_operator_jacobi): off-diagonal
    // coefficient c_off = −1/diag (rounded), diagonal 1; else −1 / diag.
    int jacobi;
    double c_off;
};
StencilGeom make_stencil_geom(int dims, i64 nx, i64 ny, i64 nz, i64 row_begin, i64 nloc);
// y = A·x (b == nullptr) or r = b − A·x with Σr² partials (b != nullptr);
// returns the number of partials written.
int launch_stencil(cudaStream_t s, const StencilGeom& g, const double* x, const double* halo_lo,
                   const double* halo_hi, const double* b, double* y, double* partials, int64_t& launches);
int stencil_partials(const StencilGeom& g);
// Fused 2-D MPK: out[:, k−1] = A^k·x, k = 1..s (out columns ldo apart), one
// pass; halos hold s lines each (multi-rank).
// force: skip the size heuristic (tests).
bool mpk2d_supported(const StencilGeom& g, int s, const double* x, const double* out, i64 ldo, bool force);
void launch_mpk2d(cudaStream_t st, const StencilGeom& g, const double* x, const double* halo_lo,
                  const double* halo_hi, double* out, i64 ldo, int s, int64_t& launches);
// Fused 3-D MPK (7-point stencil, temporal blocking along z): out[:, k−1] =
// A^k·x (or (D⁻¹A)^k·x with jacobi), k = 1..s ≤ 7; halos hold s planes each.
bool mpk3d_supported(const StencilGeom& g, int s, const double* x, const double* out, i64 ldo, bool force);
void launch_mpk3d(cudaStream_t st, const StencilGeom& g, const double* x, const double* halo_lo,
                  const double* halo_hi, double* out, i64 ldo, int s, int64_t& launches);
// CSR rows (row_ptr local, from 0) gathering x through int32 indices.
int launch_csr(cudaStream_t s, i64 nloc, const int64_t* row_ptr, const int32_t* col, const double* vals,
               const double* x, const double* b, double* y, double* partials, int64_t& launches);
// Column-sliced CSR (nslices ≥ 2): slice p holds each row's entries whose
// (gathered) column lies in the p-th column range, in stored order, with its
// own int32 row_ptr; the passes continue one running sum per row
// (part_sum, nloc doubles) so every row is still summed in stored order.
int launch_csr_sliced(cudaStream_t s, i64 nloc, int nslices, const int32_t* const* row_ptr,
                      const int32_t* const* col, const double* const* vals, const double* x, const double* b,
                      double* y, double* partials, double* part_sum, int64_t& launches);
int reduce_grid();  // fixed grid of every partial-sum kernel (determinism)

// ---- k_peer.cu : one-shot deterministic allreduce over NVLink peer memory --
constexpr int kPeerMaxRanks = 8;
constexpr int kPeerMaxDoubles = 16384;  // per slot (the widest packed Gram is ~2.3 K doubles)
struct PeerTable {
    double* data[kPeerMaxRanks];   // each rank's receive area [2][nranks][kPeerMaxDoubles]
    uint64_t* flags[kPeerMaxRanks];  // each rank's flags [2][nranks]
};
void launch_peer_allreduce(cudaStream_t s, double* d, int count, const PeerTable& t, int rank, int nranks,
                           uint64_t epoch, int64_t& launches);
// Jacobi (D⁻¹A formed in place on the device; D⁻¹b per solve).  One of
// rp64 / rp32 is non-null (unsliced CSR / one column slice).
void launch_csr_find_diag(cudaStream_t s, i64 nloc, const int64_t* rp64, const int32_t* rp32, const int32_t* col,
                          const double* vals, i64 diag_col0, double* d, int64_t& launches);
void launch_csr_scale_rows(cudaStream_t s, i64 nloc, const int64_t* rp64, const int32_t* rp32, double* vals,
                           const double* d, int64_t& launches);
void launch_count_zero(cudaStream_t s, i64 n, const double* d, unsigned long long* zeros, int64_t& launches);
// out = b / d (d == nullptr: b / dconst), IEEE division.
void launch_div_diag(cudaStream_t s, i64 n, const double* b, const double* d, double dconst, double* out,
                     int64_t& launches);

// ---- k_fused.cu : K6 fused first-stage pass (update j → MPK j+1 → Gram j+1)
struct FusedPassArgs {
    double* Q;              // store (column-major, ld)
    i64 ld;
    const double* V;        // raw block j (w columns, ld), read-only
    double* Vn;             // raw block j+1 out: column 0 = q, 1..s = A^k·q
    int c0, w;              // block j: prefix columns, width
    const double* coef;     // K5 coefficients of block j (k_pip.cu layout, wmax 6)
    const int* skip;        // block j's skip flag
    int c0n;                // block j+1 prefix columns (= c0 + w − 1)
    int x_first, x_count;   // panel-Gram pieces of block j+1 (prefix columns)
    double* partials;       // per-CTA Gram partials (fused_partials_doubles())
    // set by the launcher
    int xb0 = 0, nx = 0, ny = 0;
    int ntasks = 0, nbands = 0;  // (window, band) tasks
};
bool fused_pass_supported(const StencilGeom& g, int s, i64 w, i64 c0n, i64 ld, const double* Q, const double* V,
                          const double* Vn);
i64 fused_partials_doubles();
// Launches K6 and the reduce of its Gram into d_packed (K3 packed tiles of
// block j+1, the layout launch_pip_block reads).
void launch_fused_pass(cudaStream_t stream, const StencilGeom& g, int s, FusedPassArgs a, double* d_packed,
                       int64_t& launches);

void launch_finalize_sum(cudaStream_t s, const double* partials, int count, double* out,
                         int64_t& launches);
void launch_scale_div(cudaStream_t s, i64 n, const double* r, double gamma, double* out,
                      int64_t& launches);
struct Coef64 {
    double v[64];
};
void launch_xupdate(cudaStream_t s, i64 n, const double* x, const double* Q, i64 ldq, int k,
                    const Coef64& y, double* xnew, int64_t& launches);

}  // namespace kb
