// Operator and restart-loop kernels for sm_100a.
//
// K1/K2  stencil / CSR kernels: y = A·x with every row summed in the
//        reference's stored (ascending column) order, s = 0.0 start, no FMA
//        contraction (spmv, csr_matrix.hpp:69-79) — bit-identical to the CPU
//        reference.  The stencils reproduce gen_laplace2d(nx,ny,5) and
//        gen_laplace3d (matgen.hpp:134-187) matrix-free: 16 B/row of HBM
//        traffic instead of CSR's ~76 B/row.
// K9     the same kernels in residual mode: r = b − A·x fused with the Σr²
//        partials of ‖r‖ (gmres.hpp:189-194 + dense_matrix.hpp:139).
// K8     xupdate_kernel: x_new = x + Σ_l y_l q_l, l ascending (gmres.hpp:257-259).
// K10    scale_div_kernel: v1 = r / γ (gmres.hpp:286-287).
// All partial sums use one fixed grid and fixed-order trees: results are
// reproducible run to run (no float atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <type_traits>

#include "kb_common.hpp"
#include "kb_device.hpp"
#include "kb_kernels.hpp"

namespace kb {

namespace {

constexpr int kBlock = 256;

int num_sms() {
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

// Fixed-order block sum; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double warp_part[kBlock / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) warp_part[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kBlock / 32; ++w) s += warp_part[w];
    return s;
}

__device__ __forceinline__ double acc_term(double s, double coeff, double x) {
    return __dadd_rn(s, __dmul_rn(coeff, x));
}
// acc_term(s, −1, x): −1·x is exact (a sign flip), so one add of −x gives
// the same bits.
__device__ __forceinline__ double sub_term(double s, double x) { return __dadd_rn(s, -x); }
// Stencil terms of A (JAC = false: off-diagonal −1, diagonal d) or of the
// Jacobi-scaled D⁻¹A (JAC: off-diagonal c = −1/d rounded, diagonal d/d = 1),
// each in the form spmv computes it on the (pre-scaled) CSR: the rounded
// product, then the add (csr_matrix.hpp:75).
template <bool JAC>
__device__ __forceinline__ double off_term(double s, double c, double x) {
    return JAC ? acc_term(s, c, x) : sub_term(s, x);
}
template <bool JAC>
__device__ __forceinline__ double diag_term(double s, double d, double x) {
    return JAC ? __dadd_rn(s, x) : acc_term(s, d, x);
}

constexpr int kLinesPerThread = 8;

// x over one grid line (ix), y over chunks of kLinesPerThread owned lines
// that each thread walks in order.  The 2-D kernel carries the line below
// and the current line in registers, so each row loads one new line value
// plus its two (L1-resident) horizontal neighbours.  All geometry is
// precomputed on the host (no device integer division).  Ranks own whole
// lines (2D) / planes (3D); out-of-rank neighbours come from the halos.
template <int DIMS, bool RESID, bool JAC>
__global__ void __launch_bounds__(kBlock) stencil_kernel(const StencilGeom g, const double* __restrict__ x,
                                                         const double* __restrict__ halo_lo,
                                                         const double* __restrict__ halo_hi,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y,
                                                         double* __restrict__ partials) {
    KB_PDL_WAIT();
    const i64 ix = blockIdx.x * static_cast<i64>(kBlock) + threadIdx.x;
    const i64 nx = g.nx;
    double sq = 0.0;
    if (ix < nx) {
        for (i64 lc = static_cast<i64>(blockIdx.y) * kLinesPerThread; lc < g.lines;
             lc += static_cast<i64>(gridDim.y) * kLinesPerThread) {
            const i64 lend = min(lc + kLinesPerThread, g.lines);
            i64 i = lc * nx + ix;  // local row
            if (DIMS == 2) {
                i64 gl = g.line0 + lc;  // global grid line
                double down = 0.0;
                if (gl > 0) down = lc > 0 ? x[i - nx] : halo_lo[ix];
                double cur = x[i];
                for (i64 l = lc; l < lend; ++l, ++gl, i += nx) {
                    const bool has_up = gl + 1 < g.ny;
                    double up = 0.0;
                    if (has_up) up = l + 1 < g.lines ? x[i + nx] : halo_hi[ix];
                    double s = 0.0;
                    if (gl > 0) s = off_term<JAC>(s, g.c_off, down);
                    if (ix > 0) s = off_term<JAC>(s, g.c_off, x[i - 1]);
                    s = diag_term<JAC>(s, 4.0, cur);
                    if (ix + 1 < nx) s = off_term<JAC>(s, g.c_off, x[i + 1]);
                    if (has_up) s = off_term<JAC>(s, g.c_off, up);
                    if (RESID) {
                        const double r = __dsub_rn(b[i], s);
                        y[i] = r;
                        sq = fma(r, r, sq);
                    } else {
                        y[i] = s;
                    }
                    down = cur;
                    cur = up;
                }
            } else {
                const i64 plane = nx * g.ny;
                const i64 gl0 = g.line0 + lc;
                i64 iz = gl0 / g.ny;  // once per chunk
                i64 iy = gl0 - iz * g.ny;
                for (i64 l = lc; l < lend; ++l, i += nx) {
                    const i64 zl = iz - g.z0;
                    const i64 hp = iy * nx + ix;  // offset inside a halo plane
                    double s = 0.0;
                    if (iz > 0) s = off_term<JAC>(s, g.c_off, zl > 0 ? x[i - plane] : halo_lo[hp]);
                    if (iy > 0) s = off_term<JAC>(s, g.c_off, x[i - nx]);
                    if (ix > 0) s = off_term<JAC>(s, g.c_off, x[i - 1]);
                    s = diag_term<JAC>(s, 6.0, x[i]);
                    if (ix + 1 < nx) s = off_term<JAC>(s, g.c_off, x[i + 1]);
                    if (iy + 1 < g.ny) s = off_term<JAC>(s, g.c_off, x[i + nx]);
                    if (iz + 1 < g.nz) s = off_term<JAC>(s, g.c_off, zl + 1 < g.nzl ? x[i + plane] : halo_hi[hp]);
                    if (RESID) {
                        const double r = __dsub_rn(b[i], s);
                        y[i] = r;
                        sq = fma(r, r, sq);
                    } else {
                        y[i] = s;
                    }
                    if (++iy == g.ny) {
                        iy = 0;
                        ++iz;
                    }
                }
            }
        }
    }
    if (RESID) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// 2-D 5-point stencil, two adjacent columns per thread (nx even): one 16-byte
// load of the next line per step, the current/previous lines carried in
// registers, the horizontal neighbours x[i-1], x[i+2] taken from the
// neighbouring lanes by shuffle (only lanes 0/31 touch memory for them).
// Same per-row summation order as stencil_kernel (bit-identical).
template <bool RESID, bool JAC>
__global__ void __launch_bounds__(kBlock) stencil2d_vec_kernel(const StencilGeom g, const double* __restrict__ x,
                                                               const double* __restrict__ halo_lo,
                                                               const double* __restrict__ halo_hi,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ y,
                                                               double* __restrict__ partials) {
    KB_PDL_WAIT();
    const i64 ix = 2 * (blockIdx.x * static_cast<i64>(kBlock) + threadIdx.x);
    const i64 nx = g.nx;
    const bool active = ix < nx;
    const int lane = threadIdx.x & 31;
    double sq = 0.0;
    for (i64 lc = static_cast<i64>(blockIdx.y) * kLinesPerThread; lc < g.lines;
         lc += static_cast<i64>(gridDim.y) * kLinesPerThread) {
        const i64 lend = min(lc + kLinesPerThread, g.lines);
        i64 gl = g.line0 + lc;
        double2 down = make_double2(0.0, 0.0), cur = make_double2(0.0, 0.0);
        if (active) {
            if (gl > 0)
                down = lc > 0 ? *reinterpret_cast<const double2*>(x + (lc - 1) * nx + ix)
                              : *reinterpret_cast<const double2*>(halo_lo + ix);
            cur = *reinterpret_cast<const double2*>(x + lc * nx + ix);
        }
#pragma unroll
        for (int k = 0; k < kLinesPerThread; ++k) {
            const i64 l = lc + k;
            if (l >= lend) break;  // uniform across the block
            const i64 i = l * nx + ix;
            const bool has_up = gl + 1 < g.ny;
            double2 up = make_double2(0.0, 0.0);
            if (active && has_up)
                up = l + 1 < g.lines ? *reinterpret_cast<const double2*>(x + i + nx)
                                     : *reinterpret_cast<const double2*>(halo_hi + ix);
            double left = __shfl_up_sync(0xffffffffu, cur.y, 1);
            double right = __shfl_down_sync(0xffffffffu, cur.x, 1);
            if (active) {
                if (lane == 0 && ix > 0) left = x[i - 1];
                if (lane == 31 && ix + 2 < nx) right = x[i + 2];
                double s0 = 0.0, s1 = 0.0;
                if (gl > 0) s0 = off_term<JAC>(s0, g.c_off, down.x);
                if (ix > 0) s0 = off_term<JAC>(s0, g.c_off, left);
                s0 = diag_term<JAC>(s0, 4.0, cur.x);
                s0 = off_term<JAC>(s0, g.c_off, cur.y);
                if (has_up) s0 = off_term<JAC>(s0, g.c_off, up.x);
                if (gl > 0) s1 = off_term<JAC>(s1, g.c_off, down.y);
                s1 = off_term<JAC>(s1, g.c_off, cur.x);
                s1 = diag_term<JAC>(s1, 4.0, cur.y);
                if (ix + 2 < nx) s1 = off_term<JAC>(s1, g.c_off, right);
                if (has_up) s1 = off_term<JAC>(s1, g.c_off, up.y);
                if (RESID) {
                    const double2 bb = *reinterpret_cast<const double2*>(b + i);
                    const double r0 = __dsub_rn(bb.x, s0), r1 = __dsub_rn(bb.y, s1);
                    *reinterpret_cast<double2*>(y + i) = make_double2(r0, r1);
                    sq = fma(r0, r0, sq);
                    sq = fma(r1, r1, sq);
                } else {
                    *reinterpret_cast<double2*>(y + i) = make_double2(s0, s1);
                }
            }
            down = cur;
            cur = up;
            ++gl;
        }
    }
    if (RESID) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// 3-D 7-point stencil, two adjacent columns per thread (nx even): threads
// tile one plane (pairs of one grid row, rows of the plane), each walks
// kPlanesPerThread planes along z carrying the planes below and current in
// registers (one new 16-byte load per plane from HBM); the y-neighbour rows
// are the same plane's rows that neighbouring threads load (L1/L2 hits), the
// x-neighbours come by shuffle.  Same per-row summation order as
// stencil_kernel<3> (bit-identical).
constexpr int kPlanesPerThread = 8;

template <bool RESID, bool JAC>
__global__ void __launch_bounds__(kBlock, 6) stencil3d_vec_kernel(const StencilGeom g, const double* __restrict__ x,
                                                                  const double* __restrict__ halo_lo,
                                                                  const double* __restrict__ halo_hi,
                                                                  const double* __restrict__ b,
                                                                  double* __restrict__ y,
                                                                  double* __restrict__ partials) {
    KB_PDL_WAIT();
    const int nx = static_cast<int>(g.nx), ny = static_cast<int>(g.ny), half = nx / 2;
    const i64 plane = g.nx * g.ny;
    const int q = blockIdx.x * kBlock + threadIdx.x;  // pair index inside a plane
    const bool active = q < half * ny;
    const int iy = active ? q / half : 0;
    const int ix = active ? 2 * (q - iy * half) : 0;
    const int off = iy * nx + ix;
    const bool has_ym = iy > 0, has_yp = iy + 1 < ny, has_l = ix > 0, has_r = ix + 2 < nx;
    const int lane = threadIdx.x & 31;
    auto ld2 = [](const double* p) { return *reinterpret_cast<const double2*>(p); };
    // every lane of the warp has all four in-plane neighbours (the lanes at
    // the warp's ends still read their outer x-neighbour from memory): the
    // interior planes then take a branch-free path (same terms, same order;
    // MPK 3.28 -> 3.21 ms per 256³ cycle, profiles/stencil3d_fast_ab_r02.log)
    const bool warp_inside = __all_sync(0xffffffffu, active && has_ym && has_yp && has_l && has_r);
    double sq = 0.0;
    const int nzl = static_cast<int>(g.nzl), nz = static_cast<int>(g.nz), z0 = static_cast<int>(g.z0);
    for (int zc = blockIdx.y * kPlanesPerThread; zc < nzl; zc += gridDim.y * kPlanesPerThread) {
        const int zend = min(zc + kPlanesPerThread, nzl);
        int gz = z0 + zc;
        const double* xc = x + zc * plane + off;  // this thread's pair in the current plane
        double* yc = y + zc * plane + off;
        const double* bc = RESID ? b + zc * plane + off : nullptr;
        double2 down = make_double2(0.0, 0.0), cur = make_double2(0.0, 0.0);
        if (active) {
            if (gz > 0) down = zc > 0 ? ld2(xc - plane) : ld2(halo_lo + off);
            cur = ld2(xc);
        }
#pragma unroll 1
        for (int l = zc; l < zend; ++l, ++gz, xc += plane, yc += plane) {
            const bool has_dn = gz > 0, has_up = gz + 1 < nz;
            double2 up = make_double2(0.0, 0.0);
            if (active && has_up) up = l + 1 < nzl ? ld2(xc + plane) : ld2(halo_hi + off);
            double left = __shfl_up_sync(0xffffffffu, cur.y, 1);
            double right = __shfl_down_sync(0xffffffffu, cur.x, 1);
            if (warp_inside && has_dn && has_up) {
                if (lane == 0) left = xc[-1];
                if (lane == 31) right = xc[2];
                const double2 ym = ld2(xc - nx), yp = ld2(xc + nx);
                double s0 = off_term<JAC>(0.0, g.c_off, down.x);
                s0 = off_term<JAC>(s0, g.c_off, ym.x);
                s0 = off_term<JAC>(s0, g.c_off, left);
                s0 = diag_term<JAC>(s0, 6.0, cur.x);
                s0 = off_term<JAC>(s0, g.c_off, cur.y);
                s0 = off_term<JAC>(s0, g.c_off, yp.x);
                s0 = off_term<JAC>(s0, g.c_off, up.x);
                double s1 = off_term<JAC>(0.0, g.c_off, down.y);
                s1 = off_term<JAC>(s1, g.c_off, ym.y);
                s1 = off_term<JAC>(s1, g.c_off, cur.x);
                s1 = diag_term<JAC>(s1, 6.0, cur.y);
                s1 = off_term<JAC>(s1, g.c_off, right);
                s1 = off_term<JAC>(s1, g.c_off, yp.y);
                s1 = off_term<JAC>(s1, g.c_off, up.y);
                if (RESID) {
                    const double2 bb = ld2(bc);
                    bc += plane;
                    const double r0 = __dsub_rn(bb.x, s0), r1 = __dsub_rn(bb.y, s1);
                    *reinterpret_cast<double2*>(yc) = make_double2(r0, r1);
                    sq = fma(r0, r0, sq);
                    sq = fma(r1, r1, sq);
                } else {
                    *reinterpret_cast<double2*>(yc) = make_double2(s0, s1);
                }
            } else if (active) {
                if (lane == 0 && has_l) left = xc[-1];
                if (lane == 31 && has_r) right = xc[2];
                const double2 ym = has_ym ? ld2(xc - nx) : make_double2(0.0, 0.0);
                const double2 yp = has_yp ? ld2(xc + nx) : make_double2(0.0, 0.0);
                double s0 = 0.0, s1 = 0.0;
                if (has_dn) s0 = off_term<JAC>(s0, g.c_off, down.x);
                if (has_ym) s0 = off_term<JAC>(s0, g.c_off, ym.x);
                if (has_l) s0 = off_term<JAC>(s0, g.c_off, left);
                s0 = diag_term<JAC>(s0, 6.0, cur.x);
                s0 = off_term<JAC>(s0, g.c_off, cur.y);
                if (has_yp) s0 = off_term<JAC>(s0, g.c_off, yp.x);
                if (has_up) s0 = off_term<JAC>(s0, g.c_off, up.x);
                if (has_dn) s1 = off_term<JAC>(s1, g.c_off, down.y);
                if (has_ym) s1 = off_term<JAC>(s1, g.c_off, ym.y);
                s1 = off_term<JAC>(s1, g.c_off, cur.x);
                s1 = diag_term<JAC>(s1, 6.0, cur.y);
                if (has_r) s1 = off_term<JAC>(s1, g.c_off, right);
                if (has_yp) s1 = off_term<JAC>(s1, g.c_off, yp.y);
                if (has_up) s1 = off_term<JAC>(s1, g.c_off, up.y);
                if (RESID) {
                    const double2 bb = ld2(bc);
                    bc += plane;
                    const double r0 = __dsub_rn(bb.x, s0), r1 = __dsub_rn(bb.y, s1);
                    *reinterpret_cast<double2*>(yc) = make_double2(r0, r1);
                    sq = fma(r0, r0, sq);
                    sq = fma(r1, r1, sq);
                } else {
                    *reinterpret_cast<double2*>(yc) = make_double2(s0, s1);
                }
            }
            down = cur;
            cur = up;
        }
    }
    if (RESID) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// 3-D 7-point stencil, plane tiles: a CTA of 8 warps owns a 64 × 8 (x × y)
// tile of grid columns — warp w is tile row w, lane l columns 2l, 2l+1 —
// and walks kT3Planes planes along z with the planes below / current / above
// of its own columns in registers (one new 16-byte load per plane from
// HBM).  The y-neighbours of the tile's interior rows come from a shared
// copy of the current plane (double-buffered by step parity, one barrier
// per plane) instead of from L2 (stencil3d_vec_kernel reads every cell three
// times: as its own value and as both rows' y-neighbour); only the tile's
// edge rows read their outer neighbour from global memory.  x-neighbours by
// shuffle.  Same per-row summation order as stencil_kernel<3>
// (bit-identical).
constexpr int kT3Rows = 8;
constexpr int kT3Planes = 16;

template <bool RESID, bool JAC>
__global__ void __launch_bounds__(kBlock) stencil3d_tile_kernel(const StencilGeom g, const double* __restrict__ x,
                                                                const double* __restrict__ halo_lo,
                                                                const double* __restrict__ halo_hi,
                                                                const double* __restrict__ b,
                                                                double* __restrict__ y,
                                                                double* __restrict__ partials) {
    KB_PDL_WAIT();
    __shared__ double2 tile[2][kT3Rows][32];
    const int nx = static_cast<int>(g.nx), ny = static_cast<int>(g.ny);
    const i64 plane = g.nx * g.ny;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ntx = (nx + 63) / 64;
    const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
    const int ix = tx * 64 + 2 * lane, iy = ty * kT3Rows + w;
    const bool active = ix < nx && iy < ny;  // nx even: both columns or neither
    const bool has_ym = iy > 0, has_yp = iy + 1 < ny, has_l = ix > 0, has_r = ix + 2 < nx;
    const int off = iy * nx + ix;
    auto ld2 = [](const double* p) { return *reinterpret_cast<const double2*>(p); };
    const double c = g.c_off;
    double sq = 0.0;
    const int nzl = static_cast<int>(g.nzl), nz = static_cast<int>(g.nz), z0 = static_cast<int>(g.z0);
    const int zc = blockIdx.y * kT3Planes, zend = min(zc + kT3Planes, nzl);
    int gz = z0 + zc;
    const double* xc = x + static_cast<i64>(zc) * plane + off;
    double* yc = y + static_cast<i64>(zc) * plane + off;
    const double* bc = RESID ? b + static_cast<i64>(zc) * plane + off : nullptr;
    double2 down = make_double2(0.0, 0.0), cur = make_double2(0.0, 0.0);
    if (active && zc < nzl) {
        if (gz > 0) down = zc > 0 ? ld2(xc - plane) : ld2(halo_lo + off);
        cur = ld2(xc);
    }
    int par = 0;
#pragma unroll 1
    for (int l = zc; l < zend; ++l, ++gz, xc += plane, yc += plane) {
        const bool has_dn = gz > 0, has_up = gz + 1 < nz;
        double2 up = make_double2(0.0, 0.0);
        if (active && has_up) up = l + 1 < nzl ? ld2(xc + plane) : ld2(halo_hi + off);
        tile[par][w][lane] = cur;
        __syncthreads();
        double left = __shfl_up_sync(0xffffffffu, cur.y, 1);
        double right = __shfl_down_sync(0xffffffffu, cur.x, 1);
        if (active) {
            if (lane == 0 && has_l) left = xc[-1];
            if (lane == 31 && has_r) right = xc[2];
            const double2 ym = !has_ym ? make_double2(0.0, 0.0) : w > 0 ? tile[par][w - 1][lane] : ld2(xc - nx);
            const double2 yp = !has_yp ? make_double2(0.0, 0.0)
                                       : w + 1 < kT3Rows ? tile[par][w + 1][lane] : ld2(xc + nx);
            double s0 = 0.0, s1 = 0.0;
            if (has_dn) s0 = off_term<JAC>(s0, c, down.x);
            if (has_ym) s0 = off_term<JAC>(s0, c, ym.x);
            if (has_l) s0 = off_term<JAC>(s0, c, left);
            s0 = diag_term<JAC>(s0, 6.0, cur.x);
            s0 = off_term<JAC>(s0, c, cur.y);
            if (has_yp) s0 = off_term<JAC>(s0, c, yp.x);
            if (has_up) s0 = off_term<JAC>(s0, c, up.x);
            if (has_dn) s1 = off_term<JAC>(s1, c, down.y);
            if (has_ym) s1 = off_term<JAC>(s1, c, ym.y);
            s1 = off_term<JAC>(s1, c, cur.x);
            s1 = diag_term<JAC>(s1, 6.0, cur.y);
            if (has_r) s1 = off_term<JAC>(s1, c, right);
            if (has_yp) s1 = off_term<JAC>(s1, c, yp.y);
            if (has_up) s1 = off_term<JAC>(s1, c, up.y);
            if (RESID) {
                const double2 bb = ld2(bc);
                bc += plane;
                const double r0 = __dsub_rn(bb.x, s0), r1 = __dsub_rn(bb.y, s1);
                *reinterpret_cast<double2*>(yc) = make_double2(r0, r1);
                sq = fma(r0, r0, sq);
                sq = fma(r1, r1, sq);
            } else {
                *reinterpret_cast<double2*>(yc) = make_double2(s0, s1);
            }
        }
        down = cur;
        cur = up;
        par ^= 1;
    }
    if (RESID) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

dim3 stencil3d_tile_grid(const StencilGeom& g) {
    const i64 tiles = ceil_div(g.nx, 64) * ceil_div(g.ny, kT3Rows);
    const i64 chunks = std::max<i64>(1, ceil_div(g.nzl, kT3Planes));
    return dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(std::min<i64>(chunks, 65535)));
}

// K2f: the whole s-step MPK of the 5-point stencil in one pass
// (mpk_monomial, gmres.hpp:80-90): out[:, k−1] = A^k·x for k = 1..S.
// Temporal blocking: each warp owns a 64-column window (32 lanes × double2)
// and a band of grid lines, and streams the band's input lines once, bottom
// to top.  Level k runs 2k − 1 lines behind the input (skewed wavefront):
// at step t it produces line L − 2k + 1 from lines of level k − 1 finished in
// the three previous steps, so the S levels of one step are independent
// (ILP instead of an S-deep dependency chain).  Each level keeps its last
// three lines in a register ring indexed by t mod 3, and the input lines
// are prefetched three steps ahead in a second ring; the step loop is
// unrolled by 3 so no ring ever moves.  Horizontal neighbours come by
// shuffle.  Level k is valid on the window shrunk by k columns per side, so
// a window outputs its middle 64 − 2H columns (H = S rounded up to even)
// and neighbouring windows overlap by 2H; bands start S lines early
// (recomputed, never stored).  HBM traffic per MPK: one read of x (+ the
// overlaps, mostly L2) and S writes, versus S reads and S writes for S
// separate SpMVs.
//
// Bit-identity with spmv (csr_matrix.hpp:72-77): every element is
// 0.0 + t_0 + t_1 + … in stored column order with t = −x (exact, so one
// add of the negated value) or 4·x.  Absent neighbours (grid edges) are
// carried as +0.0 and added as −0.0: a running sum that starts at +0.0 can
// never be −0.0 under round-to-nearest, so s + (−0.0) = s bit for bit — the
// same result as skipping the term.
constexpr int kMpkRing = 3;

template <int S, bool JAC>
__device__ __forceinline__ void mpk2d_task(const StencilGeom& g, const double* __restrict__ x,
                                           const double* __restrict__ halo_lo, const double* __restrict__ halo_hi,
                                           double* __restrict__ out, i64 ldo, int wb, int wx, int band, int lane) {
    constexpr int H = (S + 1) & ~1;
    constexpr int STEP = 64 - 2 * H;
    // 32-bit line/column arithmetic (grid dimensions < 2^31; checked by
    // mpk2d_supported), 64-bit only in addresses.
    const int nx = static_cast<int>(g.nx), ny = static_cast<int>(g.ny);
    const int lines = static_cast<int>(g.lines), line0 = static_cast<int>(g.line0);
    const int ix = wx * STEP - H + 2 * lane;  // this lane's first column (even)
    const bool in_grid = ix >= 0 && ix < nx;  // nx even: both columns or neither
    const bool store_lane = in_grid && lane >= H / 2 && lane < 32 - H / 2;
    const int y0 = wb * band, y1 = min(y0 + band, lines);
    // Input lines from ls: S below the band (or from the grid's first line);
    // level S reaches line y1 − 1 at step y1 + 2S − 2 − ls.
    const int ls = max(y0 - S, -line0);
    const int steps = y1 + 2 * S - 1 - ls;
    const int lmax = min(lines + S, ny - line0);  // first line with no data (zeros above)
    const i64 nx64 = nx;
    auto load = [&](int l) -> double2 {
        double2 v = make_double2(0.0, 0.0);
        if (in_grid && l < lmax) {
            const double* p = l < 0        ? halo_lo + static_cast<i64>(l + S) * nx64
                              : l < lines ? x + static_cast<i64>(l) * nx64
                                          : halo_hi + static_cast<i64>(l - lines) * nx64;
            v = __ldg(reinterpret_cast<const double2*>(p + ix));
        }
        return v;
    };
    // r[t mod 3][j]: level j's line finished at step t (level 0: input line).
    double2 r[kMpkRing][S];
#pragma unroll
    for (int q = 0; q < kMpkRing; ++q)
#pragma unroll
        for (int j = 0; j < S; ++j) r[q][j] = make_double2(0.0, 0.0);
    double2 pf[kMpkRing];  // input lines of steps t, t+1, t+2
#pragma unroll
    for (int q = 0; q < kMpkRing; ++q) pf[q] = load(ls + q);
    double* const out_ix = out + ix;
    // FAST: every level's line this step lies inside the band and the grid
    // (warp-uniform), so the per-level line checks drop out; same values.
    auto step = [&](auto phase, auto fast, int st) {
        constexpr int P = decltype(phase)::value;  // st ≡ P (mod 3)
        constexpr bool FAST = decltype(fast)::value;
        constexpr int P1 = (P + 2) % 3, P2 = (P + 1) % 3, P3 = P;  // steps t−1, t−2, t−3
        const int L = ls + st;
        const double2 in = pf[P];
        pf[P] = load(L + kMpkRing);
        double* const orow = out_ix + static_cast<i64>(L) * nx64;
        // Top level first: level k reads the old lines of level k − 1
        // (slot P3 holds step t − 3 until level k − 1 overwrites it below).
#pragma unroll
        for (int k = S; k >= 1; --k) {
            const int l = L - 2 * k + 1;  // level k's line this step
            const int gl = line0 + l;
            const double2 dn = k == 1 ? r[P2][0] : r[P3][k - 1];
            const double2 cu = k == 1 ? r[P1][0] : r[P2][k - 1];
            const double2 up = k == 1 ? in : r[P1][k - 1];
            const double left = __shfl_up_sync(0xffffffffu, cu.y, 1);
            const double right = __shfl_down_sync(0xffffffffu, cu.x, 1);
            double s0 = off_term<JAC>(0.0, g.c_off, dn.x);
            s0 = off_term<JAC>(s0, g.c_off, left);
            s0 = diag_term<JAC>(s0, 4.0, cu.x);
            s0 = off_term<JAC>(s0, g.c_off, cu.y);
            s0 = off_term<JAC>(s0, g.c_off, up.x);
            double s1 = off_term<JAC>(0.0, g.c_off, dn.y);
            s1 = off_term<JAC>(s1, g.c_off, cu.x);
            s1 = diag_term<JAC>(s1, 4.0, cu.y);
            s1 = off_term<JAC>(s1, g.c_off, right);
            s1 = off_term<JAC>(s1, g.c_off, up.y);
            // outside the grid (lines or columns): exactly +0.0
            const bool live = in_grid && (FAST || (gl >= 0 && gl < ny));
            const double2 v = live ? make_double2(s0, s1) : make_double2(0.0, 0.0);
            if (store_lane && (FAST || (l >= y0 && l < y1)))
                *reinterpret_cast<double2*>(orow + ((k - 1) * ldo - (2 * k - 1) * nx64)) = v;
            if (k < S) r[P][k] = v;
        }
        r[P][0] = in;
    };
    const int lo_ok = max(y0, -line0), hi_ok = min(y1, ny - line0);
    for (int st = 0; st < steps; st += kMpkRing) {  // steps past the end are harmless (nothing stored)
        // levels' lines over these three steps: ls + st − 2S + 1 … ls + st + 1
        if (ls + st - 2 * S + 1 >= lo_ok && ls + st + 1 < hi_ok) {
            step(std::integral_constant<int, 0>{}, std::true_type{}, st);
            step(std::integral_constant<int, 1>{}, std::true_type{}, st + 1);
            step(std::integral_constant<int, 2>{}, std::true_type{}, st + 2);
        } else {
            step(std::integral_constant<int, 0>{}, std::false_type{}, st);
            step(std::integral_constant<int, 1>{}, std::false_type{}, st + 1);
            step(std::integral_constant<int, 2>{}, std::false_type{}, st + 2);
        }
    }
}

template <int S, bool JAC>
__global__ void __launch_bounds__(kBlock, 2) mpk2d_kernel(const StencilGeom g, const double* __restrict__ x,
                                                       const double* __restrict__ halo_lo,
                                                       const double* __restrict__ halo_hi,
                                                       double* __restrict__ out, i64 ldo, i64 nwx, i64 band,
                                                       i64 ntasks) {
    KB_PDL_WAIT();
    const int lane = threadIdx.x & 31;
    const i64 nwarps = static_cast<i64>(gridDim.x) * (kBlock / 32);
    for (i64 task = blockIdx.x * static_cast<i64>(kBlock / 32) + (threadIdx.x >> 5); task < ntasks;
         task += nwarps)  // whole warps only
        mpk2d_task<S, JAC>(g, x, halo_lo, halo_hi, out, ldo, static_cast<int>(task / nwx), static_cast<int>(task % nwx),
                      static_cast<int>(band), lane);
}

// K2g: the whole s-step MPK of the 7-point stencil in one pass
// (mpk_monomial, gmres.hpp:80-90, on gen_laplace3d, matgen.hpp:167-187):
// out[:, k−1] = A^k·x for k = 1..S.  Temporal blocking along z: a CTA of
// 16 warps owns a 64 × 32 (x × y) tile of grid columns — warp w holds tile
// rows 2w and 2w + 1, lane l columns 2l and 2l + 1 of both (two double2) —
// and a band of z-planes, and streams the band's input planes once, bottom
// to top.  Level k runs k planes behind the input (at step t it produces
// plane zs + t − k); the S levels of a step are computed bottom-up, so level
// k's upper neighbour (level k − 1, plane + 1) was produced earlier in the
// same step; a thread's own columns one plane below sit in registers, two
// planes below in its own cells of the shared slot.  In-plane neighbours: x by shuffle;
// y from the thread's other row, or — for the rows the next warps own —
// from a shared-memory copy of each level's plane, double-buffered by step
// parity (read slot t − 1, write slot t, one __syncthreads per step; rows
// −1 and 32 are zero padding).  Level k is valid on the tile shrunk by k
// cells per side (x by H = S rounded up to even, for the double2 columns),
// so a tile outputs its middle (64 − 2H) × (32 − 2S) columns and
// neighbouring tiles overlap; the band starts S planes early (recomputed,
// never stored).  HBM traffic: one read of x (+ the overlaps, mostly L2)
// and S writes, against S reads and S writes for S separate SpMVs.
// Bit-identity with spmv: every element is 0.0 + t_0 + … + t_6 in stored
// column order (z−1, y−1, x−1, centre, x+1, y+1, z+1); absent neighbours
// are carried as +0.0 and added as −0.0 (see K2f).  Interior tiles and
// steps (warp-uniform) skip the grid-edge masks.  JAC: the Jacobi-scaled
// operator D⁻¹A (off_term / diag_term).
constexpr int kMpk3Rows = 32;               // tile rows (y)
constexpr int kMpk3Warps = kMpk3Rows / 2;   // two tile rows per warp
constexpr int kMpk3Pad = kMpk3Rows + 2;     // shared plane rows (zero rows −1 and 32)

template <int S, bool JAC>
__global__ void __launch_bounds__(kMpk3Warps * 32, 1)
    mpk3d_kernel(const StencilGeom g, const double* __restrict__ x, const double* __restrict__ halo_lo,
                 const double* __restrict__ halo_hi, double* __restrict__ out, i64 ldo, int nwx, int nwy,
                 int band, int ntasks) {
    KB_PDL_WAIT();
    constexpr int H = (S + 1) & ~1;
    constexpr int STEPX = 64 - 2 * H;
    constexpr int STEPY = kMpk3Rows - 2 * S;
    constexpr int PLANE = kMpk3Pad * 32;  // double2 per shared plane
    extern __shared__ double2 sm3[];      // [2 slots][S levels][kMpk3Pad rows][32 lanes]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r0 = 2 * w;  // tile rows r0, r0 + 1
    const int nx = static_cast<int>(g.nx), ny = static_cast<int>(g.ny), nz = static_cast<int>(g.nz);
    const int nzl = static_cast<int>(g.nzl), z0 = static_cast<int>(g.z0);
    const i64 nx64 = nx, plane = static_cast<i64>(nx) * ny;
    const double c = g.c_off;
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
        const int wx = task % nwx, wy = (task / nwx) % nwy, wz = task / (nwx * nwy);
        const int tx0 = wx * STEPX - H, ty0 = wy * STEPY - S;  // tile origin
        const int ix = tx0 + 2 * lane, iy = ty0 + r0;
        const bool inx = ix >= 0 && ix < nx;  // nx even: both columns or neither
        const bool in0 = inx && iy >= 0 && iy < ny, in1 = inx && iy + 1 >= 0 && iy + 1 < ny;
        const bool tile_inside = tx0 >= 0 && tx0 + 64 <= nx && ty0 >= 0 && ty0 + kMpk3Rows <= ny;
        const bool st_lane = lane >= H / 2 && lane < 32 - H / 2;
        const bool st0 = st_lane && in0 && r0 >= S && r0 < kMpk3Rows - S;
        const bool st1 = st_lane && in1 && r0 + 1 >= S && r0 + 1 < kMpk3Rows - S;
        const int zb0 = wz * band, zb1 = min(zb0 + band, nzl);
        const int zs = max(zb0 - S, -z0);        // first input plane (local index)
        const int zmax = min(nzl + S, nz - z0);  // first plane with no data (zeros above)
        const int steps = zb1 - zs + S;
        const i64 cell = static_cast<i64>(iy) * nx64 + ix;
        // input plane l, rows r0 and r0 + 1 (+0.0 outside the grid)
        auto load2 = [&](int l, double2& v0, double2& v1) {
            v0 = v1 = make_double2(0.0, 0.0);
            if (l >= zmax) return;
            const double* p = (l >= 0 && l < nzl) ? x + static_cast<i64>(l) * plane
                              : l < 0           ? halo_lo + static_cast<i64>(l + S) * plane
                                                : halo_hi + static_cast<i64>(l - nzl) * plane;
            p += cell;
            if (in0) v0 = __ldg(reinterpret_cast<const double2*>(p));
            if (in1) v1 = __ldg(reinterpret_cast<const double2*>(p + nx64));
        };
        // a0/a1[j]: level j's two rows at the plane of step t − 1 (registers);
        // the plane of step t − 2 is this thread's own cell of shared slot t & 1,
        // read just before this step's value of the level replaces it
        double2 a0[S], a1[S];
#pragma unroll
        for (int j = 0; j < S; ++j) a0[j] = a1[j] = make_double2(0.0, 0.0);
        double2 pf[2][2];  // input planes of steps t, t + 1 (ring by step parity)
        load2(zs, pf[0][0], pf[0][1]);
        load2(zs + 1, pf[1][0], pf[1][1]);
        __syncthreads();  // the previous task's last reads of the shared planes are done
        // zero both slots (the "step −1" and "step −2" planes and the padding rows)
        for (int i = threadIdx.x; i < 2 * S * PLANE; i += blockDim.x) sm3[i] = make_double2(0.0, 0.0);
        __syncthreads();
        double2* const mine = sm3 + (r0 + 1) * 32 + lane;  // padded row r0 + 1 ↔ tile row r0
        double* const orow = out + cell;
        // one step: P = t mod 2 selects the prefetch slot (unrolled by two so
        // the ring never moves; the next load goes out after the slot's last use)
        // level k's output rows of plane l live at out + (k − 1)·ldo + l·plane:
        // per step one base pointer, per level one constant stride (ldo − plane)
        const i64 dk = ldo - plane;
        // one step: P = t mod 2 selects the prefetch slot and the shared slots
        // (unrolled by two so the ring never moves; the next load goes out after
        // the slot's last use).  FAST: every level's plane this step lies inside
        // the grid and the band and the tile inside the grid — no masks, no
        // per-level plane checks (same values).
        auto step = [&](auto parity, auto fastc, int t) {
            constexpr int P = decltype(parity)::value;
            constexpr bool FAST = decltype(fastc)::value;
            const int lt = zs + t;  // input plane this step
            double2 u0 = pf[P][0], u1 = pf[P][1];  // level 0 (the input) at plane lt
            double* o = orow + static_cast<i64>(lt) * plane - ldo;  // level 0 "output" base; level k: + k·dk
#pragma unroll
            for (int k = 1; k <= S; ++k) {
                o += dk;
                double2* const qc = mine + (P * S + (k - 1)) * PLANE;              // level k − 1, slot t (holds t − 2)
                const double2* const qp = mine + ((P ^ 1) * S + (k - 1)) * PLANE;  // level k − 1, slot t − 1
                const double2 dn0 = qc[0], dn1 = qc[32];
                qc[0] = u0;  // publish level k − 1's plane of this step
                qc[32] = u1;
                const double2 cu0 = a0[k - 1], cu1 = a1[k - 1];
                a0[k - 1] = u0;
                a1[k - 1] = u1;
                const double2 ym0 = qp[-32], yp1 = qp[64];
                const double l0 = __shfl_up_sync(0xffffffffu, cu0.y, 1), r0v = __shfl_down_sync(0xffffffffu, cu0.x, 1);
                const double l1 = __shfl_up_sync(0xffffffffu, cu1.y, 1), r1v = __shfl_down_sync(0xffffffffu, cu1.x, 1);
                // row r0: y−1 from the shared plane, y+1 = this thread's row r0 + 1
                double s0 = off_term<JAC>(0.0, c, dn0.x);
                s0 = off_term<JAC>(s0, c, ym0.x);
                s0 = off_term<JAC>(s0, c, l0);
                s0 = diag_term<JAC>(s0, 6.0, cu0.x);
                s0 = off_term<JAC>(s0, c, cu0.y);
                s0 = off_term<JAC>(s0, c, cu1.x);
                s0 = off_term<JAC>(s0, c, u0.x);
                double s1 = off_term<JAC>(0.0, c, dn0.y);
                s1 = off_term<JAC>(s1, c, ym0.y);
                s1 = off_term<JAC>(s1, c, cu0.x);
                s1 = diag_term<JAC>(s1, 6.0, cu0.y);
                s1 = off_term<JAC>(s1, c, r0v);
                s1 = off_term<JAC>(s1, c, cu1.y);
                s1 = off_term<JAC>(s1, c, u0.y);
                // row r0 + 1: y−1 = this thread's row r0, y+1 from the shared plane
                double s2 = off_term<JAC>(0.0, c, dn1.x);
                s2 = off_term<JAC>(s2, c, cu0.x);
                s2 = off_term<JAC>(s2, c, l1);
                s2 = diag_term<JAC>(s2, 6.0, cu1.x);
                s2 = off_term<JAC>(s2, c, cu1.y);
                s2 = off_term<JAC>(s2, c, yp1.x);
                s2 = off_term<JAC>(s2, c, u1.x);
                double s3 = off_term<JAC>(0.0, c, dn1.y);
                s3 = off_term<JAC>(s3, c, cu0.y);
                s3 = off_term<JAC>(s3, c, cu1.x);
                s3 = diag_term<JAC>(s3, 6.0, cu1.y);
                s3 = off_term<JAC>(s3, c, r1v);
                s3 = off_term<JAC>(s3, c, yp1.y);
                s3 = off_term<JAC>(s3, c, u1.y);
                double2 v0 = make_double2(s0, s1), v1 = make_double2(s2, s3);
                bool lin = true;
                if constexpr (!FAST) {
                    // outside the grid: exactly +0.0 (an absent neighbour of a valid cell)
                    const int l = lt - k;  // level k's plane this step
                    const int gz = z0 + l;
                    const bool zin = gz >= 0 && gz < nz;
                    if (!(in0 && zin)) v0 = make_double2(0.0, 0.0);
                    if (!(in1 && zin)) v1 = make_double2(0.0, 0.0);
                    lin = l >= zb0 && l < zb1;
                }
                if (lin && st0) *reinterpret_cast<double2*>(o) = v0;
                if (lin && st1) *reinterpret_cast<double2*>(o + nx64) = v1;
                u0 = v0;  // level k at plane l: level k + 1's upper neighbour
                u1 = v1;
            }
            load2(lt + 2, pf[P][0], pf[P][1]);
            __syncthreads();
        };
        const int fast_lo = max(zb0, -z0) + S, fast_hi = min(zb1, nz - z0);  // fast ⇔ lt ∈ [fast_lo, fast_hi]
        for (int t = 0; t < steps; t += 2) {
            const int lt = zs + t;
            if (tile_inside && lt >= fast_lo && lt + 1 <= fast_hi) {
                step(std::integral_constant<int, 0>{}, std::true_type{}, t);
                if (t + 1 < steps) step(std::integral_constant<int, 1>{}, std::true_type{}, t + 1);
            } else {
                step(std::integral_constant<int, 0>{}, std::false_type{}, t);
                if (t + 1 < steps) step(std::integral_constant<int, 1>{}, std::false_type{}, t + 1);
            }
        }
    }
}

// CSR SpMV, one warp per 32 consecutive rows, in two phases per chunk of
// the warp's contiguous nnz range (kCsrChunk entries):
//  1. gather — lanes stride over the chunk's entries (coalesced val / col
//     loads, streamed past L2 with evict-first so x keeps the cache) and form
//     the products val·x[col]; all kCsrChunk/32 gathers of a lane are issued
//     before any is used, so the random x reads overlap instead of
//     serialising behind each row's running sum;
//  2. sum — each lane adds its own row's products from shared memory in
//     stored order.
// The product is the same rounded __dmul_rn as in the sequential loop and
// the adds keep spmv's order (csr_matrix.hpp:72-77): bit-identical.
constexpr int kCsrChunk = 256;

// MODE: CSR_ONLY (s from 0.0, write y), or one pass of a column-sliced SpMV
// (see Operator in kb_operator.cpp): CSR_FIRST (s from 0.0, write the
// partial), CSR_MID (partial in/out), CSR_LAST (partial in, write y).
enum CsrMode { CSR_ONLY = 0, CSR_FIRST = 1, CSR_MID = 2, CSR_LAST = 3 };

template <int MODE, bool RESID, typename RP>
__global__ void __launch_bounds__(kBlock) csr_warp_kernel(i64 nloc, const RP* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ vals,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ b, double* __restrict__ y,
                                                          double* __restrict__ partials, double* part_sum) {
    KB_PDL_WAIT();
    __shared__ double s_prod[kBlock / 32][kCsrChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 stride = static_cast<i64>(gridDim.x) * (kBlock / 32) * 32;
    double sq = 0.0;
    for (i64 r0 = (static_cast<i64>(blockIdx.x) * (kBlock / 32) + warp) * 32; r0 < nloc; r0 += stride) {
        const i64 row = r0 + lane;
        const bool live = row < nloc;
        const i64 rs = live ? static_cast<i64>(row_ptr[row]) : 0, re = live ? static_cast<i64>(row_ptr[row + 1]) : 0;
        const i64 last = (nloc - 1 - r0) < 31 ? (nloc - 1 - r0) : 31;
        const i64 base = __shfl_sync(0xffffffffu, rs, 0);
        const i64 end = __shfl_sync(0xffffffffu, re, static_cast<int>(last));
        double s = 0.0;
        if ((MODE == CSR_MID || MODE == CSR_LAST) && live) s = part_sum[row];
        for (i64 cs = base; cs < end; cs += kCsrChunk) {
            const int cnt = static_cast<int>((end - cs) < kCsrChunk ? (end - cs) : kCsrChunk);
            int cidx[kCsrChunk / 32];
            double v[kCsrChunk / 32];
#pragma unroll
            for (int u = 0; u < kCsrChunk / 32; ++u) {
                const int k = lane + 32 * u;
                cidx[u] = k < cnt ? __ldcs(col + cs + k) : 0;
                v[u] = k < cnt ? __ldcs(vals + cs + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kCsrChunk / 32; ++u) {
                const int k = lane + 32 * u;
                if (k < cnt) {
                    const double xv = __ldcg(x + cidx[u]);  // no L1 allocation for random gathers
                    s_prod[warp][k] = __dmul_rn(v[u], xv);
                }
            }
            __syncwarp();
            const i64 a0 = max(rs, cs), a1 = min(re, cs + cnt);
            for (i64 k = a0; k < a1; ++k) s = __dadd_rn(s, s_prod[warp][k - cs]);
            __syncwarp();
        }
        if (live) {
            if (MODE == CSR_FIRST || MODE == CSR_MID) {
                part_sum[row] = s;
            } else if (RESID) {
                const double r = __dsub_rn(b[row], s);
                y[row] = r;
                sq = fma(r, r, sq);
            } else {
                y[row] = s;
            }
        }
    }
    if (RESID && (MODE == CSR_ONLY || MODE == CSR_LAST)) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kBlock) finalize_kernel(const double* __restrict__ partials, int count,
                                                          double* __restrict__ out) {
    KB_PDL_WAIT();
    double s = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) s += partials[i];
    const double t = block_sum(s);
    if (threadIdx.x == 0) out[0] = t;
}

__global__ void __launch_bounds__(kBlock) scale_div_kernel(i64 n, const double* __restrict__ r, double gamma,
                                                           double* __restrict__ out) {
    KB_PDL_WAIT();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = r[i] / gamma;
}

__global__ void __launch_bounds__(kBlock) xupdate_kernel(i64 n, const double* __restrict__ x,
                                                         const double* __restrict__ q, i64 ldq, int k,
                                                         const Coef64 y, double* __restrict__ xnew) {
    KB_PDL_WAIT();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        double s = x[i];
        for (int l = 0; l < k; ++l) s = fma(y.v[l], q[i + l * ldq], s);
        xnew[i] = s;
    }
}

int grid_for(i64 n) {
    const i64 g = ceil_div(n, kBlock);
    return static_cast<int>(std::max<i64>(1, std::min<i64>(g, i64(1) << 30)));  // one row per thread
}

}  // namespace

int reduce_grid() { return num_sms() * 16; }

dim3 stencil_grid(const StencilGeom& g) {
    const i64 chunks = std::max<i64>(1, ceil_div(g.lines, kLinesPerThread));
    return dim3(static_cast<unsigned>(ceil_div(g.nx, kBlock)), static_cast<unsigned>(std::min<i64>(chunks, 65535)));
}

StencilGeom make_stencil_geom(int dims, i64 nx, i64 ny, i64 nz, i64 row_begin, i64 nloc) {
    StencilGeom g{};
    g.dims = dims;
    g.nx = nx;
    g.ny = ny;
    g.nz = dims == 2 ? 1 : nz;
    g.row_begin = row_begin;
    g.nloc = nloc;
    g.halo = dims == 2 ? nx : nx * ny;
    g.lines = nloc / nx;
    g.line0 = row_begin / nx;
    g.z0 = dims == 2 ? 0 : row_begin / (nx * ny);
    g.nzl = dims == 2 ? 0 : nloc / (nx * ny);
    g.jacobi = 0;
    g.c_off = -1.0;
    return g;
}

dim3 stencil3d_vec_grid(const StencilGeom& g) {
    const i64 chunks = std::max<i64>(1, ceil_div(g.nzl, kPlanesPerThread));
    return dim3(static_cast<unsigned>(ceil_div(g.nx / 2 * g.ny, kBlock)),
                static_cast<unsigned>(std::min<i64>(chunks, 65535)));
}

int stencil_partials(const StencilGeom& g) {
    const dim3 d = stencil_grid(g), v = stencil3d_vec_grid(g), t = stencil3d_tile_grid(g);
    return static_cast<int>(std::max({d.x * d.y, g.dims == 3 ? v.x * v.y : 0u, g.dims == 3 ? t.x * t.y : 0u}));
}

int launch_stencil(cudaStream_t s, const StencilGeom& g, const double* x, const double* halo_lo,
                   const double* halo_hi, const double* b, double* y, double* partials, int64_t& launches) {
    auto a16 = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (g.dims == 2 && (g.nx & 1) == 0 && a16(x) && a16(y) && a16(b) && a16(halo_lo) && a16(halo_hi)) {
        dim3 grid = stencil_grid(g);
        grid.x = static_cast<unsigned>(ceil_div(g.nx / 2, kBlock));
        if (b)
            (g.jacobi ? launch_pdl(stencil2d_vec_kernel<true, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil2d_vec_kernel<true, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        else
            (g.jacobi ? launch_pdl(stencil2d_vec_kernel<false, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil2d_vec_kernel<false, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        KB_LAUNCHED();
        ++launches;
        return b ? static_cast<int>(grid.x * grid.y) : 0;
    }
    // KRY_STENCIL3D_VEC: 0 = scalar kernel, 1 (default) = stencil3d_vec_kernel
    // (y-neighbours from L1/L2), 2 = stencil3d_tile_kernel (y-neighbours from a
    // shared plane tile; bit-identical, measured no faster: 3.59 vs 3.49 ms of
    // MPK per 256³ cycle — the L2 re-reads were not the bound)
    static const int vec3 = [] {
        const char* e = std::getenv("KRY_STENCIL3D_VEC");
        return e ? std::atoi(e) : 1;
    }();
    if (vec3 == 2 && g.dims == 3 && (g.nx & 1) == 0 && g.nx * g.ny < (i64(1) << 30) && g.nzl < (i64(1) << 30) &&
        a16(x) && a16(y) && a16(b) && a16(halo_lo) && a16(halo_hi) && ceil_div(g.nx, 64) * ceil_div(g.ny, kT3Rows) < (i64(1) << 31)) {
        const dim3 grid = stencil3d_tile_grid(g);
        if (b)
            (g.jacobi ? launch_pdl(stencil3d_tile_kernel<true, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil3d_tile_kernel<true, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        else
            (g.jacobi ? launch_pdl(stencil3d_tile_kernel<false, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil3d_tile_kernel<false, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        KB_LAUNCHED();
        ++launches;
        return b ? static_cast<int>(grid.x * grid.y) : 0;
    }
    if (vec3 && g.dims == 3 && (g.nx & 1) == 0 && g.nx * g.ny < (i64(1) << 30) && g.nzl < (i64(1) << 30) && a16(x) && a16(y) && a16(b) && a16(halo_lo) && a16(halo_hi)) {
        const dim3 grid = stencil3d_vec_grid(g);
        if (b)
            (g.jacobi ? launch_pdl(stencil3d_vec_kernel<true, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil3d_vec_kernel<true, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        else
            (g.jacobi ? launch_pdl(stencil3d_vec_kernel<false, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil3d_vec_kernel<false, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        KB_LAUNCHED();
        ++launches;
        return b ? static_cast<int>(grid.x * grid.y) : 0;
    }
    const dim3 grid = stencil_grid(g);
    if (g.dims == 2) {
        if (b)
            (g.jacobi ? launch_pdl(stencil_kernel<2, true, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil_kernel<2, true, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        else
            (g.jacobi ? launch_pdl(stencil_kernel<2, false, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil_kernel<2, false, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
    } else {
        if (b)
            (g.jacobi ? launch_pdl(stencil_kernel<3, true, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil_kernel<3, true, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
        else
            (g.jacobi ? launch_pdl(stencil_kernel<3, false, true>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials) : launch_pdl(stencil_kernel<3, false, false>, grid, kBlock, 0, s, g, x, halo_lo, halo_hi, b, y, partials));
    }
    KB_LAUNCHED();
    ++launches;
    return b ? static_cast<int>(grid.x * grid.y) : 0;
}

int occupancy(const void* kernel, int threads, size_t smem) {
    struct Key {
        const void* k;
        int t;
        size_t s;
        bool operator==(const Key& o) const { return k == o.k && t == o.t && s == o.s; }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.k) * 31u ^ std::hash<size_t>()(k.s * 4099u + static_cast<size_t>(k.t));
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, int, Hash> cache;
    std::lock_guard<std::mutex> lock(mu);
    const Key key{kernel, threads, smem};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    cache.emplace(key, per_sm);
    return per_sm;
}

bool mpk2d_supported(const StencilGeom& g, int s, const double* x, const double* out, i64 ldo, bool force) {
    auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (!(g.dims == 2 && (g.nx & 1) == 0 && s >= 1 && s <= 8 && (ldo & 1) == 0 && a16(x) && a16(out) &&
          g.lines >= 1 && g.nx + 64 < (i64(1) << 31) && g.ny + 64 < (i64(1) << 31)))
        return false;
    // Worth it once the (window, band) tasks give every SM a warp: each
    // warp's wavefront is a serial chain, so tiny grids stay on the
    // per-SpMV kernels (at 512² the fused block already wins: 0.109 vs
    // 0.118 s to solution).
    const int h = (s + 1) & ~1;
    const i64 tasks = ceil_div(g.nx, 64 - 2 * h) * std::max<i64>(1, g.lines / (2 * s));
    return force || tasks >= static_cast<i64>(num_sms());
}

void launch_mpk2d(cudaStream_t st, const StencilGeom& g, const double* x, const double* halo_lo,
                  const double* halo_hi, double* out, i64 ldo, int s, int64_t& launches) {
    const int h = (s + 1) & ~1, step = 64 - 2 * h;
    const i64 nwx = ceil_div(g.nx, step);
    auto go = [&](auto kernel) {
        // One wave of resident warps, one (window, band) task each: bands as
        // tall as that allows (the 2s-line band overlap is recomputed), at
        // least 2 lines; very wide grids loop over tasks.  A warp walks
        // band + 2s − 1 dependent steps, so on small grids (idle warps) short
        // bands win: 512², s = 5: 16.9 → ~10 µs per block with 2-line bands.
        const int per_sm = occupancy(reinterpret_cast<const void*>(kernel), kBlock, 0);
        const i64 resident = static_cast<i64>(num_sms()) * std::max(per_sm, 1) * (kBlock / 32);
        const i64 nbands = std::max<i64>(1, std::min<i64>(resident / nwx, g.lines / 2));
        i64 band = ceil_div(g.lines, nbands);
        if (const char* e = std::getenv("KRY_MPK_BAND")) band = std::max<i64>(1, std::atoll(e));  // A/B
        const i64 ntasks = nwx * ceil_div(g.lines, band);
        const unsigned grid = static_cast<unsigned>(
            std::min<i64>(ceil_div(ntasks, kBlock / 32), static_cast<i64>(num_sms()) * std::max(per_sm, 1)));
        launch_pdl(kernel, grid, kBlock, 0, st, g, x, halo_lo, halo_hi, out, ldo, nwx, band, ntasks);
    };
    switch (s) {
        case 1: g.jacobi ? go(mpk2d_kernel<1, true>) : go(mpk2d_kernel<1, false>); break;
        case 2: g.jacobi ? go(mpk2d_kernel<2, true>) : go(mpk2d_kernel<2, false>); break;
        case 3: g.jacobi ? go(mpk2d_kernel<3, true>) : go(mpk2d_kernel<3, false>); break;
        case 4: g.jacobi ? go(mpk2d_kernel<4, true>) : go(mpk2d_kernel<4, false>); break;
        case 5: g.jacobi ? go(mpk2d_kernel<5, true>) : go(mpk2d_kernel<5, false>); break;
        case 6: g.jacobi ? go(mpk2d_kernel<6, true>) : go(mpk2d_kernel<6, false>); break;
        case 7: g.jacobi ? go(mpk2d_kernel<7, true>) : go(mpk2d_kernel<7, false>); break;
        case 8: g.jacobi ? go(mpk2d_kernel<8, true>) : go(mpk2d_kernel<8, false>); break;
        default: fail(KRY_INTERNAL, "mpk2d: unsupported s");
    }
    KB_LAUNCHED();
    ++launches;
}

bool mpk3d_supported(const StencilGeom& g, int s, const double* x, const double* out, i64 ldo, bool force) {
    auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (!(g.dims == 3 && (g.nx & 1) == 0 && s >= 1 && s <= 6 && (ldo & 1) == 0 && a16(x) && a16(out) &&
          g.nzl >= 1 && g.nx + 64 < (i64(1) << 31) && g.ny + 64 < (i64(1) << 31) && g.nz + 16 < (i64(1) << 31)))
        return false;
    // The size heuristic is the caller's (Operator::mpk): on one rank the
    // kernel is slower than s separate stencil3d_vec launches (4.4 vs 3.5 ms
    // of MPK per 256³ cycle — shared-memory traffic and latency bound it at
    // ~2 IPC, profiles/ncu_mpk3d_*r02.txt); with several ranks
    // its one s-plane halo exchange per block wins.
    return force;
}

void launch_mpk3d(cudaStream_t st, const StencilGeom& g, const double* x, const double* halo_lo,
                  const double* halo_hi, double* out, i64 ldo, int s, int64_t& launches) {
    const bool jacobi = g.jacobi != 0;
    const int h = (s + 1) & ~1;
    const i64 nwx = ceil_div(g.nx, 64 - 2 * h), nwy = ceil_div(g.ny, kMpk3Rows - 2 * s);
    const i64 sms = num_sms();
    // z-bands per tile: minimise rounds × (band + 2s) steps per CTA (one CTA per SM)
    i64 nzb = 1, best = -1;
    for (i64 b = 1; b <= std::max<i64>(1, g.nzl / s) && b <= 4096; ++b) {
        const i64 tasks = nwx * nwy * b, rounds = ceil_div(tasks, sms);
        const i64 cost = rounds * (ceil_div(g.nzl, b) + 2 * s);
        if (best < 0 || cost < best) {
            best = cost;
            nzb = b;
        }
    }
    const i64 band = ceil_div(g.nzl, nzb);
    nzb = ceil_div(g.nzl, band);
    const i64 ntasks = nwx * nwy * nzb;
    if (ntasks >= (i64(1) << 31)) fail(KRY_UNSUPPORTED, "mpk3d: too many tiles");
    const size_t smem = static_cast<size_t>(2 * s) * kMpk3Pad * 32 * sizeof(double2);
    const unsigned grid = static_cast<unsigned>(std::min<i64>(ntasks, sms));
    auto go = [&](auto kernel) {
        set_kernel_smem(reinterpret_cast<const void*>(kernel), smem);
        launch_pdl(kernel, grid, kMpk3Warps * 32, smem, st, g, x, halo_lo, halo_hi, out, ldo, static_cast<int>(nwx),
                   static_cast<int>(nwy), static_cast<int>(band), static_cast<int>(ntasks));
    };
#define KB_MPK3(SV)                                           \
    case SV:                                                  \
        if (jacobi) go(mpk3d_kernel<SV, true>);               \
        else go(mpk3d_kernel<SV, false>);                     \
        break;
    switch (s) {
        KB_MPK3(1)
        KB_MPK3(2)
        KB_MPK3(3)
        KB_MPK3(4)
        KB_MPK3(5)
        KB_MPK3(6)
        default: fail(KRY_INTERNAL, "mpk3d: unsupported s");
    }
#undef KB_MPK3
    KB_LAUNCHED();
    ++launches;
}

int launch_csr(cudaStream_t s, i64 nloc, const int64_t* row_ptr, const int32_t* col, const double* vals,
               const double* x, const double* b, double* y, double* partials, int64_t& launches) {
    // warp-staged kernel: 32 rows per warp, grid-stride (fixed grid in residual mode)
    const i64 warps = ceil_div(nloc, 32);
    const int grid = b ? reduce_grid()
                       : static_cast<int>(std::max<i64>(1, std::min<i64>(ceil_div(warps, kBlock / 32), i64(1) << 30)));
    if (b)
        launch_pdl(csr_warp_kernel<CSR_ONLY, true, int64_t>, grid, kBlock, 0, s, nloc, row_ptr, col, vals, x, b, y, partials, nullptr);
    else
        launch_pdl(csr_warp_kernel<CSR_ONLY, false, int64_t>, grid, kBlock, 0, s, nloc, row_ptr, col, vals, x, b, y, partials, nullptr);
    KB_LAUNCHED();
    ++launches;
    return b ? grid : 0;
}

int launch_csr_sliced(cudaStream_t s, i64 nloc, int nslices, const int32_t* const* row_ptr,
                      const int32_t* const* col, const double* const* vals, const double* x, const double* b,
                      double* y, double* partials, double* part_sum, int64_t& launches) {
    const i64 warps = ceil_div(nloc, 32);
    const int grid_free =
        static_cast<int>(std::max<i64>(1, std::min<i64>(ceil_div(warps, kBlock / 32), i64(1) << 30)));
    for (int p = 0; p < nslices; ++p) {
        const bool first = p == 0, lastp = p == nslices - 1;
        const int grid = (b && lastp) ? reduce_grid() : grid_free;
        if (first)
            launch_pdl(csr_warp_kernel<CSR_FIRST, false, int32_t>, grid, kBlock, 0, s, nloc, row_ptr[p], col[p], vals[p], x, b, y, partials, part_sum);
        else if (!lastp)
            launch_pdl(csr_warp_kernel<CSR_MID, false, int32_t>, grid, kBlock, 0, s, nloc, row_ptr[p], col[p], vals[p], x, b, y, partials, part_sum);
        else if (b)
            launch_pdl(csr_warp_kernel<CSR_LAST, true, int32_t>, grid, kBlock, 0, s, nloc, row_ptr[p], col[p], vals[p], x, b, y, partials, part_sum);
        else
            launch_pdl(csr_warp_kernel<CSR_LAST, false, int32_t>, grid, kBlock, 0, s, nloc, row_ptr[p], col[p], vals[p], x, b, y, partials, part_sum);
        KB_LAUNCHED();
        ++launches;
    }
    return b ? reduce_grid() : 0;
}

void launch_finalize_sum(cudaStream_t s, const double* partials, int count, double* out,
                         int64_t& launches) {
    launch_pdl(finalize_kernel, 1, kBlock, 0, s, partials, count, out);
    KB_LAUNCHED();
    ++launches;
}

void launch_scale_div(cudaStream_t s, i64 n, const double* r, double gamma, double* out,
                      int64_t& launches) {
    launch_pdl(scale_div_kernel, grid_for(n), kBlock, 0, s, n, r, gamma, out);
    KB_LAUNCHED();
    ++launches;
}

void launch_xupdate(cudaStream_t s, i64 n, const double* x, const double* Q, i64 ldq, int k,
                    const Coef64& y, double* xnew, int64_t& launches) {
    launch_pdl(xupdate_kernel, grid_for(n), kBlock, 0, s, n, x, Q, ldq, k, y, xnew);
    KB_LAUNCHED();
    ++launches;
}

// ---- Jacobi (left diagonal scaling) ------------------------------
// D⁻¹A is formed once on the device, in place over the operator's values
// (every entry divided by its row's diagonal, an IEEE division: bit for bit
// what a host pre-scaling a_ij / a_ii gives the reference); D⁻¹b per solve.
namespace {
template <typename RP>
__global__ void __launch_bounds__(kBlock) csr_find_diag_kernel(i64 nloc, const RP* __restrict__ rp,
                                                               const int32_t* __restrict__ col,
                                                               const double* __restrict__ vals, i64 diag_col0,
                                                               double* __restrict__ d) {
    KB_PDL_WAIT();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nloc; i += (i64)gridDim.x * blockDim.x) {
        const i64 dc = diag_col0 + i;
        for (i64 k = rp[i]; k < static_cast<i64>(rp[i + 1]); ++k)
            if (col[k] == dc) d[i] = vals[k];
    }
}

template <typename RP>
__global__ void __launch_bounds__(kBlock) csr_scale_rows_kernel(i64 nloc, const RP* __restrict__ rp,
                                                                double* __restrict__ vals,
                                                                const double* __restrict__ d) {
    KB_PDL_WAIT();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nloc; i += (i64)gridDim.x * blockDim.x) {
        const double di = d[i];
        for (i64 k = rp[i]; k < static_cast<i64>(rp[i + 1]); ++k) vals[k] = __ddiv_rn(vals[k], di);
    }
}

__global__ void __launch_bounds__(kBlock) count_zero_kernel(i64 n, const double* __restrict__ d,
                                                            unsigned long long* __restrict__ zeros) {
    KB_PDL_WAIT();
    unsigned long long c = 0;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        c += (d[i] == 0.0 || !(d[i] == d[i])) ? 1ull : 0ull;
    if (c) atomicAdd(zeros, c);
}

__global__ void __launch_bounds__(kBlock) div_diag_kernel(i64 n, const double* __restrict__ b,
                                                          const double* __restrict__ d, double dconst,
                                                          double* __restrict__ out) {
    KB_PDL_WAIT();
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = __ddiv_rn(b[i], d ? d[i] : dconst);
}
}  // namespace

void launch_csr_find_diag(cudaStream_t s, i64 nloc, const int64_t* rp64, const int32_t* rp32, const int32_t* col,
                          const double* vals, i64 diag_col0, double* d, int64_t& launches) {
    const int grid = grid_for(nloc);
    if (rp64)
        launch_pdl(csr_find_diag_kernel<int64_t>, grid, kBlock, 0, s, nloc, rp64, col, vals, diag_col0, d);
    else
        launch_pdl(csr_find_diag_kernel<int32_t>, grid, kBlock, 0, s, nloc, rp32, col, vals, diag_col0, d);
    KB_LAUNCHED();
    ++launches;
}

void launch_csr_scale_rows(cudaStream_t s, i64 nloc, const int64_t* rp64, const int32_t* rp32, double* vals,
                           const double* d, int64_t& launches) {
    const int grid = grid_for(nloc);
    if (rp64)
        launch_pdl(csr_scale_rows_kernel<int64_t>, grid, kBlock, 0, s, nloc, rp64, vals, d);
    else
        launch_pdl(csr_scale_rows_kernel<int32_t>, grid, kBlock, 0, s, nloc, rp32, vals, d);
    KB_LAUNCHED();
    ++launches;
}

void launch_count_zero(cudaStream_t s, i64 n, const double* d, unsigned long long* zeros, int64_t& launches) {
    launch_pdl(count_zero_kernel, grid_for(n), kBlock, 0, s, n, d, zeros);
    KB_LAUNCHED();
    ++launches;
}

void launch_div_diag(cudaStream_t s, i64 n, const double* b, const double* d, double dconst, double* out,
                     int64_t& launches) {
    launch_pdl(div_diag_kernel, grid_for(n), kBlock, 0, s, n, b, d, dconst, out);
    KB_LAUNCHED();
    ++launches;
}

}  // namespace kb
