// Device helpers shared by the sm_100a kernels (include from .cu only):
// mbarrier / TMA / DMMA wrappers and the K5 row update (k_tsqr.cu), reused
// by the fused first-stage pass (k_fused.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "kb_common.hpp"

// First statement of every kernel: with programmatic dependent launch (below)
// a kernel may start while its predecessor in the stream drains; it waits
// here until that predecessor has completed and its writes are visible
// (a no-op for a normally launched kernel).  Before any early return, so a
// kernel never completes ahead of its predecessor.
#define KB_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

namespace kb {

// Kernel launch with programmatic dependent launch (PDL): the next kernel's
// launch and CTA rasterisation overlap the previous kernel's tail.  Every
// kernel of the library begins with KB_PDL_WAIT(), so stream order is kept.
// KRY_PDL=0 launches normally (A/B).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KRY_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}
inline cudaLaunchConfig_t pdl_config(dim3 grid, dim3 block, size_t smem, cudaStream_t s, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    if (launches_suppressed()) return;
    cudaLaunchAttribute at[1];
    const cudaLaunchConfig_t cfg = pdl_config(grid, block, smem, s, at);
    KB_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
inline void launch_pdl_c(const void* kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, void** args) {
    if (launches_suppressed()) return;
    cudaLaunchAttribute at[1];
    const cudaLaunchConfig_t cfg = pdl_config(grid, block, smem, s, at);
    KB_CUDA(cudaLaunchKernelExC(&cfg, kernel, args));
}

namespace dev {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "KB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra KB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// ---- thread-block clusters (DSMEM, cross-CTA mbarriers) --------------------
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// This CTA's shared address `p` mapped into CTA `cta` of the cluster.
__device__ __forceinline__ unsigned cluster_map(const void* p, unsigned cta) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
    return r;
}
// Arrive on the barrier at `bar`'s offset in CTA `cta` (release at cluster
// scope: this thread's earlier writes — shared, DSMEM or global — are
// visible to a thread that then completes the phase wait with acquire.cluster).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, unsigned cta) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_map(bar, cta))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "KB_CWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra KB_CWAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_cluster_f64x2(const void* p, unsigned cta, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(cluster_map(p, cta)), "d"(v.x), "d"(v.y)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// K5 row update: (V − P·R_col)·R_jj⁻¹ for rows [row, row + R), row-local,
// in the order of bcgs_pip_partial's update + tri_solve_right
// (block_ortho.hpp:171-176, dense_kernels.hpp:139-154).
// coef layout (doubles): nrc[cpp][WMAX] = −R_col (rows cp..cpp zero),
// nrjj[WMAX][WMAX] = −R_jj(l,j) for l < j, inv[WMAX] = 1/R_jj(j,j).
// ---------------------------------------------------------------------------
// R rows per thread (R = 2: 16-byte loads/stores of two adjacent rows —
// half the load instructions and coefficient broadcasts per element).
template <int R>
struct RowVec;
template <>
struct RowVec<1> {
    static __device__ __forceinline__ void ld(const double* p, double (&d)[1]) { d[0] = __ldg(p); }
    static __device__ __forceinline__ void ldv(const double* p, double (&d)[1]) { d[0] = *p; }
    static __device__ __forceinline__ void st(double* p, const double (&d)[1]) { *p = d[0]; }
};
template <>
struct RowVec<2> {
    static __device__ __forceinline__ void ld(const double* p, double (&d)[2]) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        d[0] = t.x;
        d[1] = t.y;
    }
    static __device__ __forceinline__ void ldv(const double* p, double (&d)[2]) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        d[0] = t.x;
        d[1] = t.y;
    }
    static __device__ __forceinline__ void st(double* p, const double (&d)[2]) {
        *reinterpret_cast<double2*>(p) = make_double2(d[0], d[1]);
    }
};

// Right-looking substitution of one row group against R_jj (acc_j receives
// −R(k,j)·x_k for k = 0, 1, … in order, then ×1/R(j,j) — tri_solve_right's
// order), shared by K5/K5t and the fused pass K6.
template <int WMAX, int R>
__device__ __forceinline__ void update_tri(double (&acc)[WMAX][R], const double* nrjj, const double* inv) {
#pragma unroll
    for (int k = 0; k < WMAX; ++k) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[k][r] *= inv[k];
        const double* rk = nrjj + k * WMAX;
        if ((k + 1) & 1) {  // odd first column: one scalar step to reach a pair boundary
            if (k + 1 < WMAX)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[k + 1][r] = fma(rk[k + 1], acc[k][r], acc[k + 1][r]);
        }
#pragma unroll
        for (int j = (k + 2) & ~1; j < WMAX; j += 2) {
            const double2 c = *reinterpret_cast<const double2*>(rk + j);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                acc[j][r] = fma(c.x, acc[k][r], acc[j][r]);
                acc[j + 1][r] = fma(c.y, acc[k][r], acc[j + 1][r]);
            }
        }
    }
}

// Rows [row, row + R) of the update (every row computed in exactly the
// scalar order, so R = 1 and R = 2 give identical bits).
template <int WMAX, int R>
__device__ __forceinline__ void update_acc(i64 row, const double* __restrict__ P, i64 ldp, int cp, int cpp,
                                           const double* V, i64 ldv, int w, const double* nrc,
                                           const double* nrjj, const double* inv, int triangular,
                                           double (&acc)[WMAX][R]) {
    using RV = RowVec<R>;
#pragma unroll
    for (int j = 0; j < WMAX; ++j) {
        if (j < w) {
            RV::ldv(V + row + j * ldv, acc[j]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[j][r] = 0.0;
        }
    }
    // Prefix columns in batches of 4 through a 3-deep register ring: two
    // batches are in flight while one is consumed.  The coefficient rows are
    // zero-padded to a multiple of 12 (see the shared-memory fill), so there
    // is no tail loop; loads past cp are predicated off.
    const double* prow = P + row;
    const int nb = cpp / 4;
    double b0[4][R], b1[4][R], b2[4][R];
    auto ld = [&](double (&dst)[4][R], int bt) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int l = 4 * bt + u;
            if (l < cp) {
                RV::ld(prow + static_cast<i64>(l) * ldp, dst[u]);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) dst[u][r] = 0.0;
            }
        }
    };
    auto fm = [&](const double (&src)[4][R], int bt) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2* cr = reinterpret_cast<const double2*>(nrc + (4 * bt + u) * WMAX);
#pragma unroll
            for (int j = 0; j < WMAX; j += 2) {
                const double2 c = cr[j / 2];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc[j][r] = fma(c.x, src[u][r], acc[j][r]);
                    acc[j + 1][r] = fma(c.y, src[u][r], acc[j + 1][r]);
                }
            }
        }
    };
    if (nb > 0) {
        ld(b0, 0);
        ld(b1, 1);
    }
    for (int bt = 0; bt < nb; bt += 3) {  // nb is a multiple of 3
        ld(b2, bt + 2);
        fm(b0, bt);
        ld(b0, bt + 3);
        fm(b1, bt + 1);
        ld(b1, bt + 4);
        fm(b2, bt + 2);
    }
    if (triangular) update_tri<WMAX, R>(acc, nrjj, inv);
}

template <int WMAX, int R>
__device__ __forceinline__ void update_rows(i64 row, const double* __restrict__ P, i64 ldp, int cp, int cpp,
                                            const double* V, i64 ldv, int w, const double* nrc,
                                            const double* nrjj, const double* inv, int triangular, double* out,
                                            i64 ldo) {
    double acc[WMAX][R];
    update_acc<WMAX, R>(row, P, ldp, cp, cpp, V, ldv, w, nrc, nrjj, inv, triangular, acc);
#pragma unroll
    for (int j = 0; j < WMAX; ++j)
        if (j < w) RowVec<R>::st(out + row + j * ldo, acc[j]);
}

// 2-D tensor map over a column-major (ld) matrix, box box_rows × box_cols
// (k_tsqr.cu, cached).  l2_promote: 256-byte L2 promotion (whole aligned
// runs); off for boxes whose rows start at arbitrary offsets.
CUtensorMap tensor_map_2d(const double* base, i64 ld, i64 rows, i64 cols, int box_rows, int box_cols,
                          bool l2_promote = true);

}  // namespace dev
}  // namespace kb
