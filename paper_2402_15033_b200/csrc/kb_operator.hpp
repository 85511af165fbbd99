// Device operators: CSR (krylov::CsrMatrix, csr_matrix.hpp:17-65) and the
// matrix-free 5/7-point Laplacians that reproduce gen_laplace2d/3d
// (matgen.hpp:134-187).  Rows are partitioned contiguously across the
// context's ranks; apply() performs the halo exchange
// over NCCL send/recv (NVLink P2P) before the row kernel.
#pragma once

#include <vector>

#include "kb_ctx.hpp"
#include "kb_kernels.hpp"

namespace kb {

struct Operator {
    enum Kind { CSR = 0, LAPLACE2D = 1, LAPLACE3D = 2 };
    Ctx* ctx = nullptr;
    Kind kind = CSR;
    i64 n_global = 0, row_begin = 0, nloc = 0, nnz_local = 0;
    StencilGeom geom{};
    DevBuf halo_lo, halo_hi;  // stencil halos (geom.halo doubles each)
    // CSR
    DevBuf row_ptr, col, vals;
    DevBuf xfull, xsend;      // multi-rank gather of x
    // Column-sliced copy of the CSR (nslices ≥ 2 when the gathered x is
    // larger than the L2 share it should keep): one pass per column range,
    // each pass's x slice stays L2-resident (k_ops.cu launch_csr_sliced).
    int nslices = 1;
    std::vector<DevBuf> s_row_ptr, s_col, s_vals;
    DevBuf part_sum;          // running row sums between passes
    i64 max_rows = 0;
    DevBuf partials;          // Σr² partials of the residual mode

    // y = A·x (b == nullptr) or y = b − A·x with Σy² partials in `partials`;
    // returns the number of partials written (0 without b).
    int apply(const double* x, double* y, const double* b = nullptr);
    // The whole monomial MPK out[:, k−1] = A^k·x, k = 1..s, in one fused
    // pass when the operator supports it (2-D stencil); false otherwise
    // (the caller then applies s times).  Collective over the ranks.
    bool mpk(const double* x, double* out, i64 ldo, int s);
    DevBuf mpk_lo, mpk_hi;    // s-line halos of the fused MPK
    // bytes moved by one application (algorithmic)
    double bytes_per_apply() const;
    // Left Jacobi preconditioning: once set, the operator IS
    // D⁻¹A (CSR: the values divided by their row's diagonal in place on the
    // device), and solves scale b to D⁻¹b on the device (scaled_rhs).
    bool jacobi = false;
    DevBuf diag;              // CSR: a_ii per local row
    void set_jacobi();
    // D⁻¹b into buf (the caller's b when the operator is not preconditioned).
    const double* scaled_rhs(const double* b, DevBuf& buf);
};
void gen_random_sparse(i64 n_global, i64 row_begin, i64 n_local, i64 per_row, uint64_t seed, double diag_factor,
                       bool jacobi, int64_t* row_ptr, int64_t* col, double* vals);

void laplace_partition(int dims, i64 nx, i64 ny, i64 nz, int nranks, int rank, i64& row_begin, i64& nloc,
                       i64& halo);
Operator* make_laplace(Ctx& ctx, int dims, i64 nx, i64 ny, i64 nz);
Operator* make_csr(Ctx& ctx, i64 n_global, i64 row_begin, i64 nloc, const int64_t* row_ptr,
                   const int64_t* col_idx, const double* vals);

}  // namespace kb
