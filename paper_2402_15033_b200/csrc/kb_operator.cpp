#include "kb_operator.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <vector>

namespace kb {

#define KB_NCCL(expr)                                                                      \
    do {                                                                                   \
        ncclResult_t kb_r_ = (expr);                                                       \
        if (kb_r_ != ncclSuccess)                                                          \
            ::kb::fail(KRY_NCCL_ERROR, std::string(#expr) + ": " + ncclGetErrorString(kb_r_)); \
    } while (0)

void laplace_partition(int dims, i64 nx, i64 ny, i64 nz, int nranks, int rank, i64& row_begin, i64& nloc,
                       i64& halo) {
    // 1D block-row partition by whole grid lines / planes:
    // rank r owns lines [r·L/P, (r+1)·L/P); the halo is one line / plane.
    const i64 lines = dims == 2 ? ny : nz;
    const i64 plane = dims == 2 ? nx : nx * ny;
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(KRY_INVALID_ARGUMENT, "bad rank layout");
    if (lines < nranks) fail(KRY_INVALID_ARGUMENT, "fewer grid lines than ranks");
    const i64 l0 = rank * lines / nranks, l1 = (rank + 1) * lines / nranks;
    row_begin = l0 * plane;
    nloc = (l1 - l0) * plane;
    halo = nranks > 1 ? plane : 0;
}

Operator* make_laplace(Ctx& ctx, int dims, i64 nx, i64 ny, i64 nz) {
    if (dims == 2) {
        if (nx < 2 || ny < 2) fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: gen_laplace2d needs dimensions >= 2");
    } else {
        if (nx < 2 || ny < 2 || nz < 2)
            fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: gen_laplace3d needs dimensions >= 2");
    }
    auto* op = new Operator;
    op->ctx = &ctx;
    op->kind = dims == 2 ? Operator::LAPLACE2D : Operator::LAPLACE3D;
    i64 halo = 0;
    try {
        laplace_partition(dims, nx, ny, nz, ctx.nranks, ctx.rank, op->row_begin, op->nloc, halo);
    } catch (...) {
        delete op;
        throw;
    }
    op->n_global = dims == 2 ? nx * ny : nx * ny * nz;
    op->nnz_local = 0;
    op->geom = make_stencil_geom(dims, nx, ny, nz, op->row_begin, op->nloc);
    if (ctx.nranks > 1) {
        op->halo_lo.ensure(static_cast<size_t>(halo) * 8);
        op->halo_hi.ensure(static_cast<size_t>(halo) * 8);
    }
    op->partials.ensure(static_cast<size_t>(stencil_partials(op->geom) + 64) * 8);
    return op;
}

Operator* make_csr(Ctx& ctx, i64 n_global, i64 row_begin, i64 nloc, const int64_t* rp, const int64_t* ci,
                   const double* v) {
    // CsrMatrix::validate (csr_matrix.hpp:25-38), restricted to the local rows.
    dim_check(nloc >= 0 && row_begin >= 0 && row_begin + nloc <= n_global, "csr row range");
    dim_check(rp[0] == 0, "row_ptr bounds");
    for (i64 i = 0; i < nloc; ++i) {
        dim_check(rp[i] <= rp[i + 1], "row_ptr not monotone");
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            dim_check(ci[k] >= 0 && ci[k] < n_global, "column index out of range");
            dim_check(k == rp[i] || ci[k] > ci[k - 1], "column indices not strictly increasing");
        }
    }
    auto* op = new Operator;
    op->ctx = &ctx;
    op->kind = Operator::CSR;
    op->n_global = n_global;
    op->row_begin = row_begin;
    op->nloc = nloc;
    op->nnz_local = rp[nloc];

    // Rank layout (row_begin, nloc of every rank) for the x gather.
    std::vector<int64_t> layout(2 * ctx.nranks, 0);
    layout[2 * ctx.rank] = row_begin;
    layout[2 * ctx.rank + 1] = nloc;
    if (ctx.nranks > 1) {
        DevBuf d;
        d.ensure(layout.size() * 8);
        KB_CUDA(cudaMemcpyAsync(d.as<int64_t>() + 2 * ctx.rank, layout.data() + 2 * ctx.rank, 16,
                                cudaMemcpyHostToDevice, ctx.stream));
        KB_NCCL(ncclAllGather(d.as<int64_t>() + 2 * ctx.rank, d.as<int64_t>(), 2, ncclInt64, ctx.comm,
                              ctx.stream));
        KB_CUDA(cudaMemcpyAsync(layout.data(), d.p, layout.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
    }
    i64 max_rows = 0;
    for (int r = 0; r < ctx.nranks; ++r) max_rows = std::max<i64>(max_rows, layout[2 * r + 1]);
    op->max_rows = max_rows;
    if (static_cast<double>(max_rows) * ctx.nranks >= static_cast<double>(std::numeric_limits<int32_t>::max())) {
        delete op;
        fail(KRY_UNSUPPORTED, "CSR gather index exceeds int32");
    }
    std::vector<int32_t> col(static_cast<size_t>(op->nnz_local));
    for (i64 k = 0; k < op->nnz_local; ++k) {
        const i64 g = ci[k];
        if (ctx.nranks == 1) {
            col[k] = static_cast<int32_t>(g);
            continue;
        }
        int owner = -1;
        for (int r = 0; r < ctx.nranks; ++r)
            if (g >= layout[2 * r] && g < layout[2 * r] + layout[2 * r + 1]) { owner = r; break; }
        if (owner < 0) {
            delete op;
            fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: column not owned by any rank");
        }
        col[k] = static_cast<int32_t>(owner * max_rows + (g - layout[2 * owner]));
    }
    op->row_ptr.ensure(static_cast<size_t>(nloc + 1) * 8);
    op->col.ensure(std::max<size_t>(col.size(), 1) * 4);
    op->vals.ensure(std::max<size_t>(static_cast<size_t>(op->nnz_local), 1) * 8);
    KB_CUDA(cudaMemcpyAsync(op->row_ptr.p, rp, static_cast<size_t>(nloc + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (!col.empty()) {
        KB_CUDA(cudaMemcpyAsync(op->col.p, col.data(), col.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
        KB_CUDA(cudaMemcpyAsync(op->vals.p, v, static_cast<size_t>(op->nnz_local) * 8, cudaMemcpyHostToDevice,
                                ctx.stream));
    }
    if (ctx.nranks > 1) {
        op->xfull.ensure(static_cast<size_t>(max_rows * ctx.nranks) * 8);
        op->xsend.ensure(static_cast<size_t>(std::max<i64>(max_rows, 1)) * 8);
    }
    op->partials.ensure(static_cast<size_t>(reduce_grid() + 64) * 8);
    ctx.sync();  // host vectors above go out of scope

    // Column slicing (see kb_operator.hpp): x of nx_total doubles is cut
    // into ranges of about KRY_CSR_SLICE_MB (default 56 MB, inside the
    // 126 MB L2 next to the streamed matrix; 3 slices at n = 20 M measured
    // best: 2 → 207, 3 → 194, 4 → 198, 6 → 211 ms of MPK per cycle);
    // KRY_CSR_SLICES forces a count.
    const i64 nx_total = ctx.nranks > 1 ? max_rows * ctx.nranks : n_global;
    double slice_mb = 56.0;
    if (const char* e = std::getenv("KRY_CSR_SLICE_MB")) slice_mb = std::max(1.0, std::atof(e));
    i64 ns = static_cast<i64>(std::ceil(8.0 * nx_total / (slice_mb * 1048576.0)));
    if (const char* e = std::getenv("KRY_CSR_SLICES")) ns = std::atoi(e);
    ns = std::max<i64>(1, std::min<i64>(ns, 16));
    if (ns >= 2 && op->nnz_local > 0 && op->nnz_local < (i64(1) << 31)) {
        std::vector<i64> bound(static_cast<size_t>(ns + 1));
        for (i64 p = 0; p <= ns; ++p) bound[p] = (p * nx_total + ns - 1) / ns;
        std::vector<std::vector<int32_t>> rps(static_cast<size_t>(ns), std::vector<int32_t>(nloc + 1, 0));
        // count per row per slice (columns ascend within a row, so each
        // slice is a contiguous run of the row's stored entries)
        for (i64 i = 0; i < nloc; ++i) {
            i64 p = 0;
            for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
                while (col[k] >= bound[p + 1]) ++p;
                ++rps[p][i + 1];
            }
        }
        op->s_row_ptr.resize(ns);
        op->s_col.resize(ns);
        op->s_vals.resize(ns);
        for (i64 p = 0; p < ns; ++p) {
            std::vector<int32_t>& r = rps[p];
            for (i64 i = 0; i < nloc; ++i) r[i + 1] += r[i];
            const i64 cnt = r[nloc];
            std::vector<int32_t> c(static_cast<size_t>(std::max<i64>(cnt, 1)));
            std::vector<double> vv(static_cast<size_t>(std::max<i64>(cnt, 1)));
            for (i64 i = 0; i < nloc; ++i) {
                i64 o = r[i];
                for (i64 k = rp[i]; k < rp[i + 1]; ++k)
                    if (col[k] >= bound[p] && col[k] < bound[p + 1]) {
                        c[o] = col[k];
                        vv[o] = v[k];
                        ++o;
                    }
            }
            op->s_row_ptr[p].ensure(static_cast<size_t>(nloc + 1) * 4);
            op->s_col[p].ensure(c.size() * 4);
            op->s_vals[p].ensure(vv.size() * 8);
            KB_CUDA(cudaMemcpy(op->s_row_ptr[p].p, r.data(), static_cast<size_t>(nloc + 1) * 4,
                               cudaMemcpyHostToDevice));
            KB_CUDA(cudaMemcpy(op->s_col[p].p, c.data(), c.size() * 4, cudaMemcpyHostToDevice));
            KB_CUDA(cudaMemcpy(op->s_vals[p].p, vv.data(), vv.size() * 8, cudaMemcpyHostToDevice));
        }
        op->part_sum.ensure(static_cast<size_t>(std::max<i64>(nloc, 1)) * 8);
        op->nslices = static_cast<int>(ns);
        // the unsliced copy is no longer needed
        op->col.release();
        op->vals.release();
    }
    return op;
}

int Operator::apply(const double* x, double* y, const double* b) {
    Ctx& c = *ctx;
    double* part = partials.p;
    if (kind == CSR) {
        const double* xs = x;
        if (c.nranks > 1) {
            KB_CUDA(cudaMemcpyAsync(xsend.p, x, static_cast<size_t>(nloc) * 8, cudaMemcpyDeviceToDevice, c.stream));
            KB_NCCL(ncclAllGather(xsend.p, xfull.p, static_cast<size_t>(max_rows), ncclDouble, c.comm, c.stream));
            xs = xfull.p;
        }
        if (nslices >= 2) {
            std::vector<const int32_t*> rp(nslices), cl(nslices);
            std::vector<const double*> vl(nslices);
            for (int p = 0; p < nslices; ++p) {
                rp[p] = s_row_ptr[p].as<int32_t>();
                cl[p] = s_col[p].as<int32_t>();
                vl[p] = s_vals[p].p;
            }
            return launch_csr_sliced(c.stream, nloc, nslices, rp.data(), cl.data(), vl.data(), xs, b, y, part,
                                     part_sum.p, c.launches);
        }
        return launch_csr(c.stream, nloc, row_ptr.as<int64_t>(), col.as<int32_t>(), vals.p, xs, b, y, part,
                          c.launches);
    }
    if (c.nranks > 1) {
        const i64 h = geom.halo;
        KB_NCCL(ncclGroupStart());
        if (c.rank > 0) {
            KB_NCCL(ncclSend(x, static_cast<size_t>(h), ncclDouble, c.rank - 1, c.comm, c.stream));
            KB_NCCL(ncclRecv(halo_lo.p, static_cast<size_t>(h), ncclDouble, c.rank - 1, c.comm, c.stream));
        }
        if (c.rank + 1 < c.nranks) {
            KB_NCCL(ncclSend(x + nloc - h, static_cast<size_t>(h), ncclDouble, c.rank + 1, c.comm, c.stream));
            KB_NCCL(ncclRecv(halo_hi.p, static_cast<size_t>(h), ncclDouble, c.rank + 1, c.comm, c.stream));
        }
        KB_NCCL(ncclGroupEnd());
    }
    return launch_stencil(c.stream, geom, x, halo_lo.p, halo_hi.p, b, y, part, c.launches);
}

bool Operator::mpk(const double* x, double* out, i64 ldo, int s) {
    // KRY_FUSED_MPK: 0 = never, 1 (default) = when the grid is large enough
    // to fill the GPU with wavefront tasks, 2 = whenever supported (tests).
    const char* e = std::getenv("KRY_FUSED_MPK");
    const int mode = e ? std::atoi(e) : 1;
    Ctx& c = *ctx;
    if (mode == 0 || kind == CSR) return false;
    // Every rank must own at least s lines / planes (the halo is the
    // neighbour's s edge lines / planes); the partition differs by at most
    // one line / plane between ranks.  The choice pairs every rank's sends
    // with its neighbours' receives, so it must be the same on every rank:
    // the size heuristic is judged on the smallest rank's share (known to
    // all ranks), not on this rank's own.  The other inputs (s, the grid,
    // the store's even ld, 256-byte aligned allocations) are identical on
    // every rank.
    StencilGeom uniform = geom;
    i64 plane = geom.nx;
    if (kind == LAPLACE2D) {
        uniform.lines = geom.ny / c.nranks;
        if (uniform.lines < s || !mpk2d_supported(uniform, s, x, out, ldo, mode == 2)) return false;
    } else {
        uniform.nzl = geom.nz / c.nranks;
        plane = geom.nx * geom.ny;
        // One rank: s per-SpMV launches are faster than the one-pass kernel
        // (3.50 vs 4.37 ms of MPK per 256³ cycle).  Several ranks: its single
        // s-plane exchange per block beats s one-plane exchanges (256³:
        // 2.49 vs 2.91 ms at N = 2, 1.65 vs 2.72 ms at N = 4).
        if (!(mode == 2 || c.nranks > 1)) return false;
        if (uniform.nzl < s || !mpk3d_supported(uniform, s, x, out, ldo, true)) return false;
    }
    const i64 h = static_cast<i64>(s) * plane;
    if (c.nranks > 1) {
        mpk_lo.ensure(static_cast<size_t>(h) * 8);
        mpk_hi.ensure(static_cast<size_t>(h) * 8);
        KB_NCCL(ncclGroupStart());
        if (c.rank > 0) {
            KB_NCCL(ncclSend(x, static_cast<size_t>(h), ncclDouble, c.rank - 1, c.comm, c.stream));
            KB_NCCL(ncclRecv(mpk_lo.p, static_cast<size_t>(h), ncclDouble, c.rank - 1, c.comm, c.stream));
        }
        if (c.rank + 1 < c.nranks) {
            KB_NCCL(ncclSend(x + nloc - h, static_cast<size_t>(h), ncclDouble, c.rank + 1, c.comm, c.stream));
            KB_NCCL(ncclRecv(mpk_hi.p, static_cast<size_t>(h), ncclDouble, c.rank + 1, c.comm, c.stream));
        }
        KB_NCCL(ncclGroupEnd());
    }
    if (kind == LAPLACE2D)
        launch_mpk2d(c.stream, geom, x, mpk_lo.p, mpk_hi.p, out, ldo, s, c.launches);
    else
        launch_mpk3d(c.stream, geom, x, mpk_lo.p, mpk_hi.p, out, ldo, s, c.launches);
    return true;
}

void Operator::set_jacobi() {
    if (jacobi) return;
    Ctx& c = *ctx;
    if (kind != CSR) {
        // gen_laplace2d/3d: every row's diagonal is 4 / 6, so D⁻¹A is the
        // stencil with off-diagonal −1/d (rounded, as a_ij / a_ii is) and
        // diagonal 1 — applied inside the stencil and MPK kernels.
        const double d = kind == LAPLACE2D ? 4.0 : 6.0;
        geom.jacobi = 1;
        geom.c_off = -1.0 / d;
        jacobi = true;
        return;
    }
    diag.ensure(static_cast<size_t>(std::max<i64>(nloc, 1)) * 8);
    KB_CUDA(cudaMemsetAsync(diag.p, 0, static_cast<size_t>(std::max<i64>(nloc, 1)) * 8, c.stream));
    // the diagonal of local row i is gathered column (rank·max_rows + i)
    // with several ranks, global column row_begin + i with one
    const i64 dc0 = c.nranks > 1 ? static_cast<i64>(c.rank) * max_rows : row_begin;
    if (nslices >= 2) {
        for (int p = 0; p < nslices; ++p)
            launch_csr_find_diag(c.stream, nloc, nullptr, s_row_ptr[p].as<int32_t>(), s_col[p].as<int32_t>(),
                                 s_vals[p].p, dc0, diag.p, c.launches);
    } else {
        launch_csr_find_diag(c.stream, nloc, row_ptr.as<int64_t>(), nullptr, col.as<int32_t>(), vals.p, dc0, diag.p,
                             c.launches);
    }
    DevBuf cnt;
    cnt.ensure(8);
    KB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, c.stream));
    launch_count_zero(c.stream, nloc, diag.p, reinterpret_cast<unsigned long long*>(cnt.p), c.launches);
    unsigned long long zeros = 0;
    KB_CUDA(cudaMemcpyAsync(&zeros, cnt.p, 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (zeros) fail(KRY_INVALID_ARGUMENT, "Jacobi needs a nonzero diagonal entry in every row");
    if (nslices >= 2) {
        for (int p = 0; p < nslices; ++p)
            launch_csr_scale_rows(c.stream, nloc, nullptr, s_row_ptr[p].as<int32_t>(), s_vals[p].p, diag.p,
                                  c.launches);
    } else {
        launch_csr_scale_rows(c.stream, nloc, row_ptr.as<int64_t>(), nullptr, vals.p, diag.p, c.launches);
    }
    c.sync();
    jacobi = true;
}

const double* Operator::scaled_rhs(const double* b, DevBuf& buf) {
    if (!jacobi) return b;
    buf.ensure(static_cast<size_t>(std::max<i64>(nloc, 1)) * 8);
    if (kind == CSR)
        launch_div_diag(ctx->stream, nloc, b, diag.p, 0.0, buf.p, ctx->launches);
    else
        launch_div_diag(ctx->stream, nloc, b, nullptr, kind == LAPLACE2D ? 4.0 : 6.0, buf.p, ctx->launches);
    return buf.p;
}

double Operator::bytes_per_apply() const {
    if (kind == CSR) return 12.0 * nnz_local + 8.0 * (nloc + 1) + 16.0 * nloc;
    return 16.0 * nloc;
}

}  // namespace kb
