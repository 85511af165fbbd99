// Drop-in check for C++ callers: scenarios from the reference's own tests
// (tests/test_block_ortho.cpp) and its CLI solve path, written against
// krylov_b200:: exactly as they are written against krylov:: — only the
// include and the namespace differ.  Exit code 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <random>
#include <tuple>
#include <vector>

#include "krylov_b200/krylov.hpp"

using namespace krylov_b200;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond)                                                           \
    do {                                                                       \
        if (cond) {                                                            \
            ++g_pass;                                                          \
        } else {                                                               \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)

// gen_laplace2d(nx, ny, 5) (matgen.hpp:134-164) as a CSR, ascending columns.
static CsrMatrix laplace2d(index_t nx, index_t ny) {
    CsrMatrix a;
    a.n = nx * ny;
    a.row_ptr.push_back(0);
    for (index_t iy = 0; iy < ny; ++iy)
        for (index_t ix = 0; ix < nx; ++ix) {
            const index_t row = iy * nx + ix;
            auto put = [&](index_t c, double v) {
                a.col_idx.push_back(c);
                a.vals.push_back(v);
            };
            if (iy > 0) put(row - nx, -1.0);
            if (ix > 0) put(row - 1, -1.0);
            put(row, 4.0);
            if (ix + 1 < nx) put(row + 1, -1.0);
            if (iy + 1 < ny) put(row + nx, -1.0);
            a.row_ptr.push_back(a.col_idx.size());
        }
    return a;
}

static DenseMatrix random_matrix(index_t rows, index_t cols, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist;
    DenseMatrix m(rows, cols);
    for (index_t j = 0; j < cols; ++j)
        for (index_t i = 0; i < rows; ++i) m(i, j) = dist(rng);
    return m;
}

int main() {
    // BcgsPip.EmptyPrefixIsCholQrBitwise (tests/test_block_ortho.cpp:172-181)
    {
        DenseMatrix v = random_matrix(120, 5, 13);
        SyncCounter s1, s2;
        BlockOrthoResult pip = bcgs_pip(ConstMatrixView(), v, s1);
        BlockQr chol = cholqr(v, s2);
        double d = 0.0;
        for (index_t j = 0; j < 5; ++j)
            for (index_t i = 0; i < 120; ++i) d = std::max(d, std::abs(pip.q(i, j) - chol.q(i, j)));
        EXPECT(d == 0.0);
        EXPECT(s1.reduces == 1);
    }
    // NotPositiveDefinite carries the 1-based pivot (types.hpp:20-27)
    {
        DenseMatrix v = random_matrix(300, 4, 3);
        for (index_t i = 0; i < 300; ++i) v(i, 2) = 0.0;
        SyncCounter s;
        bool thrown = false;
        try {
            bcgs_pip(ConstMatrixView(), v, s);
        } catch (const NotPositiveDefinite& e) {
            thrown = (e.pivot == 3);
        }
        EXPECT(thrown);
    }
    // BasisStore.RawSequenceReconstruction (tests/test_block_ortho.cpp:331-380)
    {
        const index_t grid = 12, m = 12, s = 3;
        CsrMatrix a = laplace2d(grid, grid);
        const index_t n = a.n;
        std::vector<double> ones(n, 1.0);
        std::vector<double> b = spmv(a, ones);
        double gamma = 0.0;
        for (double x : b) gamma += x * x;
        gamma = std::sqrt(gamma);
        std::vector<double> v1(b);
        for (double& x : v1) x /= gamma;
        for (OrthoKind kind : {OrthoKind::BcgsPip2, OrthoKind::Bcgs2Cholqr2, OrthoKind::TwoStage}) {
            BasisStore store(n, m, s, m);
            SyncCounter sync;
            OrthoScheme scheme{kind, m};
            DenseMatrix raw(n, m + 1);
            index_t raw_cols = 0;
            for (index_t j = 0; j < m / s; ++j) {
                std::vector<double> start = (j == 0) ? v1 : store.column(store.filled() - 1);
                DenseMatrix blk = mpk_monomial(a, start, s);
                for (index_t c = (j == 0) ? 0 : 1; c <= s; ++c) raw.set_col(raw_cols++, blk.col(c));
                AppendOutcome oc = (kind == OrthoKind::TwoStage) ? store.preprocess_block(blk, j != 0, sync)
                                                                 : store.append_block(blk, j != 0, scheme, sync);
                EXPECT(!oc.breakdown);
            }
            if (kind == OrthoKind::TwoStage) store.finalize_big_panel(sync);
            EXPECT(raw_cols == store.filled());
            UpperTriangular r = store.coefficients();
            DenseMatrix q = store.all();
            double dev = 0.0, scale = 0.0;
            for (index_t c = 0; c < raw_cols; ++c)
                for (index_t i = 0; i < n; ++i) {
                    double rec = 0.0;
                    for (index_t l = 0; l <= c; ++l) rec += r(l, c) * q(i, l);
                    dev += (rec - raw(i, c)) * (rec - raw(i, c));
                    scale += raw(i, c) * raw(i, c);
                }
            EXPECT(std::sqrt(dev) <= 1e-12 * std::sqrt(scale));
            for (index_t c = 0; c < raw_cols; ++c) EXPECT(r(c, c) >= 0.0);
        }
    }
    // The CLI solve path (tools/krylov_main.cpp:220-229): two-stage ŝ = 60 on 100²,
    // SURVEY §8(c) anchors 300 iterations / 4 restarts / 65 reduces.
    {
        CsrMatrix a = laplace2d(100, 100);
        std::vector<double> ones(a.n, 1.0);
        std::vector<double> b = spmv(a, ones);
        SolverConfig cfg;
        cfg.scheme = OrthoScheme{OrthoKind::TwoStage, 60};
        SolveReport rep = sstep_gmres(a, b, {}, cfg);
        EXPECT(rep.status == SolveStatus::Converged);
        EXPECT(rep.iterations == 300 && rep.restarts == 4 && rep.sync.reduces == 65);
        EXPECT(rep.final_relative_residual <= 1e-6);
        cfg.scheme = OrthoScheme{OrthoKind::BcgsPip2, 0};
        rep = sstep_gmres(Operator::laplace2d(100, 100), b, {}, cfg);  // matrix-free operator, same answer
        EXPECT(rep.iterations == 270 && rep.restarts == 4 && rep.sync.reduces == 108);
        rep = standard_gmres(laplace2d(32, 32), spmv(laplace2d(32, 32), std::vector<double>(1024, 1.0)), {},
                             SolverConfig{});
        EXPECT(rep.status == SolveStatus::Converged);
    }
    std::printf("dropin_test: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
