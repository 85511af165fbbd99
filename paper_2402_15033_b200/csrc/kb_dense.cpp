// Host-side small dense algebra; see kb_dense.hpp.  Compiled without FMA
// contraction (-ffp-contract=off) so that, fed the same numbers, these
// routines reproduce the reference's host arithmetic bit for bit.
#include "kb_dense.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

namespace kb {

double dot_seq(const double* a, const double* b, i64 n) {
    double s = 0.0;
    for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static void axpy_seq(double alpha, const double* x, double* y, i64 n) {
    for (i64 i = 0; i < n; ++i) y[i] += alpha * x[i];
}

i64 try_cholesky(const Mat& s, Upper& r) {
    dim_check(s.rows == s.cols, "cholesky needs a square matrix");
    const i64 n = s.rows;
    r = Upper(n);
    for (i64 j = 0; j < n; ++j) {
        for (i64 i = 0; i < j; ++i) {
            double acc = s(i, j);
            for (i64 k = 0; k < i; ++k) acc -= r(k, i) * r(k, j);
            r.at(i, j) = acc / r(i, i);
        }
        double d = s(j, j);
        for (i64 k = 0; k < j; ++k) d -= r(k, j) * r(k, j);
        if (!(d > 0.0)) return j + 1;
        r.at(j, j) = std::sqrt(d);
    }
    return 0;
}

Upper tri_mul(const Upper& a, const Upper& b) {
    dim_check(a.dim == b.dim, "tri_mul dimensions");
    const i64 n = a.dim;
    Upper c(n);
    for (i64 j = 0; j < n; ++j)
        for (i64 i = 0; i <= j; ++i) {
            double s = 0.0;
            for (i64 l = i; l <= j; ++l) s += a(i, l) * b(l, j);
            c.at(i, j) = s;
        }
    return c;
}

Mat mat_mul_nn(const Mat& a, const Mat& b) {
    dim_check(a.cols == b.rows, "mat_mul inner dimensions");
    Mat c(a.rows, b.cols);
    for (i64 j = 0; j < b.cols; ++j) {
        double* cj = c.col(j);
        for (i64 l = 0; l < a.cols; ++l) {
            const double blj = b(l, j);
            if (blj != 0.0) axpy_seq(blj, a.col(l), cj, a.rows);
        }
    }
    return c;
}

Mat assemble_hessenberg(const Upper& r, i64 m, const std::vector<BlockRecord>& blocks) {
    dim_check(r.dim >= m + 1, "coefficient matrix too small");
    // H = R_lead · T, T the (m+1)×m monomial shift (ones on the subdiagonal).
    Mat r_lead(m + 1, m + 1);
    for (i64 j = 0; j <= m; ++j)
        for (i64 i = 0; i <= j; ++i) r_lead(i, j) = r(i, j);
    Mat t(m + 1, m);
    for (i64 k = 0; k < m; ++k) t(k + 1, k) = 1.0;
    Mat h = mat_mul_nn(r_lead, t);

    for (size_t bi = 0; bi < blocks.size(); ++bi) {
        const BlockRecord& b = blocks[bi];
        if (b.c0 >= m) break;
        const bool last = (bi + 1 == blocks.size());
        i64 owned = std::min(m - b.c0, b.width - 1);
        if (last) owned = std::min(m - b.c0, b.width);
        for (i64 k = 0; k < owned; ++k) {
            double* col = h.col(b.c0 + k);
            for (i64 l = 0; l < b.c0; ++l) {
                const double coeff = (k == 0 && b.overlap) ? b.carried[l] : r(l, b.c0 + k);
                if (coeff != 0.0) axpy_seq(-coeff, h.col(l), col, m + 1);
            }
            for (i64 i = 0; i < k; ++i) {
                const double rik = r(b.c0 + i, b.c0 + k);
                if (rik != 0.0) axpy_seq(-rik, h.col(b.c0 + i), col, m + 1);
            }
            const double diag = (k == 0 && b.overlap) ? b.carried_diag : r(b.c0 + k, b.c0 + k);
            if (diag == 0.0)
                fail(KRY_SINGULAR_R,
                     "basis coefficient matrix singular at column " + std::to_string(b.c0 + k + 1),
                     b.c0 + k + 1);
            const double inv = 1.0 / diag;
            for (i64 i = 0; i < m + 1; ++i) col[i] *= inv;
        }
    }
    for (i64 j = 0; j < m; ++j)
        for (i64 i = j + 2; i < m + 1; ++i) h(i, j) = 0.0;
    return h;
}

Lsq solve_hessenberg_lsq(const Mat& h, double gamma) {
    const i64 kc = h.cols;
    dim_check(h.rows == kc + 1, "Hessenberg shape");
    Mat w = h;
    std::vector<double> g(static_cast<size_t>(kc + 1), 0.0), cs(static_cast<size_t>(kc), 1.0),
        sn(static_cast<size_t>(kc), 0.0);
    g[0] = gamma;
    i64 valid = kc;
    for (i64 k = 0; k < kc; ++k) {
        for (i64 i = 0; i < k; ++i) {
            const double t = cs[i] * w(i, k) + sn[i] * w(i + 1, k);
            w(i + 1, k) = -sn[i] * w(i, k) + cs[i] * w(i + 1, k);
            w(i, k) = t;
        }
        const double d = std::hypot(w(k, k), w(k + 1, k));
        if (d == 0.0) {
            valid = k;
            break;
        }
        cs[k] = w(k, k) / d;
        sn[k] = w(k + 1, k) / d;
        w(k, k) = d;
        w(k + 1, k) = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
    }
    Lsq out;
    out.valid_cols = valid;
    out.implicit_residual = std::abs(g[valid]);
    out.y.assign(static_cast<size_t>(valid), 0.0);
    for (i64 i = valid; i-- > 0;) {
        double s = g[i];
        for (i64 l = i + 1; l < valid; ++l) s -= w(i, l) * out.y[l];
        out.y[i] = s / w(i, i);
    }
    return out;
}

// ---- breakdown diagnostic (spectral.hpp) ---------------------------------

namespace {

// householder_r (dense_kernels.hpp:230-258).
Upper householder_r(const Mat& v) {
    const i64 n = v.rows, k = v.cols;
    dim_check(n >= k, "householder_r needs rows >= cols");
    Mat w = v;
    for (i64 j = 0; j < k; ++j) {
        double* wj = w.col(j);
        const double sigma = std::sqrt(dot_seq(wj + j, wj + j, n - j));
        if (sigma == 0.0) continue;
        const double alpha = wj[j];
        const double beta = (alpha >= 0.0) ? -sigma : sigma;
        const double v0 = alpha - beta;
        const double tau = (beta - alpha) / beta;
        for (i64 i = j + 1; i < n; ++i) wj[i] /= v0;
        wj[j] = beta;
        for (i64 jj = j + 1; jj < k; ++jj) {
            double* wc = w.col(jj);
            double s = wc[j];
            for (i64 i = j + 1; i < n; ++i) s += wj[i] * wc[i];
            s *= tau;
            wc[j] -= s;
            for (i64 i = j + 1; i < n; ++i) wc[i] -= s * wj[i];
        }
    }
    Upper r(k);
    for (i64 j = 0; j < k; ++j)
        for (i64 i = 0; i <= j; ++i) r.at(i, j) = w(i, j);
    return r;
}

// One-sided cyclic Jacobi (spectral.hpp:27-58), then σ_max/σ_min (:60-75).
double jacobi_cond(Mat a) {
    const i64 n = a.rows, k = a.cols;
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 30; ++sweep) {
        double worst = 0.0;
        for (i64 i = 0; i + 1 < k; ++i) {
            for (i64 j = i + 1; j < k; ++j) {
                double* ci = a.col(i);
                double* cj = a.col(j);
                const double aii = dot_seq(ci, ci, n);
                const double ajj = dot_seq(cj, cj, n);
                const double aij = dot_seq(ci, cj, n);
                if (aii == 0.0 || ajj == 0.0) continue;
                const double cosang = std::abs(aij) / std::sqrt(aii * ajj);
                worst = std::max(worst, cosang);
                if (cosang <= tol) continue;
                const double zeta = (ajj - aii) / (2.0 * aij);
                const double t = (zeta == 0.0) ? 1.0
                                               : std::copysign(1.0, zeta) /
                                                     (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = c * t;
                for (i64 r = 0; r < n; ++r) {
                    const double vi = ci[r], vj = cj[r];
                    ci[r] = c * vi - s * vj;
                    cj[r] = s * vi + c * vj;
                }
            }
        }
        if (worst <= tol) break;
    }
    std::vector<double> sv(static_cast<size_t>(k));
    for (i64 j = 0; j < k; ++j) sv[j] = std::sqrt(dot_seq(a.col(j), a.col(j), n));
    std::sort(sv.begin(), sv.end(), std::greater<>());
    const double smin = sv.back(), smax = sv.front();
    double cond = (smin == 0.0) ? std::numeric_limits<double>::infinity() : smax / smin;
    if (smax == 0.0) cond = 1.0;
    return cond;
}

}  // namespace

double accumulated_cond(const Mat& q, const Mat& x) {
    if (q.cols + x.cols > 512) return 0.0;  // diagnostic_kappa cap (basis_store.hpp:384)
    if (q.cols == 0 || q.rows == 0) {
        // singular_values(x) (spectral.hpp:83-99)
        Mat work;
        if (x.rows > x.cols) {
            const Upper r = householder_r(x);
            work = Mat(r.dim, r.dim);
            for (i64 j = 0; j < r.dim; ++j)
                for (i64 i = 0; i <= j; ++i) work(i, j) = r(i, j);
        } else {
            work = x;
        }
        return jacobi_cond(work);
    }
    const i64 f = q.cols, w = x.cols, n = x.rows;
    if (w == 0) return 1.0;
    Mat c(f, w);
    for (i64 j = 0; j < w; ++j)
        for (i64 i = 0; i < f; ++i) c(i, j) = dot_seq(q.col(i), x.col(j), n);
    Mat xhat = x;
    for (i64 j = 0; j < w; ++j)
        for (i64 l = 0; l < f; ++l) axpy_seq(-c(l, j), q.col(l), xhat.col(j), n);
    const Upper rhat = householder_r(xhat);
    Mat small(f + w, f + w);
    for (i64 i = 0; i < f; ++i) small(i, i) = 1.0;
    for (i64 j = 0; j < w; ++j) {
        for (i64 i = 0; i < f; ++i) small(i, f + j) = c(i, j);
        for (i64 i = 0; i <= j; ++i) small(f + i, f + j) = rhat(i, j);
    }
    return jacobi_cond(small);
}

}  // namespace kb
