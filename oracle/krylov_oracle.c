/*
 * krylov_oracle.c — TEST INFRASTRUCTURE, NOT THE PRODUCT.  See krylov_oracle.h.
 *
 * A plain-C restatement of the CPU reference's s-step GMRES hot path.  Each
 * function names the reference file:line it follows (paths relative to
 * /root/reference/proj/include/krylov/).  Build: oracle/Makefile (gcc -O2
 * -ffp-contract=off, i.e. no FMA contraction, like the reference's x86-64
 * Release build).
 */
#include "krylov_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef int64_t I;

static _Thread_local char g_err[256];
static int err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

static double* dz(I count) { return (double*)calloc((size_t)(count > 0 ? count : 1), sizeof(double)); }
static double* dup(const double* src, I count) {
    double* d = dz(count);
    if (count > 0) memcpy(d, src, (size_t)count * sizeof(double));
    return d;
}

/* dense_matrix.hpp:133-145 — sequential dot, axpy */
static double dotp(const double* a, const double* b, I n) {
    double s = 0.0;
    for (I i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static void axpy(double alpha, const double* x, double* y, I n) {
    for (I i = 0; i < n; ++i) y[i] += alpha * x[i];
}
#define AT(m, ld, i, j) ((m)[(i) + (I)(j) * (ld)])

/* ---- operators (csr_matrix.hpp:69-79, matgen.hpp:134-193) ----------------- */
typedef struct {
    I n;
    const I* rp;
    const I* ci;
    const double* v;
} csr_t;

static void spmv(const csr_t* a, const double* x, double* y) {
    for (I i = 0; i < a->n; ++i) {
        double s = 0.0;
        for (I k = a->rp[i]; k < a->rp[i + 1]; ++k) s += a->v[k] * x[a->ci[k]];
        y[i] = s;
    }
}

int orc_spmv(I n, const I* rp, const I* ci, const double* v, const double* x, double* y) {
    csr_t a = {n, rp, ci, v};
    spmv(&a, x, y);
    return KRY_OK;
}

/* Five-point / seven-point Dirichlet Laplacians with columns already in the
 * ascending order from_triplets produces (no duplicates arise). */
int orc_laplace2d(I nx, I ny, I* n, I* nnz, I* rp, I* ci, double* v) {
    if (nx < 2 || ny < 2) return err(KRY_DIMENSION_MISMATCH, "gen_laplace2d needs dimensions >= 2");
    *n = nx * ny;
    I k = 0;
    for (I iy = 0; iy < ny; ++iy)
        for (I ix = 0; ix < nx; ++ix) {
            const I row = iy * nx + ix;
            if (rp) rp[row] = k;
            const I cols[5] = {row - nx, row - 1, row, row + 1, row + nx};
            const int ok[5] = {iy > 0, ix > 0, 1, ix + 1 < nx, iy + 1 < ny};
            for (int t = 0; t < 5; ++t) {
                if (!ok[t]) continue;
                if (ci) {
                    ci[k] = cols[t];
                    v[k] = t == 2 ? 4.0 : -1.0;
                }
                ++k;
            }
        }
    if (rp) rp[*n] = k;
    *nnz = k;
    return KRY_OK;
}

int orc_laplace3d(I nx, I ny, I nz, I* n, I* nnz, I* rp, I* ci, double* v) {
    if (nx < 2 || ny < 2 || nz < 2) return err(KRY_DIMENSION_MISMATCH, "gen_laplace3d needs dimensions >= 2");
    *n = nx * ny * nz;
    const I p = nx * ny;
    I k = 0;
    for (I iz = 0; iz < nz; ++iz)
        for (I iy = 0; iy < ny; ++iy)
            for (I ix = 0; ix < nx; ++ix) {
                const I row = (iz * ny + iy) * nx + ix;
                if (rp) rp[row] = k;
                const I cols[7] = {row - p, row - nx, row - 1, row, row + 1, row + nx, row + p};
                const int ok[7] = {iz > 0, iy > 0, ix > 0, 1, ix + 1 < nx, iy + 1 < ny, iz + 1 < nz};
                for (int t = 0; t < 7; ++t) {
                    if (!ok[t]) continue;
                    if (ci) {
                        ci[k] = cols[t];
                        v[k] = t == 3 ? 6.0 : -1.0;
                    }
                    ++k;
                }
            }
    if (rp) rp[*n] = k;
    *nnz = k;
    return KRY_OK;
}

/* gmres.hpp:80-90 */
static void mpk(const csr_t* a, const double* start, I s, double* V) {
    memcpy(V, start, (size_t)a->n * sizeof(double));
    for (I k = 0; k < s; ++k) spmv(a, V + k * a->n, V + (k + 1) * a->n);
}

int orc_mpk(I n, const I* rp, const I* ci, const double* v, const double* start, I s, double* out) {
    csr_t a = {n, rp, ci, v};
    mpk(&a, start, s, out);
    return KRY_OK;
}

/* ---- dense kernels (dense_kernels.hpp) ------------------------------------ */
/* gram :95-105 (upper computed, mirrored) */
static void gram(I n, I k, const double* v, double* g) {
    for (I j = 0; j < k; ++j)
        for (I i = 0; i <= j; ++i) AT(g, k, i, j) = dotp(v + i * n, v + j * n, n);
    for (I j = 0; j < k; ++j)
        for (I i = 0; i < j; ++i) AT(g, k, j, i) = AT(g, k, i, j);
}
int orc_gram(I n, I k, const double* v, double* g) {
    gram(n, k, v, g);
    return KRY_OK;
}

/* mat_mul(A, B, Trans, None) :71-75 — c(i,j) = dot(a_i, b_j) */
static void mat_tn(I n, I ka, const double* a, I kb, const double* b, double* c) {
    for (I j = 0; j < kb; ++j)
        for (I i = 0; i < ka; ++i) AT(c, ka, i, j) = dotp(a + i * n, b + j * n, n);
}

/* mat_mul(A, B) :63-70 — column-wise axpy, zero coefficients skipped; c zeroed */
static void mat_nn(I am, I ak, const double* a, I bn, const double* b, double* c) {
    for (I j = 0; j < bn; ++j) {
        double* cj = c + j * am;
        for (I l = 0; l < ak; ++l) {
            const double blj = AT(b, ak, l, j);
            if (blj != 0.0) axpy(blj, a + l * am, cj, am);
        }
    }
}

/* try_cholesky :111-127; r (k×k) zeroed here */
static I try_chol(I k, const double* s, double* r) {
    memset(r, 0, (size_t)(k * k) * sizeof(double));
    for (I j = 0; j < k; ++j) {
        for (I i = 0; i < j; ++i) {
            double sum = AT(s, k, i, j);
            for (I t = 0; t < i; ++t) sum -= AT(r, k, t, i) * AT(r, k, t, j);
            AT(r, k, i, j) = sum / AT(r, k, i, i);
        }
        double d = AT(s, k, j, j);
        for (I t = 0; t < j; ++t) d -= AT(r, k, t, j) * AT(r, k, t, j);
        if (!(d > 0.0)) return j + 1;
        AT(r, k, j, j) = sqrt(d);
    }
    return 0;
}
int orc_try_cholesky(I k, const double* s, double* r, I* pivot) {
    *pivot = try_chol(k, s, r);
    return KRY_OK;
}

/* tri_solve_right :139-154 — x = v R⁻¹ (x may not alias v) */
static int tri_solve_right(I n, I k, const double* v, const double* r, double* x) {
    for (I j = 0; j < k; ++j)
        if (AT(r, k, j, j) == 0.0) return err(KRY_SINGULAR_FACTOR, "triangular factor has a zero diagonal entry");
    for (I j = 0; j < k; ++j) {
        double* xj = x + j * n;
        memcpy(xj, v + j * n, (size_t)n * sizeof(double));
        for (I l = 0; l < j; ++l) axpy(-AT(r, k, l, j), x + l * n, xj, n);
        const double inv = 1.0 / AT(r, k, j, j);
        for (I i = 0; i < n; ++i) xj[i] *= inv;
    }
    return KRY_OK;
}

/* tri_mul :261-272 — c = a·b, upper */
static void tri_mul(I k, const double* a, const double* b, double* c) {
    memset(c, 0, (size_t)(k * k) * sizeof(double));
    for (I j = 0; j < k; ++j)
        for (I i = 0; i <= j; ++i) {
            double s = 0.0;
            for (I l = i; l <= j; ++l) s += AT(a, k, i, l) * AT(b, k, l, j);
            AT(c, k, i, j) = s;
        }
}

/* ---- block orthogonalization (block_ortho.hpp) ----------------------------- */
/* bcgs_pip_partial :152-178.  Returns the bad pivot (0 on success); q is
 * written only on success. */
static I pip_partial(I n, const double* qp, I c0, const double* v, I w, double* q, double* rcol, double* rchol,
                     I* reduces) {
    *reduces += 1;
    if (c0 > 0) mat_tn(n, c0, qp, w, v, rcol);
    double* s = dz(w * w);
    gram(n, w, v, s);
    if (c0 > 0)
        for (I j = 0; j < w; ++j)
            for (I i = 0; i <= j; ++i) {
                const double c = dotp(rcol + i * c0, rcol + j * c0, c0);
                AT(s, w, i, j) -= c;
                if (i != j) AT(s, w, j, i) = AT(s, w, i, j);
            }
    const I bad = try_chol(w, s, rchol);
    free(s);
    if (bad) return bad;
    double* vhat = dup(v, n * w);
    for (I j = 0; j < w; ++j)
        for (I l = 0; l < c0; ++l) axpy(-AT(rcol, c0, l, j), qp + l * n, vhat + j * n, n);
    tri_solve_right(n, w, vhat, rchol, q);
    free(vhat);
    return 0;
}

int orc_bcgs_pip_partial(I n, const double* qp, I c0, const double* v, I w, double* q, double* r_col,
                         double* r_chol, I* bad_pivot, I* reduces) {
    I red = 0;
    *bad_pivot = pip_partial(n, qp, c0, v, w, q, r_col, r_chol, &red);
    if (reduces) *reduces += red;
    return KRY_OK;
}

/* bcgs_pip :180-189 */
int orc_bcgs_pip(I n, const double* qp, I c0, const double* v, I w, double* q, double* r_col, double* r_jj,
                 I* pivot, I* reduces) {
    I red = 0;
    const I bad = pip_partial(n, qp, c0, v, w, q, r_col, r_jj, &red);
    if (reduces) *reduces += red;
    if (pivot) *pivot = bad;
    return bad ? err(KRY_NOT_POSITIVE_DEFINITE, "matrix not positive definite") : KRY_OK;
}

/* R_col := R_col₁ + R_col₂·R_jj₁ ; R_jj := R_jj₂·R_jj₁ (bcgs_pip2 :197-206) */
static void combine_two(I c0, I w, double* rcol1, const double* rjj1, const double* rcol2, const double* rjj2,
                        double* rjj_out) {
    if (c0 > 0) {
        double* corr = dz(c0 * w);
        mat_nn(c0, w, rcol2, w, rjj1, corr);
        for (I j = 0; j < w; ++j)
            for (I i = 0; i < c0; ++i) AT(rcol1, c0, i, j) += AT(corr, c0, i, j);
        free(corr);
    }
    tri_mul(w, rjj2, rjj1, rjj_out);
}

/* bcgs_pip2 :192-208 */
int orc_bcgs_pip2(I n, const double* qp, I c0, const double* v, I w, double* q, double* r_col, double* r_jj,
                  I* pivot, I* reduces) {
    double *q1 = dz(n * w), *rj1 = dz(w * w), *rc2 = dz(c0 * w), *rj2 = dz(w * w);
    I red = 0;
    int rc = KRY_OK;
    I bad = pip_partial(n, qp, c0, v, w, q1, r_col, rj1, &red);
    if (!bad) bad = pip_partial(n, qp, c0, q1, w, q, rc2, rj2, &red);
    if (bad) {
        rc = err(KRY_NOT_POSITIVE_DEFINITE, "matrix not positive definite");
    } else {
        combine_two(c0, w, r_col, rj1, rc2, rj2, r_jj);
    }
    if (pivot) *pivot = bad;
    if (reduces) *reduces += red;
    free(q1), free(rj1), free(rc2), free(rj2);
    return rc;
}

/* cholqr :49-54 — returns pivot (0 ok) */
static I cholqr(I n, const double* v, I w, double* q, double* r, I* red) {
    *red += 1;
    double* g = dz(w * w);
    gram(n, w, v, g);
    const I bad = try_chol(w, g, r);
    free(g);
    if (!bad) tri_solve_right(n, w, v, r, q);
    return bad;
}
/* cholqr2 :57-61 */
static I cholqr2(I n, const double* v, I w, double* q, double* r, I* red) {
    double *q1 = dz(n * w), *r1 = dz(w * w), *r2 = dz(w * w);
    I bad = cholqr(n, v, w, q1, r1, red);
    if (!bad) bad = cholqr(n, q1, w, q, r2, red);
    if (!bad) tri_mul(w, r2, r1, r);
    free(q1), free(r1), free(r2);
    return bad;
}
/* bcgs_project :70-87 (c0 > 0 here) */
static void project(I n, const double* qp, I c0, const double* v, I w, double* vhat, double* rblock, I* red) {
    *red += 1;
    mat_tn(n, c0, qp, w, v, rblock);
    memcpy(vhat, v, (size_t)(n * w) * sizeof(double));
    for (I j = 0; j < w; ++j)
        for (I l = 0; l < c0; ++l) axpy(-AT(rblock, c0, l, j), qp + l * n, vhat + j * n, n);
}

/* ---- breakdown diagnostic (spectral.hpp, dense_kernels.hpp:230-258) --------- */
static void householder_r(I n, I k, const double* v, double* r) {
    double* w = dup(v, n * k);
    for (I j = 0; j < k; ++j) {
        double* wj = w + j * n;
        const double sigma = sqrt(dotp(wj + j, wj + j, n - j));
        if (sigma == 0.0) continue;
        const double alpha = wj[j];
        const double beta = (alpha >= 0.0) ? -sigma : sigma;
        const double v0 = alpha - beta;
        const double tau = (beta - alpha) / beta;
        for (I i = j + 1; i < n; ++i) wj[i] /= v0;
        wj[j] = beta;
        for (I jj = j + 1; jj < k; ++jj) {
            double* wc = w + jj * n;
            double s = wc[j];
            for (I i = j + 1; i < n; ++i) s += wj[i] * wc[i];
            s *= tau;
            wc[j] -= s;
            for (I i = j + 1; i < n; ++i) wc[i] -= s * wj[i];
        }
    }
    memset(r, 0, (size_t)(k * k) * sizeof(double));
    for (I j = 0; j < k; ++j)
        for (I i = 0; i <= j; ++i) AT(r, k, i, j) = AT(w, n, i, j);
    free(w);
}

static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

static double jacobi_cond(I n, I k, double* a) {
    for (int sweep = 0; sweep < 30; ++sweep) {
        double worst = 0.0;
        for (I i = 0; i + 1 < k; ++i)
            for (I j = i + 1; j < k; ++j) {
                double *ci = a + i * n, *cj = a + j * n;
                const double aii = dotp(ci, ci, n), ajj = dotp(cj, cj, n), aij = dotp(ci, cj, n);
                if (aii == 0.0 || ajj == 0.0) continue;
                const double cosang = fabs(aij) / sqrt(aii * ajj);
                if (cosang > worst) worst = cosang;
                if (cosang <= 1e-15) continue;
                const double zeta = (ajj - aii) / (2.0 * aij);
                const double t = (zeta == 0.0) ? 1.0 : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (I r = 0; r < n; ++r) {
                    const double vi = ci[r], vj = cj[r];
                    ci[r] = c * vi - s * vj;
                    cj[r] = s * vi + c * vj;
                }
            }
        if (worst <= 1e-15) break;
    }
    double* sv = dz(k);
    for (I j = 0; j < k; ++j) sv[j] = sqrt(dotp(a + j * n, a + j * n, n));
    qsort(sv, (size_t)k, sizeof(double), cmp_desc);
    const double smax = sv[0], smin = sv[k - 1];
    free(sv);
    if (smax == 0.0) return 1.0;
    return smin == 0.0 ? INFINITY : smax / smin;
}

/* accumulated_cond(q, x).cond (spectral.hpp:151-176) */
static double accumulated_cond(I n, I f, const double* q, I w, const double* x) {
    if (f + w > 512) return 0.0;
    if (f == 0) {
        if (n > w) {
            double* r = dz(w * w);
            householder_r(n, w, x, r);
            const double c = jacobi_cond(w, w, r);
            free(r);
            return c;
        }
        double* cpy = dup(x, n * w);
        const double c = jacobi_cond(n, w, cpy);
        free(cpy);
        return c;
    }
    if (w == 0) return 1.0;
    double* c = dz(f * w);
    mat_tn(n, f, q, w, x, c);
    double* xhat = dup(x, n * w);
    for (I j = 0; j < w; ++j)
        for (I l = 0; l < f; ++l) axpy(-AT(c, f, l, j), q + l * n, xhat + j * n, n);
    double* rhat = dz(w * w);
    householder_r(n, w, xhat, rhat);
    const I k = f + w;
    double* small = dz(k * k);
    for (I i = 0; i < f; ++i) AT(small, k, i, i) = 1.0;
    for (I j = 0; j < w; ++j) {
        for (I i = 0; i < f; ++i) AT(small, k, i, f + j) = AT(c, f, i, j);
        for (I i = 0; i <= j; ++i) AT(small, k, f + i, f + j) = AT(rhat, w, i, j);
    }
    const double cond = jacobi_cond(k, k, small);
    free(c), free(xhat), free(rhat), free(small);
    return cond;
}

/* ---- basis store (basis_store.hpp) ------------------------------------------ */
typedef struct {
    I c0, width;
    int overlap;
    double* carried; /* c0 entries (overlap records) */
    double carried_diag;
} record_t;

struct orc_store {
    I n, maxc, s, shat, filled, finalized, bps;
    int seam;
    double* q; /* n × maxc */
    double* r; /* maxc × maxc */
    int* states;
    I nstates;
    record_t* recs;
    I nrecs;
};

typedef struct {
    double* q;    /* n × w */
    double* rcol; /* c0 × w */
    double* rjj;  /* w × w */
} res_t;

static void res_free(res_t* r) { free(r->q), free(r->rcol), free(r->rjj); }

enum { OK_ = 0, FIRST_FAIL = 1, SECOND_FAIL = 2 };

/* ctor :44-55 */
int orc_store_create(I n, I m, I s, I shat, orc_store** out) {
    const I eff = shat == 0 ? m : shat;
    if (s == 0 || m % s != 0) return err(KRY_DIMENSION_MISMATCH, "panel size must divide the restart length");
    if (eff % s != 0 || eff > m)
        return err(KRY_DIMENSION_MISMATCH, "big panel size must be a multiple of the panel size, <= m");
    orc_store* st = (orc_store*)calloc(1, sizeof(orc_store));
    st->n = n, st->maxc = m + 1, st->s = s, st->shat = eff;
    st->q = dz(n * (m + 1));
    st->r = dz((m + 1) * (m + 1));
    st->states = (int*)calloc((size_t)(m + 2) * 4, sizeof(int));
    st->recs = (record_t*)calloc((size_t)(m + 2) * 4, sizeof(record_t));
    *out = st;
    return KRY_OK;
}

static void store_reset(orc_store* st) { /* :84-93 */
    st->filled = st->finalized = st->bps = 0;
    st->seam = 0;
    st->nstates = 0;
    for (I i = 0; i < st->nrecs; ++i) free(st->recs[i].carried);
    st->nrecs = 0;
    memset(st->q, 0, (size_t)(st->n * st->maxc) * sizeof(double));
    memset(st->r, 0, (size_t)(st->maxc * st->maxc) * sizeof(double));
}

void orc_store_destroy(orc_store* st) {
    if (!st) return;
    for (I i = 0; i < st->nrecs; ++i) free(st->recs[i].carried);
    free(st->q), free(st->r), free(st->states), free(st->recs), free(st);
}

#define R_(st, i, j) AT((st)->r, (st)->maxc, i, j)

/* run_scheme :215-283.  Returns OK_, FIRST_FAIL or SECOND_FAIL (pivot in *piv). */
static int run_scheme(orc_store* st, I c0, const double* v, I w, int kind, I* red, res_t* out, I* piv) {
    const I n = st->n;
    const double* pre = st->q;
    out->q = dz(n * w), out->rcol = dz(c0 * w), out->rjj = dz(w * w);
    if (kind == KRY_ORTHO_TWO_STAGE) {
        *piv = pip_partial(n, pre, c0, v, w, out->q, out->rcol, out->rjj, red);
        return *piv ? FIRST_FAIL : OK_;
    }
    if (kind == KRY_ORTHO_BCGS_PIP2) {
        double *q1 = dz(n * w), *rj1 = dz(w * w), *rc2 = dz(c0 * w), *rj2 = dz(w * w);
        int status = OK_;
        *piv = pip_partial(n, pre, c0, v, w, q1, out->rcol, rj1, red);
        if (*piv) {
            status = FIRST_FAIL;
        } else {
            *piv = pip_partial(n, pre, c0, q1, w, out->q, rc2, rj2, red);
            if (*piv)
                status = SECOND_FAIL;
            else
                combine_two(c0, w, out->rcol, rj1, rc2, rj2, out->rjj);
        }
        free(q1), free(rj1), free(rc2), free(rj2);
        return status;
    }
    /* Bcgs2Cholqr2 (the single-column case is CholQR, i.e. CGS2) */
    const int single = (w == 1);
    if (c0 == 0) {
        *piv = single ? cholqr(n, v, w, out->q, out->rjj, red) : cholqr2(n, v, w, out->q, out->rjj, red);
        return *piv ? FIRST_FAIL : OK_;
    }
    double *vhat = dz(n * w), *rb1 = dz(c0 * w), *qi = dz(n * w), *ri = dz(w * w);
    int status = OK_;
    project(n, pre, c0, v, w, vhat, rb1, red);
    *piv = single ? cholqr(n, vhat, w, qi, ri, red) : cholqr2(n, vhat, w, qi, ri, red);
    if (*piv) {
        status = FIRST_FAIL;
    } else {
        double *vh2 = dz(n * w), *rb2 = dz(c0 * w), *ro = dz(w * w);
        project(n, pre, c0, qi, w, vh2, rb2, red);
        *piv = cholqr(n, vh2, w, out->q, ro, red);
        if (*piv) {
            status = SECOND_FAIL;
        } else {
            double* corr = dz(c0 * w);
            mat_nn(c0, w, rb2, w, ri, corr);
            for (I j = 0; j < w; ++j)
                for (I i = 0; i < c0; ++i) AT(out->rcol, c0, i, j) = AT(rb1, c0, i, j) + AT(corr, c0, i, j);
            tri_mul(w, ro, ri, out->rjj);
            free(corr);
        }
        free(vh2), free(rb2), free(ro);
    }
    free(vhat), free(rb1), free(qi), free(ri);
    return status;
}

/* commit :285-327 */
static void commit(orc_store* st, I c0, int overlap, const res_t* res, I w, int state) {
    record_t* rec = &st->recs[st->nrecs++];
    rec->c0 = c0, rec->width = w, rec->overlap = overlap, rec->carried = NULL, rec->carried_diag = 1.0;
    if (overlap) {
        const double rho = R_(st, c0, c0);
        if (c0 > 0) rec->carried = dup(res->rcol, c0);
        rec->carried_diag = AT(res->rjj, w, 0, 0);
        for (I i = 0; i < c0; ++i) R_(st, i, c0) += rho * AT(res->rcol, c0, i, 0);
        R_(st, c0, c0) = rho * AT(res->rjj, w, 0, 0);
        for (I j = 1; j < w; ++j) {
            for (I i = 0; i < c0; ++i) R_(st, i, c0 + j) = AT(res->rcol, c0, i, j);
            for (I i = 0; i <= j; ++i) R_(st, c0 + i, c0 + j) = AT(res->rjj, w, i, j);
        }
    } else {
        for (I j = 0; j < w; ++j) {
            for (I i = 0; i < c0; ++i) R_(st, i, c0 + j) = AT(res->rcol, c0, i, j);
            for (I i = 0; i <= j; ++i) R_(st, c0 + i, c0 + j) = AT(res->rjj, w, i, j);
        }
    }
    memcpy(st->q + c0 * st->n, res->q, (size_t)(st->n * w) * sizeof(double));
    st->filled = c0 + w;
    st->seam = 0;
    if (state == KRY_PANEL_FINAL) {
        st->finalized = st->bps = st->filled;
    } else {
        if (c0 < st->bps) st->bps = c0;
        if (c0 < st->finalized) st->finalized = c0;
    }
    st->states[st->nstates++] = state;
}

/* record_seam :374-381 */
static void record_seam(orc_store* st, const double* dropped, I* red) {
    if (st->filled >= st->maxc) return;
    *red += 1;
    for (I i = 0; i < st->filled; ++i) R_(st, i, st->filled) = dotp(st->q + i * st->n, dropped, st->n);
    R_(st, st->filled, st->filled) = 0.0;
    st->seam = 1;
}

static double diag_kappa(orc_store* st, I c0, const double* v, I w) { /* :383-387 */
    if (c0 + w > 512) return 0.0;
    return accumulated_cond(st->n, c0, st->q, w, v);
}

/* append_block :112-118 → append_impl :169-209 */
static int append(orc_store* st, const double* v, I w, int overlap, int kind, kry_append_outcome* o, I* red) {
    memset(o, 0, sizeof *o);
    if (overlap && st->filled == 0) return err(KRY_DIMENSION_MISMATCH, "basis store capacity exceeded");
    const I c0 = overlap ? st->filled - 1 : st->filled;
    I width = w;
    if (c0 + width > st->maxc) return err(KRY_DIMENSION_MISMATCH, "basis store capacity exceeded");
    while (width >= 1) {
        res_t res;
        I piv = 0;
        const int status = run_scheme(st, c0, v, width, kind, red, &res, &piv);
        if (status == OK_) {
            commit(st, c0, overlap, &res, width,
                   kind == KRY_ORTHO_TWO_STAGE ? KRY_PANEL_PREPROCESSED : KRY_PANEL_FINAL);
            res_free(&res);
            o->committed = width;
            if (o->truncated) record_seam(st, v + width * st->n, red);
            return KRY_OK;
        }
        res_free(&res);
        if (status == SECOND_FAIL) {
            o->breakdown = 1, o->truncated = 0, o->pivot = piv;
            o->kappa_estimate = diag_kappa(st, c0, v, width);
            return KRY_OK;
        }
        o->truncated = 1, o->pivot = piv;
        if (piv <= 1) break;
        if (piv - 1 < width) width = piv - 1;
    }
    o->breakdown = 1, o->truncated = 0;
    o->kappa_estimate = diag_kappa(st, c0, v, w);
    return KRY_OK;
}

int orc_store_append_block(orc_store* st, const double* v, I w, int overlap, int32_t kind, kry_append_outcome* out,
                           I* delta) {
    I red = 0;
    const int rc = append(st, v, w, overlap, kind, out, &red);
    if (delta) *delta = red;
    return rc;
}

int orc_store_preprocess_block(orc_store* st, const double* v, I w, int overlap, kry_append_outcome* out,
                               I* delta) {
    return orc_store_append_block(st, v, w, overlap, KRY_ORTHO_TWO_STAGE, out, delta);
}

/* combine_column :331-345 */
static void combine_column(orc_store* st, I col, I c0, I w, const res_t* res) {
    double* part = dz(w);
    const I top = col < c0 + w - 1 ? col : c0 + w - 1;
    for (I i = c0; i <= top; ++i) part[i - c0] = R_(st, i, col);
    for (I i = 0; i < c0; ++i) {
        double s = 0.0;
        for (I l = 0; l < w; ++l) s += AT(res->rcol, c0, i, l) * part[l];
        R_(st, i, col) += s;
    }
    for (I i = 0; i < w && c0 + i <= col; ++i) {
        double s = 0.0;
        for (I l = i; l < w; ++l) s += AT(res->rjj, w, i, l) * part[l];
        R_(st, c0 + i, col) = s;
    }
    free(part);
}

/* combine_record :347-369 (a non-overlap record with c0 > 0 has no carried
 * column — the reference reads past an empty vector there; skipped, as in
 * the product) */
static void combine_record(record_t* rec, I c0, I w, const res_t* res) {
    if (!rec->overlap && rec->c0 > 0) return;
    double* full = dz(rec->c0 + 1);
    for (I i = 0; i < rec->c0; ++i) full[i] = rec->carried[i];
    full[rec->c0] = rec->carried_diag;
    double* part = dz(w);
    const I top = rec->c0 < c0 + w - 1 ? rec->c0 : c0 + w - 1;
    for (I i = c0; i <= top; ++i) part[i - c0] = full[i];
    for (I i = 0; i < c0; ++i) {
        double s = 0.0;
        for (I l = 0; l < w; ++l) s += AT(res->rcol, c0, i, l) * part[l];
        full[i] += s;
    }
    for (I i = 0; i < w && c0 + i <= rec->c0; ++i) {
        double s = 0.0;
        for (I l = i; l < w; ++l) s += AT(res->rjj, w, i, l) * part[l];
        full[c0 + i] = s;
    }
    for (I i = 0; i < rec->c0; ++i) rec->carried[i] = full[i];
    rec->carried_diag = full[rec->c0];
    free(full), free(part);
}

/* finalize_big_panel :131-166 */
static int finalize(orc_store* st, kry_append_outcome* o, I* red, int* pushed) {
    memset(o, 0, sizeof *o);
    *pushed = 0;
    if (!(st->filled > st->bps)) return KRY_OK;
    *pushed = 1;
    const I c0 = st->bps, w = st->filled - c0, n = st->n;
    res_t res = {dz(n * w), dz(c0 * w), dz(w * w)};
    const double* panel = st->q + c0 * n;
    const I piv = pip_partial(n, st->q, c0, panel, w, res.q, res.rcol, res.rjj, red);
    if (piv) {
        o->breakdown = 1, o->pivot = piv;
        o->kappa_estimate = diag_kappa(st, c0, panel, w);
        res_free(&res);
        return KRY_OK;
    }
    for (I col = c0; col < st->filled; ++col) combine_column(st, col, c0, w, &res);
    for (I i = 0; i < st->nrecs; ++i)
        if (st->recs[i].c0 >= c0) combine_record(&st->recs[i], c0, w, &res);
    memcpy(st->q + c0 * n, res.q, (size_t)(n * w) * sizeof(double));
    st->finalized = st->bps = st->filled;
    for (I i = 0; i < st->nstates; ++i)
        if (st->states[i] == KRY_PANEL_PREPROCESSED) st->states[i] = KRY_PANEL_FINAL;
    o->committed = w;
    res_free(&res);
    return KRY_OK;
}

int orc_store_finalize_big_panel(orc_store* st, kry_append_outcome* out, I* delta) {
    I red = 0;
    int pushed = 0;
    const int rc = finalize(st, out, &red, &pushed);
    if (delta) *delta = red;
    return rc;
}

int orc_store_get_info(orc_store* st, kry_store_info* info) {
    memset(info, 0, sizeof *info);
    info->rows = st->n, info->capacity = st->maxc, info->filled = st->filled, info->finalized = st->finalized;
    info->big_panel_start = st->bps, info->panel_size = st->s, info->big_panel_size = st->shat;
    info->seam_valid = st->seam, info->big_panel_open = st->filled > st->bps;
    info->big_panel_full = st->filled > st->bps && st->filled - st->bps >= st->shat + 1;
    info->n_records = st->nrecs, info->n_panel_states = st->nstates, info->ld = st->n;
    return KRY_OK;
}

int orc_store_coefficients(orc_store* st, double* r) {
    memcpy(r, st->r, (size_t)(st->maxc * st->maxc) * sizeof(double));
    return KRY_OK;
}

int orc_store_columns(orc_store* st, I first, I count, double* out) {
    memcpy(out, st->q + first * st->n, (size_t)(count * st->n) * sizeof(double));
    return KRY_OK;
}

/* ---- restart-loop host algebra (gmres.hpp:100-185) -------------------------- */
/* assemble_hessenberg with ChangeOfBasis::monomial(m) (:40-49, :100-136); h is (m+1)×m */
static int hessenberg(const orc_store* st, I m, double* h, I* singular) {
    const I k1 = m + 1, ldr = st->maxc;
    double* rl = dz(k1 * k1);
    for (I j = 0; j < k1; ++j)
        for (I i = 0; i <= j; ++i) AT(rl, k1, i, j) = AT(st->r, ldr, i, j);
    double* t = dz(k1 * m);
    for (I k = 0; k < m; ++k) AT(t, k1, k + 1, k) = 1.0;
    memset(h, 0, (size_t)(k1 * m) * sizeof(double));
    mat_nn(k1, k1, rl, m, t, h);
    free(rl), free(t);
    for (I bi = 0; bi < st->nrecs; ++bi) {
        const record_t* b = &st->recs[bi];
        if (b->c0 >= m) break;
        const int last = (bi + 1 == st->nrecs);
        I owned = (m - b->c0 < b->width - 1) ? m - b->c0 : b->width - 1;
        if (last) owned = (m - b->c0 < b->width) ? m - b->c0 : b->width;
        for (I k = 0; k < owned; ++k) {
            double* col = h + (b->c0 + k) * k1;
            for (I l = 0; l < b->c0; ++l) {
                const double coeff = (k == 0 && b->overlap) ? b->carried[l] : AT(st->r, ldr, l, b->c0 + k);
                if (coeff != 0.0) axpy(-coeff, h + l * k1, col, k1);
            }
            for (I i = 0; i < k; ++i) {
                const double rik = AT(st->r, ldr, b->c0 + i, b->c0 + k);
                if (rik != 0.0) axpy(-rik, h + (b->c0 + i) * k1, col, k1);
            }
            const double diag = (k == 0 && b->overlap) ? b->carried_diag : AT(st->r, ldr, b->c0 + k, b->c0 + k);
            if (diag == 0.0) {
                if (singular) *singular = b->c0 + k + 1;
                return err(KRY_SINGULAR_R, "basis coefficient matrix singular");
            }
            const double inv = 1.0 / diag;
            for (I i = 0; i < k1; ++i) col[i] *= inv;
        }
    }
    for (I j = 0; j < m; ++j)
        for (I i = j + 2; i < k1; ++i) AT(h, k1, i, j) = 0.0;
    return KRY_OK;
}

int orc_store_hessenberg(orc_store* st, I k, double* h, I* singular) { return hessenberg(st, k, h, singular); }

/* solve_hessenberg_lsq :146-185 */
static void lsq(I kc, const double* h, double gamma, double* y, double* implicit, I* valid_out) {
    const I k1 = kc + 1;
    double* w = dup(h, k1 * kc);
    double *g = dz(k1), *cs = dz(kc), *sn = dz(kc);
    for (I i = 0; i < kc; ++i) cs[i] = 1.0;
    g[0] = gamma;
    I valid = kc;
    for (I k = 0; k < kc; ++k) {
        for (I i = 0; i < k; ++i) {
            const double t = cs[i] * AT(w, k1, i, k) + sn[i] * AT(w, k1, i + 1, k);
            AT(w, k1, i + 1, k) = -sn[i] * AT(w, k1, i, k) + cs[i] * AT(w, k1, i + 1, k);
            AT(w, k1, i, k) = t;
        }
        const double d = hypot(AT(w, k1, k, k), AT(w, k1, k + 1, k));
        if (d == 0.0) {
            valid = k;
            break;
        }
        cs[k] = AT(w, k1, k, k) / d;
        sn[k] = AT(w, k1, k + 1, k) / d;
        AT(w, k1, k, k) = d;
        AT(w, k1, k + 1, k) = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
    }
    *valid_out = valid;
    *implicit = fabs(g[valid]);
    for (I i = valid; i-- > 0;) {
        double s = g[i];
        for (I l = i + 1; l < valid; ++l) s -= AT(w, k1, i, l) * y[l];
        y[i] = s / AT(w, k1, i, i);
    }
    free(w), free(g), free(cs), free(sn);
}

int orc_hessenberg_lsq(I k, const double* h, double gamma, double* y, double* implicit, I* valid) {
    lsq(k, h, gamma, y, implicit, valid);
    return KRY_OK;
}

/* ---- the restart loop (gmres.hpp:187-411) ------------------------------------ */
typedef struct {
    int implicit_crossed, applied;
    double explicit_rel;
} check_t;

typedef struct {
    const csr_t* a;
    const double* b;
    const kry_solver_config* cfg;
    orc_store* st;
    double *x, *r, r0;
    kry_report* rep;
} solver_t;

static double norm2(const double* v, I n) { return sqrt(dotp(v, v, n)); }

static void residual(const csr_t* a, const double* b, const double* x, double* r) { /* :189-194 */
    spmv(a, x, r);
    for (I i = 0; i < a->n; ++i) r[i] = b[i] - r[i];
}

static I usable_cols(const orc_store* st) { /* :227-234 */
    I k = st->filled == 0 ? 0 : st->filled - 1;
    if (st->seam) ++k;
    for (I j = 0; j < k; ++j)
        if (AT(st->r, st->maxc, j, j) == 0.0) return j;
    return k;
}

static int check_and_update(solver_t* S, double gamma, int force, check_t* res) { /* :247-269 */
    res->implicit_crossed = res->applied = 0;
    res->explicit_rel = INFINITY;
    const I k = usable_cols(S->st);
    if (k == 0) return KRY_OK;
    const I n = S->a->n;
    double* h = dz((k + 1) * k);
    I sing = 0;
    int rc = hessenberg(S->st, k, h, &sing);
    if (rc) {
        free(h);
        return rc;
    }
    double* y = dz(k);
    double imp = 0;
    I valid = 0;
    lsq(k, h, gamma, y, &imp, &valid);
    free(h);
    res->implicit_crossed = imp <= S->cfg->rel_tol * S->r0;
    if (!res->implicit_crossed && !force) {
        free(y);
        return KRY_OK;
    }
    double* xn = dup(S->x, n);
    for (I l = 0; l < valid; ++l) axpy(y[l], S->st->q + l * n, xn, n);
    double* rn = dz(n);
    residual(S->a, S->b, xn, rn);
    const double nrm = norm2(rn, n);
    res->explicit_rel = nrm / S->r0;
    if (nrm <= gamma * (1.0 + 1e-12)) {
        memcpy(S->x, xn, (size_t)n * sizeof(double));
        memcpy(S->r, rn, (size_t)n * sizeof(double));
        res->applied = 1;
    }
    free(xn), free(rn), free(y);
    return KRY_OK;
}

static void push_i64(int64_t* arr, I cap, I* count, I v) {
    if (*count < cap) arr[*count] = v;
    ++*count;
}

static int gmres_impl(const csr_t* a, const double* b, const double* x0, const kry_solver_config* cfg_in,
                      int standard, kry_report* rep, double* x_out) {
    kry_solver_config cfg = *cfg_in;
    if (standard) cfg.step = 1, cfg.big_step = 0, cfg.scheme_kind = KRY_ORTHO_BCGS2_CHOLQR2;
    /* SolverConfig::validate :28-35 */
    if (cfg.restart_len <= 0 || cfg.step <= 0 || cfg.restart_len % cfg.step)
        return err(KRY_DIMENSION_MISMATCH, "step size must divide the restart length");
    const I m = cfg.restart_len, shat_eff = cfg.big_step == 0 ? m : cfg.big_step;
    if (shat_eff < cfg.step || shat_eff > m || shat_eff % cfg.step)
        return err(KRY_DIMENSION_MISMATCH, "second step size must be a multiple of s in [s, m]");
    if (!(cfg.rel_tol > 0.0)) return err(KRY_INVALID_ARGUMENT, "rel_tol must be positive");
    const clock_t t0 = clock();
    const I n = a->n, s = standard ? 1 : cfg.step;
    const int two = cfg.scheme_kind == KRY_ORTHO_TWO_STAGE && !standard;
    const I shat = two ? shat_eff : s;
    rep->status = KRY_STATUS_MAX_ITERS, rep->breakdown = 0, rep->iterations = rep->restarts = 0;
    rep->reduces = 0, rep->n_cycle_residuals = rep->n_per_block = rep->n_per_big_panel = 0;
    rep->breakdown_kappa = 0.0, rep->reduces_per_iteration = 0.0;

    double* x = dz(n);
    if (x0) memcpy(x, x0, (size_t)n * sizeof(double));
    double* r = dz(n);
    residual(a, b, x, r);
    const double r0 = norm2(r, n);
    rep->initial_residual = r0;
    if (r0 == 0.0) {
        rep->status = KRY_STATUS_CONVERGED;
        if (x_out) memcpy(x_out, x, (size_t)n * sizeof(double));
        free(x), free(r);
        return KRY_OK;
    }
    orc_store* st = NULL;
    int rc = orc_store_create(n, m, s, shat, &st);
    if (rc) {
        free(x), free(r);
        return rc;
    }
    solver_t S = {a, b, &cfg, st, x, r, r0, rep};
    int done = 0, strikes = 0;
    const I blocks = m / s;
    double* v1 = dz(n);
    double* V = dz(n * (s + 1));
    check_t ck;
    while (!done) {
        const double gamma = norm2(r, n);
        if (gamma / r0 <= cfg.rel_tol) {
            rep->status = KRY_STATUS_CONVERGED;
            break;
        }
        if (rep->iterations >= cfg.max_iters) {
            rep->status = KRY_STATUS_MAX_ITERS;
            break;
        }
        store_reset(st);
        for (I i = 0; i < n; ++i) v1[i] = r[i] / gamma;
        if (standard) { /* seed_unit_column :97-104 */
            memcpy(st->q, v1, (size_t)n * sizeof(double));
            R_(st, 0, 0) = 1.0;
            st->filled = st->finalized = st->bps = 1;
        }
        int updated = 0;
        for (I j = 0; j < blocks && !done; ++j) {
            kry_append_outcome oc;
            I red = 0;
            if (standard) {
                spmv(a, st->q + (st->filled - 1) * n, V);
                rc = append(st, V, 1, 0, cfg.scheme_kind, &oc, &red);
            } else {
                const double* start = (j == 0) ? v1 : st->q + (st->filled - 1) * n;
                mpk(a, start, s, V);
                rc = append(st, V, s + 1, j != 0, two ? KRY_ORTHO_TWO_STAGE : cfg.scheme_kind, &oc, &red);
            }
            if (rc) goto out;
            rep->reduces += red;
            push_i64(rep->per_block, rep->per_block_cap, &rep->n_per_block, red);
            rep->iterations += s;
            if (oc.breakdown || oc.truncated) {
                rep->breakdown = 1;
                rep->breakdown_kappa = oc.kappa_estimate;
                if (two && st->filled > st->bps) {
                    kry_append_outcome fo;
                    I fr = 0;
                    int pushed = 0;
                    finalize(st, &fo, &fr, &pushed);
                    rep->reduces += fr;
                    if (pushed) push_i64(rep->per_big_panel, rep->per_big_panel_cap, &rep->n_per_big_panel, fr);
                }
                if ((rc = check_and_update(&S, gamma, 1, &ck))) goto out;
                updated = 1;
                rep->status = ck.explicit_rel <= cfg.rel_tol ? KRY_STATUS_CONVERGED : KRY_STATUS_ORTHO_BREAKDOWN;
                done = 1;
                break;
            }
            if (two) {
                const int last_block = (j + 1 == blocks);
                const int full = st->filled > st->bps && st->filled - st->bps >= st->shat + 1;
                if (full || last_block) {
                    kry_append_outcome fo;
                    I fr = 0;
                    int pushed = 0;
                    finalize(st, &fo, &fr, &pushed);
                    rep->reduces += fr;
                    if (pushed) push_i64(rep->per_big_panel, rep->per_big_panel_cap, &rep->n_per_big_panel, fr);
                    if (fo.breakdown) {
                        rep->breakdown = 1;
                        rep->breakdown_kappa = fo.kappa_estimate;
                        if ((rc = check_and_update(&S, gamma, 1, &ck))) goto out;
                        updated = 1;
                        rep->status =
                            ck.explicit_rel <= cfg.rel_tol ? KRY_STATUS_CONVERGED : KRY_STATUS_ORTHO_BREAKDOWN;
                        done = 1;
                        break;
                    }
                } else {
                    continue;
                }
            }
            if ((rc = check_and_update(&S, gamma, 0, &ck))) goto out;
            if (ck.implicit_crossed) {
                updated = 1;
                if (ck.explicit_rel <= cfg.rel_tol) {
                    rep->status = KRY_STATUS_CONVERGED;
                    done = 1;
                } else {
                    break;
                }
            }
        }
        if (!updated && (rc = check_and_update(&S, gamma, 1, &ck))) goto out;
        const double rnorm = norm2(r, n);
        if (rep->n_cycle_residuals < rep->cycle_residuals_cap) rep->cycle_residuals[rep->n_cycle_residuals] = rnorm / r0;
        ++rep->n_cycle_residuals;
        if (done) break;
        ++rep->restarts;
        if (rnorm / r0 <= cfg.rel_tol) {
            rep->status = KRY_STATUS_CONVERGED;
            break;
        }
        if (rnorm > 0.99 * gamma) {
            if (++strikes >= 2) {
                rep->status = KRY_STATUS_STAGNATION;
                break;
            }
        } else {
            strikes = 0;
        }
    }
    rep->final_relative_residual = norm2(r, n) / r0;
    if (rep->iterations > 0) rep->reduces_per_iteration = (double)rep->reduces / (double)rep->iterations;
    if (x_out) memcpy(x_out, x, (size_t)n * sizeof(double));
    rc = KRY_OK;
out:
    rep->wall_seconds = (double)(clock() - t0) / CLOCKS_PER_SEC;
    orc_store_destroy(st);
    free(x), free(r), free(v1), free(V);
    return rc;
}

int orc_sstep_gmres(I n, const I* rp, const I* ci, const double* v, const double* b, const double* x0,
                    const kry_solver_config* cfg, kry_report* rep, double* x_out) {
    csr_t a = {n, rp, ci, v};
    return gmres_impl(&a, b, x0, cfg, 0, rep, x_out);
}

int orc_standard_gmres(I n, const I* rp, const I* ci, const double* v, const double* b, const double* x0,
                       const kry_solver_config* cfg, kry_report* rep, double* x_out) {
    csr_t a = {n, rp, ci, v};
    return gmres_impl(&a, b, x0, cfg, 1, rep, x_out);
}
