/*
 * krylov_oracle.h — TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * Plain-C restatement of the CPU reference's hot path
 * (/root/reference/proj/include/krylov: csr_matrix.hpp, dense_kernels.hpp,
 * block_ortho.hpp, basis_store.hpp, gmres.hpp, spectral.hpp) used as the
 * parity checker.  Every routine performs the reference's floating-point
 * operations in the reference's order, so — compiled without FMA contraction
 * like the reference's Release build — its results are bit-identical to the
 * reference's (pinned by tests/test_oracle.py against tests/golden/ and the
 * live reference in oracle/_ref).  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs may call it.
 *
 * Matrices are column-major with ld == rows.  Structs are shared with the
 * product header (include/krylov_b200.h) so reports compare field by field.
 */
#ifndef KRYLOV_ORACLE_H
#define KRYLOV_ORACLE_H

#include <stdint.h>

#include "../include/krylov_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* return codes: the KRY_* status codes; *aux receives a pivot/column */
const char* orc_last_error(void);

/* generators (matgen.hpp) — CSR with int64 indices; call with NULL arrays to get sizes */
int orc_laplace2d(int64_t nx, int64_t ny, int64_t* n, int64_t* nnz, int64_t* rp, int64_t* ci, double* v);
int orc_laplace3d(int64_t nx, int64_t ny, int64_t nz, int64_t* n, int64_t* nnz, int64_t* rp, int64_t* ci, double* v);

/* kernels */
int orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x, double* y);
int orc_mpk(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* start, int64_t s,
            double* out);
int orc_gram(int64_t n, int64_t k, const double* v, double* g);
int orc_try_cholesky(int64_t k, const double* s, double* r, int64_t* pivot);

/* block orthogonalization; *reduces += SyncCounter increments; *pivot = failing pivot */
int orc_bcgs_pip_partial(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* q,
                         double* r_col, double* r_chol, int64_t* bad_pivot, int64_t* reduces);
int orc_bcgs_pip(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* q, double* r_col,
                 double* r_jj, int64_t* pivot, int64_t* reduces);
int orc_bcgs_pip2(int64_t n, const double* qp, int64_t c0, const double* v, int64_t w, double* q, double* r_col,
                  double* r_jj, int64_t* pivot, int64_t* reduces);

/* basis store */
typedef struct orc_store orc_store;
int orc_store_create(int64_t n, int64_t m, int64_t s, int64_t shat, orc_store** out);
void orc_store_destroy(orc_store* st);
int orc_store_append_block(orc_store* st, const double* v, int64_t w, int overlap, int32_t kind,
                           kry_append_outcome* out, int64_t* reduces_delta);
int orc_store_preprocess_block(orc_store* st, const double* v, int64_t w, int overlap, kry_append_outcome* out,
                               int64_t* reduces_delta);
int orc_store_finalize_big_panel(orc_store* st, kry_append_outcome* out, int64_t* reduces_delta);
int orc_store_get_info(orc_store* st, kry_store_info* info);
int orc_store_coefficients(orc_store* st, double* r);
int orc_store_columns(orc_store* st, int64_t first, int64_t count, double* out);
int orc_store_hessenberg(orc_store* st, int64_t k, double* h, int64_t* singular_column);
int orc_hessenberg_lsq(int64_t k, const double* h, double gamma, double* y, double* implicit, int64_t* valid);

/* solvers */
int orc_sstep_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b,
                    const double* x0, const kry_solver_config* cfg, kry_report* rep, double* x_out);
int orc_standard_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b,
                       const double* x0, const kry_solver_config* cfg, kry_report* rep, double* x_out);

#ifdef __cplusplus
}
#endif
#endif
