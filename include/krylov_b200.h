/*
 * krylov_b200.h — C ABI of the B200-native s-step GMRES hot path.
 *
 * This is the drop-in boundary for the hot path of the CPU reference
 * (/root/reference/proj/include/krylov): the solver entry, the block
 * orthogonalization entries, the basis store and the operator/MPK.  Every
 * entry point takes plain pointers and sizes (no C++ or torch types),
 * never throws, and returns a status code that maps 1:1 onto the
 * reference's exception types (types.hpp).  `include/krylov_b200/krylov.hpp`
 * rebuilds the reference's C++ API (names, value semantics, exceptions) on
 * top of this header; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Dense matrices are column-major.  Host-side views use ld == rows, like
 *    krylov::ConstMatrixView (dense_matrix.hpp:13-38).  Device-side entry
 *    points (suffix _device) take an explicit leading dimension.
 *  - Sizes are int64_t (the reference's index_t is size_t, types.hpp:9).
 *  - In a multi-GPU context (nranks > 1) every vector argument holds the
 *    calling rank's contiguous block of rows [row_begin, row_end) of the
 *    operator; small matrices (R, H, y) are replicated on every rank.
 *  - The library never falls back to the CPU: without a usable sm_100 device
 *    every compute entry returns KRY_NO_DEVICE.
 */
#ifndef KRYLOV_B200_H
#define KRYLOV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRY_ABI_VERSION 2

/* ---- status codes (reference exceptions, types.hpp) -------------------- */
enum kry_status {
    KRY_OK = 0,
    KRY_DIMENSION_MISMATCH = 1,    /* krylov::DimensionMismatch     types.hpp:11  */
    KRY_NOT_POSITIVE_DEFINITE = 2, /* krylov::NotPositiveDefinite   types.hpp:20 (pivot out-param, 1-based) */
    KRY_SINGULAR_FACTOR = 3,       /* krylov::SingularFactor        types.hpp:29  */
    KRY_SINGULAR_R = 4,            /* krylov::SingularR             types.hpp:34 (column out-param) */
    KRY_INVALID_ARGUMENT = 5,      /* std::invalid_argument         gmres.hpp:34  */
    KRY_UNSUPPORTED = 6,           /* a configuration this build does not implement */
    KRY_CUDA_ERROR = 7,
    KRY_NCCL_ERROR = 8,
    KRY_NO_DEVICE = 9,
    KRY_INTERNAL = 10
};

/* krylov::OrthoKind (block_ortho.hpp:23) */
enum kry_ortho_kind {
    KRY_ORTHO_BCGS2_HHQR = 0,
    KRY_ORTHO_BCGS2_CHOLQR2 = 1,
    KRY_ORTHO_BCGS_PIP2 = 2,
    KRY_ORTHO_TWO_STAGE = 3
};

/* krylov::SolveStatus (gmres.hpp:51) */
enum kry_solve_status {
    KRY_STATUS_CONVERGED = 0,
    KRY_STATUS_MAX_ITERS = 1,
    KRY_STATUS_ORTHO_BREAKDOWN = 2,
    KRY_STATUS_STAGNATION = 3
};

/* krylov::PanelState (basis_store.hpp:14) */
enum kry_panel_state { KRY_PANEL_RAW = 0, KRY_PANEL_PREPROCESSED = 1, KRY_PANEL_FINAL = 2 };

/* krylov::SolverConfig (gmres.hpp:18-36) + OrthoScheme (block_ortho.hpp:28-31) */
typedef struct kry_solver_config {
    int64_t restart_len;           /* m   (default 60)                 */
    int64_t step;                  /* s   (default 5)                  */
    int64_t big_step;              /* ŝ   (0 → m)                      */
    int32_t scheme_kind;           /* enum kry_ortho_kind (default PIP2) */
    int32_t reserved0;
    int64_t scheme_big_panel_size; /* OrthoScheme::big_panel_size      */
    double rel_tol;                /* default 1e-6                      */
    int64_t max_iters;             /* default 500000                    */
} kry_solver_config;

/* krylov::AppendOutcome (basis_store.hpp:16-22) */
typedef struct kry_append_outcome {
    int64_t committed;
    int32_t truncated;
    int32_t breakdown;
    int64_t pivot;
    double kappa_estimate;
} kry_append_outcome;

/* krylov::SolveReport (gmres.hpp:63-76) plus device telemetry.  The three
 * arrays are caller-owned (may be NULL with capacity 0); the n_* counts are
 * always the full counts, so a caller can size a second call. */
typedef struct kry_report {
    int32_t status;                /* enum kry_solve_status */
    int32_t breakdown;
    int64_t iterations;
    int64_t restarts;
    double initial_residual;
    double final_relative_residual;
    double breakdown_kappa;
    int64_t reduces;               /* SyncCounter::reduces */
    double reduces_per_iteration;
    double wall_seconds;

    double* cycle_residuals;
    int64_t cycle_residuals_cap;
    int64_t n_cycle_residuals;
    int64_t* per_block;            /* SyncCounter::per_block     */
    int64_t per_block_cap;
    int64_t n_per_block;
    int64_t* per_big_panel;        /* SyncCounter::per_big_panel */
    int64_t per_big_panel_cap;
    int64_t n_per_big_panel;

    /* ---- telemetry (zero unless kry_ctx_set_timing(ctx, 1)) ----------
     * Seconds are summed CUDA-event intervals on the solver stream; bytes
     * are the algorithmic bytes of DESIGN.md §4 for this rank's rows. */
    double mpk_seconds;            /* all SpMV / stencil applications in MPK blocks */
    double ortho_seconds;          /* BlkOrtho: Gram + allreduce + Cholesky + update */
    double gram_kernel_seconds;    /* fused Gram kernel only */
    double update_kernel_seconds;  /* fused basis-update kernel only */
    double restart_seconds;        /* residual, x update, norms */
    double mpk_bytes;
    double ortho_bytes;
    double gram_bytes;
    double update_bytes;
    int64_t gram_launches;
    int64_t update_launches;
    int64_t gpu_launches;          /* every kernel this library launched */
    int64_t allreduces;            /* device collectives issued (Gram + norms) */
    double fused_kernel_seconds;   /* fused first-stage pass (update → MPK → Gram), k_fused.cu */
    double fused_bytes;            /* its necessary HBM bytes: prefix + raw block read, 2 blocks written */
    int64_t fused_launches;
} kry_report;

/* ---- library ------------------------------------------------------------ */
int kry_abi_version(void);
const char* kry_last_error(void);       /* thread-local message of the last failure */
const char* kry_status_name(int status);
void kry_solver_config_default(kry_solver_config* cfg);

/* ---- context: one device, one stream, optional NCCL communicator --------- */
typedef struct kry_ctx kry_ctx;
int kry_device_count(int* count);
int kry_nccl_unique_id_size(void);                 /* bytes (128) */
int kry_nccl_get_unique_id(void* out);             /* call on rank 0, broadcast the bytes */
int kry_ctx_create(int device, int nranks, int rank, const void* nccl_unique_id, kry_ctx** out);
int kry_ctx_destroy(kry_ctx* ctx);
int kry_ctx_synchronize(kry_ctx* ctx);
int kry_ctx_set_timing(kry_ctx* ctx, int enabled);
int kry_ctx_launch_count(kry_ctx* ctx, int64_t* launches);
int kry_ctx_rank(kry_ctx* ctx, int* rank, int* nranks);
/* The cudaStream_t every kernel of this context is launched on (for event timing). */
int kry_ctx_stream(kry_ctx* ctx, void** stream);

/* ---- operators (krylov::CsrMatrix csr_matrix.hpp:17-65, spmv :69-79) ----- */
typedef struct kry_operator kry_operator;
/* CSR rows [row_begin, row_begin + n_local) of an n_global×n_global matrix.
 * row_ptr has n_local+1 entries starting at 0; col_idx are global columns,
 * strictly increasing per row (CsrMatrix::validate, csr_matrix.hpp:25-38). */
int kry_operator_create_csr(kry_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t n_local,
                            const int64_t* row_ptr, const int64_t* col_idx, const double* vals,
                            kry_operator** out);
/* Matrix-free operators bit-identical to gen_laplace2d(nx, ny, 5) and
 * gen_laplace3d(nx, ny, nz) (matgen.hpp:134-187).  Rows are partitioned by
 * whole grid lines (2D) / planes (3D) across the context's ranks. */
int kry_operator_create_laplace2d(kry_ctx* ctx, int64_t nx, int64_t ny, kry_operator** out);
int kry_operator_create_laplace3d(kry_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, kry_operator** out);
/* Host-only: the rows a rank owns under the matrix-free operators' partition
 * (whole grid lines in 2D, whole planes in 3D; dims = 2 or 3, nz ignored for
 * 2D) and the halo length it exchanges with each neighbour.  No device use. */
int kry_laplace_partition(int dims, int64_t nx, int64_t ny, int64_t nz, int nranks, int rank, int64_t* row_begin,
                          int64_t* n_local, int64_t* halo);
int kry_operator_destroy(kry_operator* op);
int kry_operator_rows(const kry_operator* op, int64_t* n_global, int64_t* row_begin, int64_t* n_local);
int kry_operator_nnz(const kry_operator* op, int64_t* nnz_local);
/* Left Jacobi preconditioning (the reference has no
 * preconditioner hook, gmres.hpp:80-90).  From this call on the
 * operator is D⁻¹A, D = diag(A): the CSR values are divided by their row's
 * diagonal in place on the device (IEEE division, so the operator is
 * bit-identical to a host pre-scaling a_ij / a_ii), kry_spmv/kry_mpk apply
 * D⁻¹A, and the solvers take the ORIGINAL b and solve D⁻¹A x = D⁻¹b (D⁻¹b
 * formed on the device; residual histories are those of the scaled
 * system, exactly what the reference reports when handed D⁻¹A and D⁻¹b).
 * Irreversible; calling it twice is a no-op.  KRY_INVALID_ARGUMENT if a row
 * has no (or a zero) diagonal entry; KRY_UNSUPPORTED for the matrix-free
 * Laplacians unless built with stencil Jacobi. */
int kry_operator_jacobi(kry_operator* op);
int kry_operator_is_jacobi(const kry_operator* op, int* enabled);
/* Host-only generator of the BASELINE configs[4] workload: rows
 * [row_begin, row_begin + n_local) of an n_global×n_global nonsymmetric
 * random sparse matrix with per_row entries per row (the diagonal and
 * per_row − 1 distinct random columns), built on the reference's SplitMix64
 * (rng.hpp:19-42) — a function of (n_global, per_row, seed, diag_factor)
 * only, whatever the rank layout.  Off-diagonal values uniform in [−1, 1),
 * a_ii = 1 + diag_factor·Σ|a_ij| (diag_factor 0.15: GMRES(60) restarts
 * 5-6 times at tol 1e-6); jacobi != 0 returns D⁻¹A instead.  row_ptr has
 * n_local+1 entries from 0 (row_ptr[i] = i·per_row), col_idx/vals
 * n_local·per_row, ascending columns per row.  Multithreaded.  The numpy
 * restatement is oracle/randsparse.py. */
int kry_gen_random_sparse(int64_t n_global, int64_t row_begin, int64_t n_local, int64_t per_row, uint64_t seed,
                          double diag_factor, int jacobi, int64_t* row_ptr, int64_t* col_idx, double* vals);
/* y = A·x for this rank's rows (spmv, csr_matrix.hpp:69). Host buffers. */
int kry_spmv(kry_ctx* ctx, kry_operator* op, const double* x, double* y);
/* Device buffers (ld irrelevant: vectors). */
int kry_spmv_device(kry_ctx* ctx, kry_operator* op, const double* d_x, double* d_y);
/* V = mpk_monomial(A, start, s) (gmres.hpp:80-90): V is n_local×(s+1). */
int kry_mpk(kry_ctx* ctx, kry_operator* op, const double* start, int64_t s, double* v);

/* ---- block orthogonalization (block_ortho.hpp) — host views ---------------
 * q_prev: n×c0 (may be NULL when c0 == 0), v: n×w.  Outputs: q n×w,
 * r_col c0×w, r_jj w×w (upper, col-major).  `reduces` (nullable) is
 * incremented exactly like SyncCounter::add. */
int kry_gram(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
             double* r_col, double* g);    /* [Q_prev V]ᵀV: r_col = Q_prevᵀV, g = VᵀV (full, mirrored) */
int kry_bcgs_pip_partial(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v,
                         int64_t w, double* q, double* r_col, double* r_chol, int64_t* bad_pivot,
                         int64_t* reduces);                                  /* block_ortho.hpp:152 */
int kry_bcgs_pip(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                 double* q, double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces); /* :180 */
int kry_bcgs_pip2(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                  double* q, double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces); /* :192 */
int kry_cholqr(kry_ctx* ctx, int64_t n, const double* v, int64_t w, double* q, double* r,
               int64_t* pivot, int64_t* reduces);                            /* :49 */
/* The BCGS2 baseline pieces (block_ortho.hpp:57-137):
 * cholqr2 = CholQR twice, R = R₂·R₁ (2 reduces); bcgs_project: r_block =
 * Q_prevᵀV (c0×w), vhat = V − Q_prev·r_block (1 reduce, 0 when c0 == 0);
 * bcgs2 = project, intra (CholQR2, or CholQR for one column), re-project,
 * CholQR.  intra_kind: 1 = CholQR2 (IntraKind::Cholqr2); 0 = HHQR is
 * KRY_UNSUPPORTED for w > 1 (not on the device path).  A failed Cholesky
 * returns KRY_NOT_POSITIVE_DEFINITE with its pivot. */
int kry_cholqr2(kry_ctx* ctx, int64_t n, const double* v, int64_t w, double* q, double* r,
                int64_t* pivot, int64_t* reduces);                           /* :57 */
int kry_bcgs_project(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
                     double* vhat, double* r_block, int64_t* reduces);       /* :70 */
int kry_bcgs2(kry_ctx* ctx, int64_t n, const double* q_prev, int64_t c0, const double* v, int64_t w,
              int32_t intra_kind, double* q, double* r_col, double* r_jj, int64_t* pivot,
              int64_t* reduces);                                            /* :102 */
/* Device views with explicit leading dimensions; out may alias v. */
int kry_bcgs_pip_device(kry_ctx* ctx, int64_t n, const double* d_q_prev, int64_t ldq, int64_t c0,
                        const double* d_v, int64_t ldv, int64_t w, double* d_out, int64_t ldo,
                        double* r_col, double* r_jj, int64_t* pivot, int64_t* reduces);
/* ‖I − QᵀQ‖-style diagnostics need the Gram of Q: G = QᵀQ (k×k, host). */
int kry_gram_full(kry_ctx* ctx, int64_t n, const double* q, int64_t k, double* g);

/* ---- basis store (krylov::BasisStore basis_store.hpp:42-401) -------------- */
typedef struct kry_store kry_store;
int kry_store_create(kry_ctx* ctx, int64_t n, int64_t m, int64_t panel_size, int64_t big_panel_size,
                     kry_store** out);                                      /* :44-55 */
int kry_store_destroy(kry_store* st);
int kry_store_reset(kry_store* st);                                          /* :84-93 */
int kry_store_seed_unit_column(kry_store* st, const double* v);              /* :97-104 */
int kry_store_append_block(kry_store* st, const double* v, int64_t w, int overlap, int32_t scheme_kind,
                           int64_t big_panel_size, kry_append_outcome* out,
                           int64_t* reduces_delta);                          /* :112-118 */
int kry_store_preprocess_block(kry_store* st, const double* v, int64_t w, int overlap,
                               kry_append_outcome* out, int64_t* reduces_delta); /* :122-125 */
int kry_store_finalize_big_panel(kry_store* st, kry_append_outcome* out,
                                 int64_t* reduces_delta);                    /* :131-166 */
/* MPK straight into the store: start = column filled-1 (or `start` when
 * non-NULL, written to column `c0`), columns c0+1..c0+s = A^k·start. */
int kry_store_mpk(kry_store* st, kry_operator* op, const double* start, int64_t c0, int64_t s);
/* Append the block that kry_store_mpk left in columns [c0, c0+w) in place. */
int kry_store_append_inplace(kry_store* st, int64_t w, int overlap, int32_t scheme_kind,
                             int64_t big_panel_size, kry_append_outcome* out, int64_t* reduces_delta);

typedef struct kry_store_info {
    int64_t rows, capacity, filled, finalized, big_panel_start, panel_size, big_panel_size;
    int32_t seam_valid;        /* has_seam_column() */
    int32_t big_panel_open;    /* :75 */
    int32_t big_panel_full;    /* :76-78 */
    int32_t reserved0;
    int64_t n_records;
    int64_t n_panel_states;
    int64_t ld;                /* device leading dimension of Q */
} kry_store_info;
int kry_store_get_info(kry_store* st, kry_store_info* info);
int kry_store_coefficients(kry_store* st, double* r);          /* (m+1)×(m+1), col-major */
int kry_store_column(kry_store* st, int64_t j, double* out);   /* host copy of column j  */
int kry_store_columns(kry_store* st, int64_t first, int64_t count, double* out); /* n×count */
int kry_store_panel_states(kry_store* st, int32_t* states);    /* n_panel_states entries */
/* BlockRecord (basis_store.hpp:28-34): carried has c0 entries. */
int kry_store_block_record(kry_store* st, int64_t index, int64_t* c0, int64_t* width, int32_t* overlap,
                           double* carried, double* carried_diag);
int kry_store_device_ptr(kry_store* st, double** d_q, int64_t* ld);
/* Debug (KRY_GUARD=1 at store creation): KRY_INTERNAL if any kernel wrote the
 * store's guard columns or padding rows [n, ld); KRY_OK otherwise, or when
 * the store was created without guards. */
int kry_store_check_guards(kry_store* st);

/* ---- restart-loop pieces (gmres.hpp:100-185), host arithmetic ------------- */
/* H ((k+1)×k, col-major) from the store's R and records (assemble_hessenberg). */
int kry_store_hessenberg(kry_store* st, int64_t k, double* h, int64_t* singular_column);
/* solve_hessenberg_lsq: y has k entries (valid_cols are set). */
int kry_hessenberg_lsq(int64_t k, const double* h, double gamma, double* y, double* implicit_residual,
                       int64_t* valid_cols);
/* try_cholesky (dense_kernels.hpp:111): returns KRY_OK and *pivot (0 or 1-based). */
int kry_try_cholesky(int64_t k, const double* s, double* r, int64_t* pivot);

/* ---- the solver (sstep_gmres gmres.hpp:396, standard_gmres :404) ---------- */
int kry_sstep_gmres(kry_ctx* ctx, kry_operator* op, const double* b, const double* x0,
                    const kry_solver_config* cfg, kry_report* report, double* x_out);
int kry_standard_gmres(kry_ctx* ctx, kry_operator* op, const double* b, const double* x0,
                       const kry_solver_config* cfg, kry_report* report, double* x_out);
/* Inputs already resident in HBM (d_x0 may be NULL; d_x_out may be NULL). */
int kry_sstep_gmres_device(kry_ctx* ctx, kry_operator* op, const double* d_b, const double* d_x0,
                           const kry_solver_config* cfg, kry_report* report, double* d_x_out);
int kry_standard_gmres_device(kry_ctx* ctx, kry_operator* op, const double* d_b, const double* d_x0,
                              const kry_solver_config* cfg, kry_report* report, double* d_x_out);

#ifdef __cplusplus
}
#endif
#endif /* KRYLOV_B200_H */
