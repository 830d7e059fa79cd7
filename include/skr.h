/* skr.h — C-ABI of the B200-native hot path for skridge (arXiv 1602.02350).
 *
 * This is the drop-in boundary: plain pointers, sizes and int status codes, no
 * C++ or torch types.  Each entry point names the reference interface it
 * replaces (paths relative to the reference's proj/).  The reference's C++
 * callers keep their own types; include/skridge_b200.hpp is the header-only
 * C++ adapter that maps these calls back onto the reference's names and
 * exception types (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - A data matrix is passed as n x d ROW-major (point i = row i).  That is
 *    byte-identical to the reference's d x n column-major DenseMatrix
 *    (dense_matrix.hpp:12-15), so a reference DataMatrix's storage can be
 *    handed over without transposition.
 *  - Dense factors (U, V) are COLUMN-major like DenseMatrix: U is d x k with
 *    basis vector j at U + j*d.
 *  - Host pointers unless the name says _device.  Outputs go to caller-owned
 *    memory.  Vectors are double regardless of the data dtype.
 *  - Every call returns SKR_OK or an error code; skr_last_error() gives the
 *    message (thread-local).  Error codes map 1:1 onto the reference's
 *    exception types (errors.hpp:10-60, svrg.hpp:27-35).
 *  - All work is ordered on the context's CUDA stream; calls on one context
 *    must be serialised by the caller (the reference is single-threaded on
 *    this path).
 */
#ifndef SKR_H
#define SKR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKR_ABI_VERSION 1

typedef enum {
  SKR_OK = 0,
  SKR_EDIM = 1,       /* DimensionError      (errors.hpp:10) */
  SKR_EPARAM = 2,     /* ParameterError      (errors.hpp:16) */
  SKR_EINPUT = 3,     /* InputError          (errors.hpp:22) */
  SKR_EGUARD = 4,     /* ScaleGuardError     (errors.hpp:34) */
  SKR_EDIVERGED = 5,  /* DivergenceError     (svrg.hpp:27-35) */
  SKR_ECUDA = 6,      /* CUDA runtime / library failure (new: DeviceError) */
  SKR_ENCCL = 7,      /* NCCL failure (new: DeviceError) */
  SKR_EEMPTY = 8,     /* EmptyBasisError     (errors.hpp:28) */
  SKR_ENOMEM = 9,     /* device allocation failed */
  SKR_EINTERNAL = 10
} skr_status;

typedef enum { SKR_F64 = 0, SKR_F32 = 1 } skr_dtype;

typedef struct skr_ctx skr_ctx;         /* one per process and GPU */
typedef struct skr_data skr_data;       /* DataMatrix (data_matrix.hpp:18-61) */
typedef struct skr_problem skr_problem; /* PreconditionedRidge (ridge.hpp:78-119) */

const char* skr_last_error(void);
int skr_abi_version(void);

/* ---- context ----------------------------------------------------------- */
int skr_ctx_create(int device, skr_ctx** out);
/* NCCL bootstrap for row sharding across ranks (one process per GPU). */
int skr_nccl_unique_id(char id_out[128]);
int skr_ctx_create_dist(int device, int rank, int world, const char id[128], skr_ctx** out);

/* Row sharding of the distributed path (host only, no device needed).
 * skr_shard_rows: the shard skr_data_generate gives `rank` of `world` for n rows:
 *   n_local = n / world + (rank < n % world), row0 = rank * (n / world) + min(rank, n % world).
 * skr_shard_layout: (n_global, row0) of `rank` from every rank's local row count in rank
 *   order (skr_data_create gathers the counts; shards are concatenated in rank order). */
int skr_shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* n_local);
int skr_shard_layout(const int64_t* counts, int world, int rank, int64_t* n_global, int64_t* row0);
int skr_ctx_destroy(skr_ctx* ctx);
int skr_ctx_synchronize(skr_ctx* ctx);
/* Buffers of 1 GiB and more are parked on release for the next request of the
 * same size (cudaFree of a multi-GiB mapping stalls the host); at most 80 GiB per
 * GPU, given back whenever an allocation would otherwise fail and on
 * skr_ctx_destroy.  skr_ctx_trim returns them to the driver now, together with the
 * unused part of the device's stream-ordered pool; bytes_released (may be NULL)
 * counts the parked buffers. */
int skr_ctx_trim(skr_ctx* ctx, int64_t* bytes_released);
void* skr_ctx_stream(skr_ctx* ctx); /* cudaStream_t the context orders work on */
/* number of this library's kernel launches so far on the context */
int64_t skr_ctx_kernel_launches(const skr_ctx* ctx);
/* CUDA-event timing of the hot kernels on the context stream: enable (resets
 * the counters) and read the summed device time of a key ("fullgrad": the K9
 * streaming kernel; "svrg_epoch": the K10 inner loop). */
int skr_ctx_profile(skr_ctx* ctx, int enable);
int skr_ctx_profile_read(skr_ctx* ctx, const char* key, double* total_ms, int64_t* launches);
/* cap the grid of the SVRG inner loop's PREP kernel (blocks are grid-strided);
 * 0 = one CTA per block (default).  Concurrent chains on one GPU (the eta-grid
 * protocol of bench.cpp:140-193, one context per lane) keep SMs for each
 * other's clusters this way. */
int skr_ctx_set_prep_cap(skr_ctx* ctx, int ctas);

/* ---- data: DataMatrix (data_matrix.hpp:18-61) -------------------------- */
/* rows: n x d row-major host array of `dtype`.  On a distributed context the
 * caller passes its LOCAL row shard; n_global/row0 describe the global layout
 * (skr_data_create passes n_global = sum of shards via an allreduce). */
int skr_data_create(skr_ctx* ctx, const void* rows, int64_t n, int64_t d, int dtype,
                    skr_data** out);
/* same, but the rows already live in device memory (ld = row stride in elements) */
/* DataMatrix(SparseMatrix) (data_matrix.hpp:24; sparse_matrix.hpp:12-14): this
 * rank's points as CSR — byte-identical to the reference's CSC over points —
 * row_ptr (n+1), strictly increasing col_idx (< d) per row, finite nonzero values.
 * Sparse handles go through block_lanczos, the preconditioned problem (Lazy mode:
 * X~ is never materialised), SVRG, the objective, reference_minimum and the
 * Gram-based diagnostics; skr_data_download is dense-only. */
int skr_data_create_csr(skr_ctx* ctx, int64_t n, int64_t d, const int64_t* row_ptr, const int32_t* col_idx,
                        const double* vals, skr_data** out);
int skr_data_is_sparse(const skr_data* x, int* sparse, int64_t* nnz);
int skr_data_create_device(skr_ctx* ctx, const void* dev_rows, int64_t ld, int64_t n,
                           int64_t d, int dtype, skr_data** out);
/* DataMatrix::scaled (data_matrix.cpp:56-61): shares storage, scale *= factor */
int skr_data_scaled(const skr_data* src, double factor, skr_data** out);
int skr_data_info(const skr_data* x, int64_t* n, int64_t* d, int* dtype, double* scale,
                  int64_t* n_global, int64_t* row0);
int skr_data_download(const skr_data* x, void* rows_out); /* local n x d, dtype */
int skr_data_destroy(skr_data* x);

/* Synthetic BASELINE instance generated on the device:
 * X = G diag(sigma) V^T (G iid N(0,1) by Philox4x32-10, V Haar), optional
 * |Student-t(3)| row scaling, y = X w* + tau N(0,1).  Labels are returned on the
 * device inside the data handle and fetched with skr_data_labels. */
typedef struct {
  int64_t n, d;
  int dtype;            /* SKR_F64 or SKR_F32 */
  uint64_t seed;
  int spectrum;         /* 0: 1/j, 1: r^j, 2: j^-p, 3: 1/j (j<=50) and 0.02/j beyond */
  double spectrum_param;/* r (kind 1) or p (kind 2) */
  int t_scale;          /* 1: multiply each row by |t_3| */
  double tau;           /* label noise */
} skr_synth_spec;
int skr_data_generate(skr_ctx* ctx, const skr_synth_spec* spec, skr_data** out);
int skr_data_labels(const skr_data* x, double* y_out); /* generated labels (local rows) */

/* ---- block_lanczos (sketch.hpp:55, sketch.cpp:41-90) ------------------- */
/* A is the (scaled) data handle, e.g. skr_data_scaled(X, 1/sqrt(n)) for
 * scaled_design (ridge.cpp:54-56).  q <= 0 -> lanczos_iterations(n, eps_prime).
 * U: d x k col-major; sigma: k; V (nullable): n_local x k col-major. */
int skr_lanczos(skr_ctx* ctx, const skr_data* A, int64_t k, int64_t q, double eps_prime,
                uint64_t seed, double* U, double* sigma, double* V, int64_t* k_used,
                int64_t* q_used, int* rank_reduced);

/* ---- preconditioned_components (ridge.hpp:121-123, ridge.cpp:93-150) ----
 * Builds build_sketched(sv, lambda) (precond.cpp:120-136) from (U, sigma, k)
 * — k == 0 means Preconditioner::identity (precond.cpp:51-60) — then the
 * Dense-mode components: X~ = c X + (X U) diag(D - c) U^T, beta (N = n + d),
 * and the materialised regulariser rows B = P^{-1/2} (d x d).
 * y: n_local labels (double). */
int skr_problem_create(skr_ctx* ctx, const skr_data* X, const double* y, double lambda,
                       const double* U, const double* sigma, int64_t k, skr_problem** out);
/* Second handle on the same problem bound to another context (same device, one
 * GPU): X~ shared, tables copied, private workspaces — for concurrent SVRG chains
 * (the eta-grid x seed protocol of bench.cpp:140-193). */
int skr_problem_clone(const skr_problem* src, skr_ctx* ctx, skr_problem** out);
int skr_problem_destroy(skr_problem* p);
/* alpha = strong_convexity (ridge.cpp:152-157), beta_hat = mean_beta
 * (svrg.cpp:213-217), max_row_sq = max_i ||x~_i||^2 over data rows */
/* preconditioned_components(p, P, mode) (ridge.hpp:121-123) with the reference's
 * ApplyMode: SKR_MODE_DENSE materialises X~ (and, like ridge.cpp:110-113, raises
 * SKR_EGUARD above kDenseModeMaxEntries = 2e8 entries; sparse data are densified
 * on the device); SKR_MODE_LAZY keeps X and the k x n projections (sparse data as
 * is; dense data are converted to CSR over points, zeros dropped, one GPU);
 * SKR_MODE_AUTO is the device's own choice (Dense for dense data, which HBM
 * holds at every BASELINE size; Lazy for sparse) — ridge.cpp:104-109 picks by
 * n d <= 2e8 instead, for host memory; the two modes agree to ~1e-8
 * (test_ridge.cpp:272-291).  skr_problem_create == mode Auto. */
enum { SKR_MODE_DENSE = 0, SKR_MODE_LAZY = 1, SKR_MODE_AUTO = 2 };
int skr_problem_create_mode(skr_ctx* ctx, const skr_data* X, const double* y, double lambda, const double* U,
                            const double* sigma, int64_t k, int mode, skr_problem** out);
/* PreconditionedRidge::mode() (ridge.hpp:96): the mode the device problem runs in. */
int skr_problem_mode(const skr_problem* p, int* mode);
int skr_problem_info(const skr_problem* p, int64_t* n, int64_t* d, int64_t* k, double* alpha,
                     double* beta_hat, double* max_row_sq);
int skr_problem_betas(const skr_problem* p, double* out);          /* N = n_global + d */
int skr_problem_transformed(const skr_problem* p, void* rows_out); /* X~ local n x d, dtype */
/* PreconditionedRidge::objective (ridge.cpp:174-198) */
int skr_objective(skr_problem* p, const double* w, double* out);
/* PreconditionedRidge::full_gradient (ridge.cpp:200-236); fused with the
 * objective at the same w when obj != NULL (one pass over X~). */
int skr_full_gradient(skr_problem* p, const double* w, double* mu, double* obj);
/* device-pointer variant, asynchronous on the context stream (bench/kernel timing) */
int skr_full_gradient_device(skr_problem* p, const double* w_dev, double* mu_dev,
                             double* obj_dev);
/* PreconditionedRidge::component_gradient (ridge.cpp:238-278) */
int skr_component_gradient(skr_problem* p, int64_t i, const double* w, double* out);
/* Preconditioner::apply_inv_sqrt (precond.cpp:67-80) on the problem's preconditioner */
int skr_apply_inv_sqrt(skr_problem* p, const double* v, double* out);

/* ---- svrg (svrg.hpp:39-45,125-137; svrg.cpp:152-211) ------------------ */
typedef struct {
  int64_t epochs;       /* S */
  int64_t epoch_length; /* m */
  double step_size;     /* eta */
  uint64_t seed;
} skr_svrg_config;

typedef struct {
  int64_t epoch; /* 1-based */
  double objective;
  double suboptimality; /* NaN when no reference value */
  double elapsed_ms;
} skr_epoch_record;

/* One EpochState epoch (svrg.hpp:53-62) driven by caller-supplied indices
 * (replay of the reference engine's stream): w <- snapshot, m steps, w_avg. */
int skr_epoch(skr_problem* p, const double* snapshot, const double* mu, const int64_t* idx,
              int64_t m, double eta, double* w_avg);
/* GPU-native svrg_solve: identical index stream (device mt19937_64 +
 * lower_bound on the exact sequential cumulative table).  reference = NaN for
 * none.  On divergence returns SKR_EDIVERGED with the partial trace written. */
int skr_svrg(skr_problem* p, const skr_svrg_config* cfg, const double* w0, double reference,
             double* w_out, skr_epoch_record* trace, int64_t* epochs_done);
/* skr_svrg that stops after the first epoch whose suboptimality (objective -
 * reference) is <= target: the time-to-epsilon protocol of bench.cpp:182-189. */
int skr_svrg_until(skr_problem* p, const skr_svrg_config* cfg, const double* w0, double reference, double target,
                   double* w_out, skr_epoch_record* trace, int64_t* epochs_done);
/* the index stream skr_svrg would draw (test hook; `count` steps from seed) */
int skr_index_stream(skr_problem* p, uint64_t seed, int64_t count, int64_t* out);
/* make_cumulative_weights (svrg.cpp:90-106) on the device for a host table beta[N] (>= 0):
 * cum[i] = the reference's sequential fp64 running sum of beta_i / total (cum[N-1] = 1),
 * *total = its sequential sum.  sequential = 0: the block-scan form (what the solver
 * uses); 1: the one-thread chains.  Both are bit-identical to the reference loop.
 * SKR_EINPUT with the reference's messages for an empty table, a negative (or NaN)
 * weight and a zero total. */
int skr_cumulative_weights(skr_ctx* ctx, const double* beta, int64_t N, int sequential, double* cum, double* total);
/* NormalSampler(seed).uniform() x count from the device mt19937_64 (test hook) */
int skr_mt_uniforms(skr_ctx* ctx, uint64_t seed, int64_t count, double* out);
/* tcgen05 3xTF32 GEMM check: C (M x N fp64) = A (M x K fp32) . B (N x K fp32)^T (test hook) */
int skr_tc_gemm_test(skr_ctx* ctx, const float* A, const float* B, int64_t M, int64_t N, int64_t K, int splits,
                     double* C);
/* same with A given as its K x M row-major transpose (MN-major operand, the X^T products) (test hook) */
int skr_tc_gemm_mn_test(skr_ctx* ctx, const float* At, const float* B, int64_t M, int64_t N, int64_t K, int splits,
                        double* C);
/* gaussian_matrix(rows, cols, seed) on the device, column-major (random.cpp:28-41) */
int skr_gaussian_matrix(skr_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* out);

/* ---- diagnostics ------------------------------------------------------- */
/* dataset_spectrum (bench.cpp:205-212) on the UNSCALED data handle: eigenvalues of
 * X^T X / n, descending, zero past rank min(d, n); eigs has d entries.  The ratio
 * diagnostics over it (theoretical_ratio, avg_condition_number, run_ratio_curve)
 * are O(d) host arithmetic in skridge_b200.hpp. */
int skr_dataset_spectrum(skr_ctx* ctx, const skr_data* X, double* eigs);
/* sym_eigs(data.gram()) of the (scaled) data handle on the device, reference
 * conventions (factorize.cpp:87-165): evals descending (d), evecs d x d
 * column-major with eigenvector j in column j — the input of build_optimal
 * (precond.cpp:144-162). */
int skr_gram_eigs(skr_ctx* ctx, const skr_data* X, double* evals, double* evecs);
/* objective(p, w) of the ORIGINAL ridge problem (ridge.cpp:33-43) */
int skr_ridge_objective(skr_ctx* ctx, const skr_data* X, const double* y, double lambda,
                        const double* w, double* out);
/* reference_minimum (bench.cpp:84-94): SYRK + Cholesky on the device for d <= 5000
 * (kDirectSolveGuardDim, bench.cpp:19), the conjugate-gradient route of
 * reference_minimum_cg(p, 1e-12, 20 d) above it (bench.cpp:56-82). */
int skr_reference_minimum(skr_ctx* ctx, const skr_data* X, const double* y, double lambda,
                          double* w_out, double* min_out);
/* reference_minimum_cg (bench.hpp:26, bench.cpp:56-82) on the device: CG on
 * (Xb^T Xb + lambda I) w = X^T y / n from w = 0, stopping before the first
 * iteration with ||r|| <= rel_residual_tol ||rhs|| or after max_iterations;
 * *iterations (optional) = iterations run. */
int skr_reference_minimum_cg(skr_ctx* ctx, const skr_data* X, const double* y, double lambda,
                             double rel_residual_tol, int64_t max_iterations, double* w_out, int64_t* iterations);
/* conditioned_condition_number (precond.cpp:196-206) without the d <= 2000
 * guard: tr(M) / lambda_min(M), M = P^{-1/2}(A^T A + lambda I)P^{-1/2} where A
 * is the handle as passed (the reference passes scaled_design(p)). */
int skr_conditioned_cond(skr_ctx* ctx, const skr_data* X, double lambda, const double* U,
                         const double* sigma, int64_t k, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SKR_H */
