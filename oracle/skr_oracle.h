/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference (skridge, arXiv 1602.02350) hot path:
 * block-Lanczos sketch, sketched preconditioner, preconditioned (n+d)-component
 * ridge decomposition (Dense mode) and beta-weighted SVRG, with the exact
 * mt19937_64 / Box-Muller streams.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity pin: tests/test_oracle_golden.py checks every entry point here
 * against golden vectors produced by the UNMODIFIED reference library
 * (oracle/_ref, tests/golden/make_golden.py) — bitwise where the loop order
 * is restated exactly, else to 1e-13 relative.
 *
 * Data convention: X is n x d ROW-major (point i = row i), byte-identical to
 * the reference's d x n column-major DenseMatrix.  Dense outputs (U, V, Q)
 * are column-major like DenseMatrix.  All arithmetic is double.
 */
#ifndef SKR_ORACLE_H
#define SKR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes share include/skr.h's numbering */
enum { SKRO_OK = 0, SKRO_EDIM = 1, SKRO_EPARAM = 2, SKRO_EINPUT = 3, SKRO_EGUARD = 4,
       SKRO_EDIVERGED = 5, SKRO_EEMPTY = 8, SKRO_EINTERNAL = 10 };

const char* skro_last_error(void);

/* ---- random.cpp ------------------------------------------------------- */
typedef struct { uint64_t mt[312]; int mti; int has_spare; double spare; } skro_sampler;
void skro_sampler_init(skro_sampler* s, uint64_t seed);
uint64_t skro_mt_next(skro_sampler* s);
double skro_uniform(skro_sampler* s);
double skro_normal(skro_sampler* s);
int skro_uniforms(uint64_t seed, int64_t count, double* out);
int skro_raw_u64(uint64_t seed, int64_t count, uint64_t* out);
int skro_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* ---- factorize.cpp ---------------------------------------------------- */
int skro_sym_eigs(const double* a, int64_t n, double* values, double* vectors);
/* orthonormalize(m) (factorize.cpp:81-87): out is rows x (*cols_out) col-major */
int skro_orthonormalize(const double* m, int64_t rows, int64_t cols, double* out,
                        int64_t* cols_out);

/* ---- sketch.cpp ------------------------------------------------------- */
int64_t skro_lanczos_iterations(int64_t n, double eps_prime);
int skro_block_lanczos(const double* x, int64_t n, int64_t d, double scale, int64_t k,
                       int64_t q, double eps_prime, uint64_t seed, double* U, double* sigma,
                       double* V, int64_t* k_used, int64_t* q_used, int* rank_reduced,
                       int64_t* width);

/* ---- precond.cpp ------------------------------------------------------ */
/* inv_sqrt_j = 1/sqrt(sigma_j^2 + lambda), c = inv_sqrt_{k-1} (precond.cpp:120-136) */
int skro_build_sketched(const double* sigma, int64_t k, double lambda, double* inv_sqrt,
                        double* tail);
int skro_apply_inv_sqrt(int64_t d, const double* U, const double* inv_sqrt, int64_t k,
                        double c, const double* v, double* out);
int skro_apply_sqrt(int64_t d, const double* U, const double* inv_sqrt, int64_t k, double c,
                    const double* v, double* out);

/* ---- ridge.cpp: PreconditionedRidge (Dense mode) ----------------------- */
typedef struct skro_problem skro_problem;
/* k == 0 -> identity preconditioner (c = 1). U is d x k col-major. */
int skro_problem_create(const double* x, int64_t n, int64_t d, const double* y, double lambda,
                        const double* U, const double* inv_sqrt, int64_t k, double c,
                        skro_problem** out);
void skro_problem_destroy(skro_problem* p);
int skro_problem_betas(const skro_problem* p, double* out);
int skro_problem_transformed(const skro_problem* p, double* out); /* n x d row-major */
int skro_problem_scalars(const skro_problem* p, double* alpha, double* beta_hat,
                         double* max_row_sq);
int skro_problem_objective(const skro_problem* p, const double* w, double* out);
int skro_problem_full_gradient(const skro_problem* p, const double* w, double* out);
int skro_problem_component_gradient(const skro_problem* p, int64_t i, const double* w,
                                    double* out);

/* ---- svrg.cpp --------------------------------------------------------- */
int skro_cumulative_weights(const double* betas, int64_t N, double* cum);
int64_t skro_lookup_index(const double* cum, int64_t N, double u);
int skro_index_stream(const double* betas, int64_t N, uint64_t seed, int64_t count,
                      int64_t* out);
/* svrg_solve on the problem (svrg.cpp:152-211).  reference = NaN -> none.
 * trace_obj sized epochs; *done records written (partial on divergence). */
int skro_svrg_solve(const skro_problem* p, int64_t epochs, int64_t m, double eta,
                    uint64_t seed, const double* w0, double reference, double* w_out,
                    double* trace_obj, int64_t* done);

/* ---- ridge.cpp / bench.cpp / precond.cpp diagnostics ------------------- */
int skro_objective(const double* x, int64_t n, int64_t d, const double* y, double lambda,
                   const double* w, double* out);
int skro_reference_minimum(const double* x, int64_t n, int64_t d, const double* y,
                           double lambda, double* w_out, double* min_out);
int skro_conditioned_cond(const double* x, int64_t n, int64_t d, double lambda,
                          const double* U, const double* inv_sqrt, int64_t k, double c,
                          int unguarded, double* out);

#ifdef __cplusplus
}
#endif
#endif
