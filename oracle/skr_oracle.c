/* TEST INFRASTRUCTURE ONLY — the CPU checker ("port" oracle).  See skr_oracle.h.
 *
 * Restates the reference's serial loops in the same arithmetic order so that,
 * compiled without FMA contraction, results are bitwise identical to the
 * reference library on the same inputs (pinned by tests/test_oracle_golden.py).
 * Paths in citations are relative to /root/reference/proj.
 */
#include "skr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* skro_last_error(void) { return g_err; }

/* ===================================================================== */
/* random.cpp + <random> mt19937_64                                        */
/* ===================================================================== */

#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

/* std::mt19937_64(seed) single-value seeding (random.hpp:17, C++ [rand.eng.mers]) */
void skro_sampler_init(skro_sampler* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  s->mti = MT_N;
  s->has_spare = 0;
  s->spare = 0.0;
}

static void mt_twist(uint64_t* mt) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (mt[i] & MT_UPPER) | (mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    mt[i] = mt[(i + MT_M) % MT_N] ^ xa;
  }
}

uint64_t skro_mt_next(skro_sampler* s) {
  if (s->mti >= MT_N) {
    mt_twist(s->mt);
    s->mti = 0;
  }
  uint64_t y = s->mt[s->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* NormalSampler::uniform (random.cpp:10-12) */
double skro_uniform(skro_sampler* s) { return (double)(skro_mt_next(s) >> 11) * 0x1.0p-53; }

/* NormalSampler::normal (random.cpp:14-26): cos first, sin cached */
double skro_normal(skro_sampler* s) {
  if (s->has_spare) {
    s->has_spare = 0;
    return s->spare;
  }
  const double u1 = 1.0 - skro_uniform(s);
  const double u2 = skro_uniform(s);
  const double r = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
  s->spare = r * sin(angle);
  s->has_spare = 1;
  return r * cos(angle);
}

int skro_uniforms(uint64_t seed, int64_t count, double* out) {
  skro_sampler s;
  skro_sampler_init(&s, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = skro_uniform(&s);
  return SKRO_OK;
}

int skro_raw_u64(uint64_t seed, int64_t count, uint64_t* out) {
  skro_sampler s;
  skro_sampler_init(&s, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = skro_mt_next(&s);
  return SKRO_OK;
}

/* gaussian_matrix / fill_gaussian (random.cpp:28-41): column-major fill */
int skro_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  if (rows <= 0 || cols <= 0) return fail(SKRO_EDIM, "gaussian_matrix: rows and cols must be at least 1");
  skro_sampler s;
  skro_sampler_init(&s, seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = skro_normal(&s);
  return SKRO_OK;
}

/* ===================================================================== */
/* kernels.cpp serial loops (kernels.cpp:47-104)                           */
/* ===================================================================== */

static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(const double* a, int64_t n) { return sqrt(dot(a, a, n)); }
static void axpy(double coef, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] += coef * x[i];
}
static void scal(double coef, double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] *= coef;
}
/* dense_mul_vec: y = A x, A rows x cols col-major (kernels.cpp:65-69) */
static void mul_vec(const double* a, int64_t rows, int64_t cols, const double* x, double* y) {
  memset(y, 0, sizeof(double) * (size_t)rows);
  for (int64_t j = 0; j < cols; ++j) axpy(x[j], a + j * rows, y, rows);
}
/* dense_tmul_vec: y = A^T x (kernels.cpp:71-74) */
static void tmul_vec(const double* a, int64_t rows, int64_t cols, const double* x, double* y) {
  for (int64_t j = 0; j < cols; ++j) y[j] = dot(a + j * rows, x, rows);
}
/* dense_mul_mat: C (rows x bc) = A B (kernels.cpp:76-80) */
static void mul_mat(const double* a, int64_t rows, int64_t cols, const double* b, int64_t bc,
                    double* c) {
  for (int64_t l = 0; l < bc; ++l) mul_vec(a, rows, cols, b + l * cols, c + l * rows);
}
/* dense_tmul_mat: C (cols x bc) = A^T B (kernels.cpp:82-86) */
static void tmul_mat(const double* a, int64_t rows, int64_t cols, const double* b, int64_t bc,
                     double* c) {
  for (int64_t l = 0; l < bc; ++l) tmul_vec(a, rows, cols, b + l * rows, c + l * cols);
}
/* dense_gram: C = A A^T, lower triangle then mirrored (kernels.cpp:88-104) */
static void gram(const double* a, int64_t d, int64_t cols, double* c) {
  memset(c, 0, sizeof(double) * (size_t)(d * d));
  for (int64_t j = 0; j < cols; ++j) {
    const double* col = a + j * d;
    for (int64_t q = 0; q < d; ++q) {
      const double v = col[q];
      if (v == 0.0) continue;
      double* out = c + q * d;
      for (int64_t i = q; i < d; ++i) out[i] += v * col[i];
    }
  }
  for (int64_t q = 0; q < d; ++q)
    for (int64_t i = q + 1; i < d; ++i) c[i * d + q] = c[q * d + i];
}

/* ===================================================================== */
/* factorize.cpp                                                           */
/* ===================================================================== */

typedef struct {
  int64_t rows, size, cap;
  double* cols; /* size x rows, column j at cols + j*rows */
} basis_t;

static double max_col_norm(const double* m, int64_t rows, int64_t cols) {
  double best = 0.0;
  for (int64_t j = 0; j < cols; ++j) {
    double v = nrm2(m + j * rows, rows);
    if (v > best) best = v;
  }
  return best;
}

/* MgsBasis::append_block (factorize.cpp:53-71): two MGS passes, drop < 1e-12 * ref */
static int64_t basis_append(basis_t* b, const double* block, int64_t bcols, double* v) {
  const double ref = max_col_norm(block, b->rows, bcols);
  if (ref == 0.0) return 0;
  const double drop = 1e-12 * ref;
  int64_t appended = 0;
  for (int64_t j = 0; j < bcols; ++j) {
    memcpy(v, block + j * b->rows, sizeof(double) * (size_t)b->rows);
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t t = 0; t < b->size; ++t) {
        const double* bt = b->cols + t * b->rows;
        axpy(-dot(bt, v, b->rows), bt, v, b->rows);
      }
    }
    const double nv = nrm2(v, b->rows);
    if (nv < drop) continue;
    scal(1.0 / nv, v, b->rows);
    memcpy(b->cols + b->size * b->rows, v, sizeof(double) * (size_t)b->rows);
    b->size++;
    appended++;
  }
  return appended;
}

int skro_orthonormalize(const double* m, int64_t rows, int64_t cols, double* out,
                        int64_t* cols_out) {
  if (cols == 0) return fail(SKRO_EDIM, "orthonormalize: input has no columns");
  if (max_col_norm(m, rows, cols) == 0.0) return fail(SKRO_EEMPTY, "orthonormalize: all columns are zero");
  basis_t b = {rows, 0, cols, out};
  double* v = malloc(sizeof(double) * (size_t)rows);
  basis_append(&b, m, cols, v);
  free(v);
  *cols_out = b.size;
  return SKRO_OK;
}

/* sym_eigs: cyclic Jacobi, <= 60 sweeps, stable descending sort, largest-|entry| positive
 * (factorize.cpp:87-165).  a, vectors are n x n column-major. */
int skro_sym_eigs(const double* s, int64_t n, double* values, double* vectors) {
  double max_abs = 0.0;
  for (int64_t i = 0; i < n * n; ++i)
    if (fabs(s[i]) > max_abs) max_abs = fabs(s[i]);
  const double sym_tol = 1e-10 * (max_abs > 1.0 ? max_abs : 1.0);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j + 1; i < n; ++i)
      if (fabs(s[j * n + i] - s[i * n + j]) > sym_tol)
        return fail(SKRO_EINPUT, "sym_eigs: matrix not symmetric");
#define A(i, j) a[(j) * n + (i)]
#define V(i, j) v[(j) * n + (i)]
  double* a = malloc(sizeof(double) * (size_t)(n * n));
  double* v = calloc((size_t)(n * n), sizeof(double));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) A(i, j) = 0.5 * (s[j * n + i] + s[i * n + j]);
  for (int64_t i = 0; i < n; ++i) V(i, i) = 1.0;
  double fro = 0.0;
  for (int64_t i = 0; i < n * n; ++i) fro += a[i] * a[i];
  fro = sqrt(fro);
  const double rot_tol = 1e-15 * (fro > 1e-300 ? fro : 1e-300);
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int64_t p = 0; p + 1 < n; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (fabs(apq) <= rot_tol) continue;
        rotated = 1;
        const double tau = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                      : 1.0 / (tau - sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double sn = t * c;
        for (int64_t i = 0; i < n; ++i) {
          const double aip = A(i, p), aiq = A(i, q);
          A(i, p) = c * aip - sn * aiq;
          A(i, q) = sn * aip + c * aiq;
        }
        for (int64_t i = 0; i < n; ++i) {
          const double api = A(p, i), aqi = A(q, i);
          A(p, i) = c * api - sn * aqi;
          A(q, i) = sn * api + c * aqi;
        }
        A(p, q) = 0.0;
        A(q, p) = 0.0;
        for (int64_t i = 0; i < n; ++i) {
          const double vip = V(i, p), viq = V(i, q);
          V(i, p) = c * vip - sn * viq;
          V(i, q) = sn * vip + c * viq;
        }
      }
    }
    if (!rotated) break;
    if (sweep == 59) {
      free(a);
      free(v);
      return fail(SKRO_EINTERNAL, "sym_eigs: Jacobi iteration did not converge");
    }
  }
  /* stable sort descending by diagonal (insertion sort is stable) */
  int64_t* order = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    int64_t key = order[i];
    int64_t j = i - 1;
    while (j >= 0 && A(key, key) > A(order[j], order[j])) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = key;
  }
  for (int64_t j = 0; j < n; ++j) {
    values[j] = A(order[j], order[j]);
    memcpy(vectors + j * n, v + order[j] * n, sizeof(double) * (size_t)n);
  }
  for (int64_t j = 0; j < n; ++j) {
    double* col = vectors + j * n;
    int64_t arg = 0;
    for (int64_t i = 1; i < n; ++i)
      if (fabs(col[i]) > fabs(col[arg])) arg = i;
    if (col[arg] < 0.0) scal(-1.0, col, n);
  }
#undef A
#undef V
  free(order);
  free(a);
  free(v);
  return SKRO_OK;
}

/* normalize_svd_signs (factorize.cpp:167-178) */
static void normalize_signs(double* left, int64_t lrows, int64_t k, double* right,
                            int64_t rrows) {
  for (int64_t j = 0; j < k; ++j) {
    double* u = left + j * lrows;
    int64_t arg = 0;
    for (int64_t i = 1; i < lrows; ++i)
      if (fabs(u[i]) > fabs(u[arg])) arg = i;
    if (u[arg] < 0.0) {
      scal(-1.0, u, lrows);
      if (right) scal(-1.0, right + j * rrows, rrows);
    }
  }
}

/* ===================================================================== */
/* sketch.cpp                                                              */
/* ===================================================================== */

/* lanczos_iterations (sketch.cpp:13-16) */
int64_t skro_lanczos_iterations(int64_t n, double eps_prime) {
  const double q = ceil(log((double)n) / sqrt(eps_prime));
  return q < 2.0 ? 2 : (int64_t)q;
}

/* A = scale * X^T (d x n, the reference's DataMatrix).  mul: C (d x bc) = A B. */
static void data_mul_mat(const double* x, int64_t n, int64_t d, double scale, const double* b,
                         int64_t bc, double* c) {
  mul_mat(x, d, n, b, bc, c);
  if (scale != 1.0) scal(scale, c, d * bc);
}
/* tmul: C (n x bc) = A^T B */
static void data_tmul_mat(const double* x, int64_t n, int64_t d, double scale, const double* b,
                          int64_t bc, double* c) {
  tmul_mat(x, d, n, b, bc, c);
  if (scale != 1.0) scal(scale, c, n * bc);
}

/* krylov_block (sketch.cpp:18-39) + block_lanczos (sketch.cpp:41-90) */
int skro_block_lanczos(const double* x, int64_t n, int64_t d, double scale, int64_t k,
                       int64_t q, double eps_prime, uint64_t seed, double* U, double* sigma,
                       double* V, int64_t* k_used, int64_t* q_used, int* rank_reduced,
                       int64_t* width_out) {
  if (k < 1 || k > (d < n ? d : n)) return fail(SKRO_EPARAM, "block_lanczos: k must satisfy 1 <= k <= min(d, n)");
  if (!(eps_prime > 0.0 && eps_prime < 1.0)) return fail(SKRO_EPARAM, "block_lanczos: eps_prime must lie in (0, 1)");
  if (q <= 0) q = skro_lanczos_iterations(n, eps_prime);
  double* pi = malloc(sizeof(double) * (size_t)(n * k));
  skro_gaussian_matrix(n, k, seed, pi);

  basis_t b = {d, 0, q * k, malloc(sizeof(double) * (size_t)(d * q * k))};
  double* v = malloc(sizeof(double) * (size_t)d);
  double* block = malloc(sizeof(double) * (size_t)(d * k));
  double* t = malloc(sizeof(double) * (size_t)(n * k));
  data_mul_mat(x, n, d, scale, pi, k, block);
  int64_t appended = basis_append(&b, block, k, v);
  int rc = SKRO_OK;
  if (b.size == 0) {
    rc = fail(SKRO_EEMPTY, "krylov_block: A * Pi is numerically zero");
    goto done;
  }
  for (int64_t j = 1; j < q && appended > 0; ++j) {
    const double* prev = b.cols + (b.size - appended) * d;
    data_tmul_mat(x, n, d, scale, prev, appended, t);
    data_mul_mat(x, n, d, scale, t, appended, block);
    appended = basis_append(&b, block, appended, v);
  }
  {
    const int64_t W = b.size;
    const int64_t kk = k < W ? k : W;
    /* proj = (A^T Q)^T, W x n; gram = proj proj^T */
    double* projT = malloc(sizeof(double) * (size_t)(n * W));
    double* proj = malloc(sizeof(double) * (size_t)(n * W));
    data_tmul_mat(x, n, d, scale, b.cols, W, projT); /* n x W col-major */
    for (int64_t j = 0; j < W; ++j)
      for (int64_t i = 0; i < n; ++i) proj[i * W + j] = projT[j * n + i];
    double* g = malloc(sizeof(double) * (size_t)(W * W));
    gram(proj, W, n, g);
    double* ev = malloc(sizeof(double) * (size_t)W);
    double* evec = malloc(sizeof(double) * (size_t)(W * W));
    rc = skro_sym_eigs(g, W, ev, evec);
    if (rc == SKRO_OK) {
      for (int64_t j = 0; j < kk; ++j) sigma[j] = sqrt(ev[j] > 0.0 ? ev[j] : 0.0);
      mul_mat(b.cols, d, W, evec, kk, U); /* U = Q W_k */
      if (V) {
        double* tmp = malloc(sizeof(double) * (size_t)n);
        for (int64_t j = 0; j < kk; ++j) {
          tmul_vec(proj, W, n, evec + j * W, tmp);
          const double nrm = nrm2(tmp, n);
          if (nrm > 0.0) scal(1.0 / nrm, tmp, n);
          memcpy(V + j * n, tmp, sizeof(double) * (size_t)n);
        }
        free(tmp);
      }
      normalize_signs(U, d, kk, V, n);
      *k_used = kk;
      *q_used = q;
      *rank_reduced = kk < k;
      if (width_out) *width_out = W;
    }
    free(projT);
    free(proj);
    free(g);
    free(ev);
    free(evec);
  }
done:
  free(pi);
  free(b.cols);
  free(v);
  free(block);
  free(t);
  return rc;
}

/* ===================================================================== */
/* precond.cpp                                                             */
/* ===================================================================== */

/* build_sketched + validate (precond.cpp:120-136, :34-49) */
int skro_build_sketched(const double* sigma, int64_t k, double lambda, double* inv_sqrt,
                        double* tail) {
  if (!(lambda > 0.0) || !isfinite(lambda)) return fail(SKRO_EPARAM, "preconditioner: lambda must be positive");
  if (k < 1) return fail(SKRO_EPARAM, "build_sketched: factors must have rank >= 1");
  for (int64_t j = 0; j < k; ++j) inv_sqrt[j] = 1.0 / sqrt(sigma[j] * sigma[j] + lambda);
  *tail = inv_sqrt[k - 1];
  const double cap = 1.0 / sqrt(lambda) * (1.0 + 1e-12);
  double prev = 0.0;
  for (int64_t j = 0; j < k; ++j) {
    if (!(inv_sqrt[j] > 0.0) || inv_sqrt[j] > cap) return fail(SKRO_EINPUT, "preconditioner: coefficient out of range");
    if (inv_sqrt[j] < prev) return fail(SKRO_EINPUT, "preconditioner: coefficients must be non-decreasing");
    prev = inv_sqrt[j];
  }
  return SKRO_OK;
}

/* apply_inv_sqrt (precond.cpp:67-80) */
int skro_apply_inv_sqrt(int64_t d, const double* U, const double* D, int64_t k, double c,
                        const double* v, double* out) {
  for (int64_t i = 0; i < d; ++i) out[i] = c * v[i];
  if (k == 0) return SKRO_OK;
  double* proj = malloc(sizeof(double) * (size_t)k);
  double* lift = malloc(sizeof(double) * (size_t)d);
  tmul_vec(U, d, k, v, proj);
  for (int64_t j = 0; j < k; ++j) proj[j] *= D[j] - c;
  mul_vec(U, d, k, proj, lift);
  axpy(1.0, lift, out, d);
  free(proj);
  free(lift);
  return SKRO_OK;
}

/* apply_sqrt (precond.cpp:82-96) */
int skro_apply_sqrt(int64_t d, const double* U, const double* D, int64_t k, double c,
                    const double* v, double* out) {
  const double inv_tail = 1.0 / c;
  for (int64_t i = 0; i < d; ++i) out[i] = inv_tail * v[i];
  if (k == 0) return SKRO_OK;
  double* proj = malloc(sizeof(double) * (size_t)k);
  double* lift = malloc(sizeof(double) * (size_t)d);
  tmul_vec(U, d, k, v, proj);
  for (int64_t j = 0; j < k; ++j) proj[j] *= 1.0 / D[j] - inv_tail;
  mul_vec(U, d, k, proj, lift);
  axpy(1.0, lift, out, d);
  free(proj);
  free(lift);
  return SKRO_OK;
}

/* inv_sqrt_sq_norm (precond.cpp:110-118) */
static double inv_sqrt_sq_norm(const double* D, int64_t k, double c, double v_sq,
                               const double* proj, int64_t stride) {
  double s = c * c * v_sq;
  for (int64_t j = 0; j < k; ++j) {
    const double dj = D[j];
    s += (dj * dj - c * c) * proj[j * stride] * proj[j * stride];
  }
  return s;
}

/* ===================================================================== */
/* ridge.cpp: PreconditionedRidge, Dense mode (ridge.cpp:93-278)           */
/* ===================================================================== */

struct skro_problem {
  int64_t n, d, k;
  double lambda, c, data_coef, reg_coef;
  double* y;     /* n */
  double* U;     /* d x k col-major */
  double* D;     /* k */
  double* proj;  /* k x n col-major: column i = U^T x_i */
  double* xt;    /* transformed_: d x n col-major (= n x d row-major) */
  double* betas; /* n + d */
};

/* floor_betas (ridge.cpp:16-21) */
static void floor_betas(double* b, int64_t N) {
  double top = 0.0;
  for (int64_t i = 0; i < N; ++i)
    if (b[i] > top) top = b[i];
  const double fl = top * 1e-12;
  for (int64_t i = 0; i < N; ++i)
    if (b[i] < fl) b[i] = fl;
}

int skro_problem_create(const double* x, int64_t n, int64_t d, const double* y, double lambda,
                        const double* U, const double* D, int64_t k, double c,
                        skro_problem** out) {
  if (!(lambda > 0.0)) return fail(SKRO_EPARAM, "ridge problem: lambda must be positive");
  for (int64_t i = 0; i < n * d; ++i)
    if (!isfinite(x[i])) return fail(SKRO_EINPUT, "data matrix: entries must be finite");
  skro_problem* p = calloc(1, sizeof *p);
  p->n = n;
  p->d = d;
  p->k = k;
  p->lambda = lambda;
  p->c = k > 0 ? c : 1.0;
  p->data_coef = (double)(n + d) / (double)n;
  p->reg_coef = lambda * (double)(n + d);
  p->y = malloc(sizeof(double) * (size_t)n);
  memcpy(p->y, y, sizeof(double) * (size_t)n);
  p->U = malloc(sizeof(double) * (size_t)(d * (k > 0 ? k : 1)));
  p->D = malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
  if (k > 0) {
    memcpy(p->U, U, sizeof(double) * (size_t)(d * k));
    memcpy(p->D, D, sizeof(double) * (size_t)k);
  }
  p->proj = malloc(sizeof(double) * (size_t)(n * (k > 0 ? k : 1)));
  p->xt = malloc(sizeof(double) * (size_t)(n * d));
  p->betas = malloc(sizeof(double) * (size_t)(n + d));
  /* proj_ = (data^T U)^T (ridge.cpp:117) */
  if (k > 0) {
    double* tmp = malloc(sizeof(double) * (size_t)(n * k));
    tmul_mat(x, d, n, p->U, k, tmp); /* n x k */
    for (int64_t l = 0; l < k; ++l)
      for (int64_t i = 0; i < n; ++i) p->proj[i * k + l] = tmp[l * n + i];
    free(tmp);
  }
  /* betas (ridge.cpp:124-131) */
  for (int64_t i = 0; i < n; ++i) {
    const double* col = x + i * d;
    p->betas[i] = p->data_coef * inv_sqrt_sq_norm(p->D, k, p->c, dot(col, col, d),
                                                  p->proj + i * k, 1);
  }
  for (int64_t j = 0; j < d; ++j) {
    /* basis_rows_.col(j) = row j of U */
    p->betas[n + j] = p->reg_coef * inv_sqrt_sq_norm(p->D, k, p->c, 1.0, p->U + j, d);
  }
  floor_betas(p->betas, n + d);
  /* transformed_ = c X + U ((D - c) o proj) (ridge.cpp:133-149) */
  memcpy(p->xt, x, sizeof(double) * (size_t)(n * d));
  scal(p->c, p->xt, n * d);
  if (k > 0) {
    double* scaled = malloc(sizeof(double) * (size_t)(n * k));
    memcpy(scaled, p->proj, sizeof(double) * (size_t)(n * k));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < k; ++j) scaled[i * k + j] *= p->D[j] - p->c;
    double* lift = malloc(sizeof(double) * (size_t)(n * d));
    mul_mat(p->U, d, k, scaled, n, lift);
    axpy(1.0, lift, p->xt, n * d);
    free(lift);
    free(scaled);
  }
  *out = p;
  return SKRO_OK;
}

void skro_problem_destroy(skro_problem* p) {
  if (!p) return;
  free(p->y);
  free(p->U);
  free(p->D);
  free(p->proj);
  free(p->xt);
  free(p->betas);
  free(p);
}

int skro_problem_betas(const skro_problem* p, double* out) {
  memcpy(out, p->betas, sizeof(double) * (size_t)(p->n + p->d));
  return SKRO_OK;
}

int skro_problem_transformed(const skro_problem* p, double* out) {
  memcpy(out, p->xt, sizeof(double) * (size_t)(p->n * p->d));
  return SKRO_OK;
}

/* strong_convexity = lambda * min_inv_eigenvalue (ridge.cpp:152-157, precond.cpp:62-65);
 * mean_beta (svrg.cpp:213-217); max data-row ||x~_i||^2 for the step-size rule. */
int skro_problem_scalars(const skro_problem* p, double* alpha, double* beta_hat,
                         double* max_row_sq) {
  const double lead = p->k > 0 ? p->D[0] : p->c;
  *alpha = p->lambda * (lead * lead);
  double total = 0.0;
  for (int64_t i = 0; i < p->n + p->d; ++i) total += p->betas[i];
  *beta_hat = total / (double)(p->n + p->d);
  double mx = 0.0;
  for (int64_t i = 0; i < p->n; ++i) {
    const double* r = p->xt + i * p->d;
    const double v = dot(r, r, p->d);
    if (v > mx) mx = v;
  }
  *max_row_sq = mx;
  return SKRO_OK;
}

/* PreconditionedRidge::objective, Dense (ridge.cpp:174-198) */
int skro_problem_objective(const skro_problem* p, const double* w, double* out) {
  const int64_t n = p->n, d = p->d, k = p->k;
  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = dot(p->xt + i * d, w, d) - p->y[i];
    loss += e * e;
  }
  double* uw = malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
  if (k > 0) tmul_vec(p->U, d, k, w, uw);
  const double reg_sq = inv_sqrt_sq_norm(p->D, k, p->c, dot(w, w, d), uw, 1);
  free(uw);
  *out = loss / (2.0 * (double)n) + 0.5 * p->lambda * reg_sq;
  return SKRO_OK;
}

/* PreconditionedRidge::full_gradient, Dense (ridge.cpp:200-236) */
int skro_problem_full_gradient(const skro_problem* p, const double* w, double* out) {
  const int64_t n = p->n, d = p->d;
  double* r = malloc(sizeof(double) * (size_t)n);
  tmul_vec(p->xt, d, n, w, r);
  for (int64_t i = 0; i < n; ++i) r[i] -= p->y[i];
  mul_vec(p->xt, d, n, r, out);
  const double inv_n = 1.0 / (double)n;
  scal(inv_n, out, d);
  double* half = malloc(sizeof(double) * (size_t)d);
  double* full = malloc(sizeof(double) * (size_t)d);
  skro_apply_inv_sqrt(d, p->U, p->D, p->k, p->c, w, half);
  skro_apply_inv_sqrt(d, p->U, p->D, p->k, p->c, half, full);
  axpy(p->lambda, full, out, d);
  free(half);
  free(full);
  free(r);
  return SKRO_OK;
}

/* PreconditionedRidge::component_gradient, Dense (ridge.cpp:238-278) */
static void component_gradient(const skro_problem* p, int64_t i, const double* w, double* out,
                               double* uw, double* coef, double* lift) {
  const int64_t n = p->n, d = p->d, k = p->k;
  memset(out, 0, sizeof(double) * (size_t)d);
  if (i < n) {
    const double* col = p->xt + i * d;
    const double g = p->data_coef * (dot(col, w, d) - p->y[i]);
    axpy(g, col, out, d);
    return;
  }
  const int64_t j = i - n;
  if (k > 0) tmul_vec(p->U, d, k, w, uw);
  double wb = p->c * w[j];
  for (int64_t l = 0; l < k; ++l) wb += (p->D[l] - p->c) * p->U[l * d + j] * uw[l];
  const double g = p->reg_coef * wb;
  out[j] += g * p->c;
  if (k == 0) return;
  for (int64_t l = 0; l < k; ++l) coef[l] = g * (p->D[l] - p->c) * p->U[l * d + j];
  mul_vec(p->U, d, k, coef, lift);
  axpy(1.0, lift, out, d);
}

int skro_problem_component_gradient(const skro_problem* p, int64_t i, const double* w,
                                    double* out) {
  if (i < 0 || i >= p->n + p->d) return fail(SKRO_EINPUT, "component_gradient: index out of range");
  const int64_t kk = p->k > 0 ? p->k : 1;
  double* uw = malloc(sizeof(double) * (size_t)kk);
  double* coef = malloc(sizeof(double) * (size_t)kk);
  double* lift = malloc(sizeof(double) * (size_t)p->d);
  component_gradient(p, i, w, out, uw, coef, lift);
  free(uw);
  free(coef);
  free(lift);
  return SKRO_OK;
}

/* ===================================================================== */
/* svrg.cpp                                                                */
/* ===================================================================== */

/* make_cumulative_weights (svrg.cpp:90-106) */
int skro_cumulative_weights(const double* betas, int64_t N, double* cum) {
  if (N <= 0) return fail(SKRO_EINPUT, "sampling: no weights");
  double total = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    if (!(betas[i] >= 0.0)) return fail(SKRO_EINPUT, "sampling: negative weight");
    total += betas[i];
  }
  if (!(total > 0.0)) return fail(SKRO_EINPUT, "sampling: zero total weight");
  double run = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    run += betas[i] / total;
    cum[i] = run;
  }
  cum[N - 1] = 1.0;
  return SKRO_OK;
}

/* lookup_index (svrg.cpp:122-126): first i with cum[i] >= u, clamped to N-1 */
int64_t skro_lookup_index(const double* cum, int64_t N, double u) {
  int64_t lo = 0, len = N;
  while (len > 0) {
    int64_t half = len / 2;
    if (cum[lo + half] < u) {
      lo = lo + half + 1;
      len = len - half - 1;
    } else {
      len = half;
    }
  }
  return lo == N ? N - 1 : lo;
}

int skro_index_stream(const double* betas, int64_t N, uint64_t seed, int64_t count,
                      int64_t* out) {
  double* cum = malloc(sizeof(double) * (size_t)N);
  int rc = skro_cumulative_weights(betas, N, cum);
  if (rc == SKRO_OK) {
    skro_sampler s;
    skro_sampler_init(&s, seed);
    for (int64_t t = 0; t < count; ++t) out[t] = skro_lookup_index(cum, N, skro_uniform(&s));
  }
  free(cum);
  return rc;
}

/* svrg_solve with DenseEpochState (svrg.cpp:18-54, :142-211) */
int skro_svrg_solve(const skro_problem* p, int64_t epochs, int64_t m, double eta,
                    uint64_t seed, const double* w0, double reference, double* w_out,
                    double* trace_obj, int64_t* done) {
  (void)reference;
  if (epochs < 1 || m < 1) return fail(SKRO_EPARAM, "svrg: epochs and epoch length must be >= 1");
  if (!(eta > 0.0)) return fail(SKRO_EPARAM, "svrg: step size must be positive");
  const int64_t d = p->d, N = p->n + p->d;
  for (int64_t j = 0; j < d; ++j)
    if (!isfinite(w0[j])) return fail(SKRO_EINPUT, "svrg: start point must be finite");
  double* cum = malloc(sizeof(double) * (size_t)N);
  double* inv_nq = malloc(sizeof(double) * (size_t)N);
  int rc = skro_cumulative_weights(p->betas, N, cum);
  if (rc != SKRO_OK) {
    free(cum);
    free(inv_nq);
    return rc;
  }
  double total = 0.0;
  for (int64_t i = 0; i < N; ++i) total += p->betas[i];
  for (int64_t i = 0; i < N; ++i) inv_nq[i] = total / ((double)N * p->betas[i]);
  skro_sampler rng;
  skro_sampler_init(&rng, seed);
  const int64_t kk = p->k > 0 ? p->k : 1;
  double* w = malloc(sizeof(double) * (size_t)d);
  double* snap = malloc(sizeof(double) * (size_t)d);
  double* mu = malloc(sizeof(double) * (size_t)d);
  double* sum = malloc(sizeof(double) * (size_t)d);
  double* dir = malloc(sizeof(double) * (size_t)d);
  double* scratch = malloc(sizeof(double) * (size_t)d);
  double* uw = malloc(sizeof(double) * (size_t)kk);
  double* coef = malloc(sizeof(double) * (size_t)kk);
  double* lift = malloc(sizeof(double) * (size_t)d);
  double initial;
  skro_problem_objective(p, w0, &initial);
  memcpy(w, w0, sizeof(double) * (size_t)d);
  *done = 0;
  for (int64_t s = 1; s <= epochs; ++s) {
    skro_problem_full_gradient(p, w, mu);
    memcpy(snap, w, sizeof(double) * (size_t)d);
    memset(sum, 0, sizeof(double) * (size_t)d);
    for (int64_t t = 0; t < m; ++t) {
      const int64_t i = skro_lookup_index(cum, N, skro_uniform(&rng));
      component_gradient(p, i, w, dir, uw, coef, lift);
      component_gradient(p, i, snap, scratch, uw, coef, lift);
      for (int64_t j = 0; j < d; ++j) dir[j] = (dir[j] - scratch[j]) * inv_nq[i] + mu[j];
      axpy(-eta, dir, w, d);
      axpy(1.0, w, sum, d);
    }
    memcpy(w, sum, sizeof(double) * (size_t)d);
    scal(1.0 / (double)m, w, d);
    double obj;
    skro_problem_objective(p, w, &obj);
    trace_obj[s - 1] = obj;
    *done = s;
    if (!isfinite(obj) || (initial > 0.0 && obj > 1e6 * initial)) {
      rc = fail(SKRO_EDIVERGED, "svrg: objective diverged");
      break;
    }
  }
  memcpy(w_out, w, sizeof(double) * (size_t)d);
  free(cum);
  free(inv_nq);
  free(w);
  free(snap);
  free(mu);
  free(sum);
  free(dir);
  free(scratch);
  free(uw);
  free(coef);
  free(lift);
  return rc;
}

/* ===================================================================== */
/* ridge.cpp:33-43 objective, bench.cpp:22-94 reference_minimum,           */
/* precond.cpp:174-206 conditioned matrix / condition number               */
/* ===================================================================== */

int skro_objective(const double* x, int64_t n, int64_t d, const double* y, double lambda,
                   const double* w, double* out) {
  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = dot(x + i * d, w, d) - y[i];
    loss += e * e;
  }
  const double sq = dot(w, w, d);
  *out = loss / (2.0 * (double)n) + 0.5 * lambda * sq;
  return SKRO_OK;
}

/* scaled_design(p).gram() (ridge.cpp:54-56, data_matrix.cpp:111-119) */
static void scaled_gram(const double* x, int64_t n, int64_t d, double* g) {
  const double scale = 1.0 * (1.0 / sqrt((double)n));
  gram(x, d, n, g);
  scal(scale * scale, g, d * d);
}

/* cholesky_solve (bench.cpp:22-48) */
static int cholesky_solve(double* a, int64_t n, double* b) {
#define M(i, j) a[(j) * n + (i)]
  for (int64_t j = 0; j < n; ++j) {
    double diag = M(j, j);
    for (int64_t p = 0; p < j; ++p) diag -= M(j, p) * M(j, p);
    if (!(diag > 0.0)) return fail(SKRO_EINPUT, "cholesky: matrix not positive definite");
    diag = sqrt(diag);
    M(j, j) = diag;
    for (int64_t i = j + 1; i < n; ++i) {
      double v = M(i, j);
      for (int64_t p = 0; p < j; ++p) v -= M(i, p) * M(j, p);
      M(i, j) = v / diag;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    double v = b[i];
    for (int64_t p = 0; p < i; ++p) v -= M(i, p) * b[p];
    b[i] = v / M(i, i);
  }
  for (int64_t ii = n; ii-- > 0;) {
    double v = b[ii];
    for (int64_t p = ii + 1; p < n; ++p) v -= M(p, ii) * b[p];
    b[ii] = v / M(ii, ii);
  }
#undef M
  return SKRO_OK;
}

int skro_reference_minimum(const double* x, int64_t n, int64_t d, const double* y,
                           double lambda, double* w_out, double* min_out) {
  if (d > 5000) return fail(SKRO_EGUARD, "reference_minimum: CG route not restated (d > 5000)");
  double* sys = malloc(sizeof(double) * (size_t)(d * d));
  scaled_gram(x, n, d, sys);
  for (int64_t i = 0; i < d; ++i) sys[i * d + i] += lambda;
  mul_vec(x, d, n, y, w_out);
  scal(1.0 / (double)n, w_out, d);
  int rc = cholesky_solve(sys, d, w_out);
  free(sys);
  if (rc != SKRO_OK) return rc;
  return skro_objective(x, n, d, y, lambda, w_out, min_out);
}

int skro_conditioned_cond(const double* x, int64_t n, int64_t d, double lambda,
                          const double* U, const double* D, int64_t k, double c, int unguarded,
                          double* out) {
  if (!unguarded && d > 2000) return fail(SKRO_EGUARD, "conditioned_condition_number: dimension exceeds the dense guard");
  if (k == 0) c = 1.0;
  double* b = malloc(sizeof(double) * (size_t)(d * d));
  double* half = malloc(sizeof(double) * (size_t)(d * d));
  double* m = malloc(sizeof(double) * (size_t)(d * d));
  scaled_gram(x, n, d, b);
  for (int64_t i = 0; i < d; ++i) b[i * d + i] += lambda;
  for (int64_t j = 0; j < d; ++j) skro_apply_inv_sqrt(d, U, D, k, c, b + j * d, half + j * d);
  /* half_t = half^T, then m.col(j) = apply_inv_sqrt(half_t.col(j)) */
  double* col = malloc(sizeof(double) * (size_t)d);
  for (int64_t j = 0; j < d; ++j) {
    for (int64_t i = 0; i < d; ++i) col[i] = half[i * d + j];
    skro_apply_inv_sqrt(d, U, D, k, c, col, m + j * d);
  }
  for (int64_t j = 0; j < d; ++j)
    for (int64_t i = j + 1; i < d; ++i) {
      const double v = 0.5 * (m[j * d + i] + m[i * d + j]);
      m[j * d + i] = v;
      m[i * d + j] = v;
    }
  double* ev = malloc(sizeof(double) * (size_t)d);
  double* evec = malloc(sizeof(double) * (size_t)(d * d));
  int rc = skro_sym_eigs(m, d, ev, evec);
  if (rc == SKRO_OK) {
    double tr = 0.0;
    for (int64_t i = 0; i < d; ++i) tr += m[i * d + i];
    *out = tr / ev[d - 1];
  }
  free(b);
  free(half);
  free(m);
  free(col);
  free(ev);
  free(evec);
  return rc;
}
