// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" shim over the UNMODIFIED reference library (skridge, built from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).  It lets
// the Python tests, tests/golden/make_golden.py and bench.py's reference arm /
// cpu_baseline call the reference's own public C++ API through ctypes.
//
// Layout convention at this boundary: the data matrix is passed as n x d
// ROW-major doubles, which is byte-identical to the reference's d x n
// column-major DenseMatrix (dense_matrix.hpp:12-15).  Dense
// results (U, V) are returned column-major exactly as DenseMatrix stores them.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "skridge/bench.hpp"
#include "skridge/dataset.hpp"
#include "skridge/sparse_matrix.hpp"
#include "skridge/data_matrix.hpp"
#include "skridge/errors.hpp"
#include "skridge/factorize.hpp"
#include "skridge/kernels.hpp"
#include "skridge/precond.hpp"
#include "skridge/random.hpp"
#include "skridge/ridge.hpp"
#include "skridge/sketch.hpp"
#include "skridge/svrg.hpp"

using namespace skridge;

namespace {

thread_local std::string g_err;

// Error codes mirror include/skr.h so tests can compare error behaviour.
int classify(const std::exception& e) {
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const ParameterError*>(&e)) return 2;
  if (dynamic_cast<const InputError*>(&e)) return 3;
  if (dynamic_cast<const ScaleGuardError*>(&e)) return 4;
  if (dynamic_cast<const DivergenceError*>(&e)) return 5;
  if (dynamic_cast<const EmptyBasisError*>(&e)) return 8;
  return 10;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

DenseMatrix colmajor(const double* p, std::size_t rows, std::size_t cols) {
  return DenseMatrix(rows, cols, Vector(p, p + rows * cols));
}

struct RefProblem {
  RidgeProblem problem;
  Preconditioner precond;
  std::shared_ptr<PreconditionedRidge> pre;
};

Preconditioner make_precond(std::size_t d, const double* U, const double* sigma, std::size_t k,
                            double lambda) {
  if (k == 0) return Preconditioner::identity(d, lambda);
  SketchedSvd sv;
  sv.left = colmajor(U, d, k);
  sv.singular_values = Vector(sigma, sigma + k);
  sv.right = DenseMatrix(1, k);
  sv.k = k;
  return build_sketched(sv, lambda);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_threads_serial(int serial) {
  kernels::set_execution(serial ? kernels::Execution::Serial : kernels::Execution::Auto);
  return 0;
}

// NormalSampler(seed).uniform() x count  (random.cpp:10-12)
int ref_uniforms(std::uint64_t seed, std::int64_t count, double* out) {
  return guard([&] {
    NormalSampler s(seed);
    for (std::int64_t i = 0; i < count; ++i) out[i] = s.uniform();
  });
}

// gaussian_matrix(rows, cols, seed), column-major (random.cpp:28-41)
int ref_gaussian_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
  return guard([&] {
    DenseMatrix m = gaussian_matrix(rows, cols, seed);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
  });
}

// sym_eigs (factorize.cpp:87-165); a is n x n column-major.
int ref_sym_eigs(const double* a, std::int64_t n, double* values, double* vectors) {
  return guard([&] {
    EigResult r = sym_eigs(colmajor(a, n, n));
    std::memcpy(values, r.values.data(), sizeof(double) * n);
    std::memcpy(vectors, r.vectors.data(), sizeof(double) * n * n);
  });
}

// krylov_block width only (sketch.cpp:18-39), used to probe rank drop.
int ref_krylov_width(const double* x, std::int64_t n, std::int64_t d, double scale,
                     std::int64_t k, std::int64_t q, std::uint64_t seed, std::int64_t* width) {
  return guard([&] {
    DataMatrix a(colmajor(x, d, n), scale);
    DenseMatrix pi = gaussian_matrix(n, k, seed);
    *width = static_cast<std::int64_t>(krylov_block(a, pi, q).cols());
  });
}

// block_lanczos (sketch.cpp:41-90).  q <= 0 -> lanczos_iterations(n, eps').
int ref_block_lanczos(const double* x, std::int64_t n, std::int64_t d, double scale,
                      std::int64_t k, std::int64_t q, double eps_prime, std::uint64_t seed,
                      double* U, double* sigma, double* V, std::int64_t* k_used,
                      std::int64_t* q_used, int* rank_reduced) {
  return guard([&] {
    DataMatrix a(colmajor(x, d, n), scale);
    LanczosConfig cfg;
    cfg.k = static_cast<std::size_t>(k);
    cfg.eps_prime = eps_prime;
    cfg.seed = seed;
    if (q > 0) cfg.q_override = static_cast<std::size_t>(q);
    SketchedSvd sv = block_lanczos(a, cfg);
    std::memcpy(U, sv.left.data(), sizeof(double) * sv.left.size());
    std::memcpy(sigma, sv.singular_values.data(), sizeof(double) * sv.k);
    if (V) std::memcpy(V, sv.right.data(), sizeof(double) * sv.right.size());
    *k_used = static_cast<std::int64_t>(sv.k);
    *q_used = static_cast<std::int64_t>(sv.q);
    *rank_reduced = sv.rank_reduced ? 1 : 0;
  });
}

// objective(p, w) on the ORIGINAL problem (ridge.cpp:33-43).
int ref_objective(const double* x, std::int64_t n, std::int64_t d, const double* y,
                  double lambda, const double* w, double* out) {
  return guard([&] {
    RidgeProblem p(DataMatrix(colmajor(x, d, n)), Vector(y, y + n), lambda);
    *out = objective(p, Vector(w, w + d));
  });
}

// reference_minimum (bench.cpp:84-94).
int ref_reference_minimum(const double* x, std::int64_t n, std::int64_t d, const double* y,
                          double lambda, double* w_out, double* min_out) {
  return guard([&] {
    RidgeProblem p(DataMatrix(colmajor(x, d, n)), Vector(y, y + n), lambda);
    ReferenceSolution r = reference_minimum(p);
    std::memcpy(w_out, r.minimizer.data(), sizeof(double) * d);
    *min_out = r.minimum;
  });
}

// reference_minimum_cg(p, tol, max_iterations) (bench.cpp:56-82) on dense rows
int ref_reference_minimum_cg(const double* x, std::int64_t n, std::int64_t d, const double* y, double lambda,
                             double tol, std::int64_t max_it, double* w_out) {
  return guard([&] {
    RidgeProblem p(DataMatrix(colmajor(x, d, n)), Vector(y, y + n), lambda);
    Vector w = reference_minimum_cg(p, tol, static_cast<std::size_t>(max_it));
    std::memcpy(w_out, w.data(), sizeof(double) * d);
  });
}

// conditioned_condition_number on scaled_design(p) (precond.cpp:196-206);
// unguarded=1 composes conditioned_matrix + sym_eigs directly (d > 2000).
int ref_conditioned_cond(const double* x, std::int64_t n, std::int64_t d, double lambda,
                         const double* U, const double* sigma, std::int64_t k, int unguarded,
                         double* out) {
  return guard([&] {
    DataMatrix a(colmajor(x, d, n), 1.0 / std::sqrt(static_cast<double>(n)));
    Preconditioner pc = make_precond(d, U, sigma, k, lambda);
    if (!unguarded) {
      *out = conditioned_condition_number(a, lambda, pc);
    } else {
      DenseMatrix m = conditioned_matrix(a, lambda, pc);
      EigResult eig = sym_eigs(m);
      double tr = 0.0;
      for (std::size_t i = 0; i < m.rows(); ++i) tr += m(i, i);
      *out = tr / eig.values.back();
    }
  });
}

// ---- sparse inputs: CSR over points (row_ptr n+1, col_idx, vals) is the
// reference's CSC over points (sparse_matrix.hpp:8-14) byte for byte ----
DataMatrix csr_data(const std::int64_t* row_ptr, const std::int32_t* col_idx, const double* vals, std::int64_t n,
                    std::int64_t d, double scale = 1.0) {
  const std::int64_t nnz = row_ptr[n];
  std::vector<std::size_t> cp(row_ptr, row_ptr + n + 1), ri(col_idx, col_idx + nnz);
  return DataMatrix(SparseMatrix(static_cast<std::size_t>(d), static_cast<std::size_t>(n), std::move(cp),
                                 std::move(ri), Vector(vals, vals + nnz)),
                    scale);
}

int ref_block_lanczos_csr(const std::int64_t* row_ptr, const std::int32_t* col_idx, const double* vals,
                          std::int64_t n, std::int64_t d, double scale, std::int64_t k, std::int64_t q,
                          double eps_prime, std::uint64_t seed, double* U, double* sigma, double* V,
                          std::int64_t* k_used, std::int64_t* q_used, int* rank_reduced) {
  return guard([&] {
    DataMatrix a = csr_data(row_ptr, col_idx, vals, n, d, scale);
    LanczosConfig cfg;
    cfg.k = static_cast<std::size_t>(k);
    cfg.eps_prime = eps_prime;
    cfg.seed = seed;
    if (q > 0) cfg.q_override = static_cast<std::size_t>(q);
    SketchedSvd sv = block_lanczos(a, cfg);
    std::memcpy(U, sv.left.data(), sizeof(double) * sv.left.size());
    std::memcpy(sigma, sv.singular_values.data(), sizeof(double) * sv.k);
    if (V) std::memcpy(V, sv.right.data(), sizeof(double) * sv.right.size());
    *k_used = static_cast<std::int64_t>(sv.k);
    *q_used = static_cast<std::int64_t>(sv.q);
    *rank_reduced = sv.rank_reduced ? 1 : 0;
  });
}

int ref_objective_csr(const std::int64_t* row_ptr, const std::int32_t* col_idx, const double* vals, std::int64_t n,
                      std::int64_t d, const double* y, double lambda, const double* w, double* out) {
  return guard([&] {
    RidgeProblem p(csr_data(row_ptr, col_idx, vals, n, d), Vector(y, y + n), lambda);
    *out = objective(p, Vector(w, w + d));
  });
}

int ref_reference_minimum_csr(const std::int64_t* row_ptr, const std::int32_t* col_idx, const double* vals,
                              std::int64_t n, std::int64_t d, const double* y, double lambda, double* w_out,
                              double* min_out) {
  return guard([&] {
    RidgeProblem p(csr_data(row_ptr, col_idx, vals, n, d), Vector(y, y + n), lambda);
    ReferenceSolution r = reference_minimum(p);
    std::memcpy(w_out, r.minimizer.data(), sizeof(double) * d);
    *min_out = r.minimum;
  });
}

int ref_problem_create_csr(const std::int64_t* row_ptr, const std::int32_t* col_idx, const double* vals,
                           std::int64_t n, std::int64_t d, const double* y, double lambda, const double* U,
                           const double* sigma, std::int64_t k, int mode, void** out) {
  return guard([&] {
    RidgeProblem p(csr_data(row_ptr, col_idx, vals, n, d), Vector(y, y + n), lambda);
    Preconditioner pc = make_precond(d, U, sigma, k, lambda);
    ApplyMode m = mode == 0 ? ApplyMode::Dense : mode == 1 ? ApplyMode::Lazy : ApplyMode::Auto;
    auto pre = preconditioned_components(p, pc, m);
    *out = new RefProblem{std::move(p), std::move(pc), std::move(pre)};
  });
}

// read_sparse_corpus (dataset.cpp:87-162): sizes, then the CSR-over-points arrays.
// Parse errors return the status of their exception type; ParseError -> 3 (input).
int ref_read_corpus_sizes(const char* path, std::int64_t* n, std::int64_t* d, std::int64_t* nnz) {
  return guard([&] {
    LabeledDataset ds = read_sparse_corpus(path);
    const SparseMatrix* sp = ds.data.sparse();
    *n = static_cast<std::int64_t>(sp->cols());
    *d = static_cast<std::int64_t>(sp->rows());
    *nnz = static_cast<std::int64_t>(sp->nnz());
  });
}

int ref_read_corpus(const char* path, std::int64_t* row_ptr, std::int32_t* col_idx, double* vals, double* labels) {
  return guard([&] {
    LabeledDataset ds = read_sparse_corpus(path);
    const SparseMatrix* sp = ds.data.sparse();
    for (std::size_t j = 0; j <= sp->cols(); ++j) row_ptr[j] = static_cast<std::int64_t>(sp->col_ptr()[j]);
    for (std::size_t t = 0; t < sp->nnz(); ++t) {
      col_idx[t] = static_cast<std::int32_t>(sp->row_idx()[t]);
      vals[t] = sp->values()[t];
    }
    std::memcpy(labels, ds.labels.data(), sizeof(double) * ds.labels.size());
  });
}

// generate_synthetic (dataset.cpp:16-79): the reference's own synthetic instance
// (decay 0: 1/q, 1: 1/q^2), written as n x d row-major (= its d x n column-major).
int ref_generate_synthetic(std::int64_t n, std::int64_t d, int decay, double noise_std, std::uint64_t seed,
                           int normalize_columns, double* x_out, double* y_out) {
  return guard([&] {
    SyntheticSpec spec;
    spec.n = static_cast<std::size_t>(n);
    spec.d = static_cast<std::size_t>(d);
    spec.decay = decay ? SpectrumDecay::Quadratic : SpectrumDecay::Linear;
    spec.noise_std = noise_std;
    spec.seed = seed;
    spec.normalize_columns = normalize_columns != 0;
    LabeledDataset ds = generate_synthetic(spec);
    DenseMatrix m = ds.data.densified();
    for (std::int64_t i = 0; i < n; ++i)
      for (std::int64_t j = 0; j < d; ++j) x_out[i * d + j] = m(static_cast<std::size_t>(j), static_cast<std::size_t>(i));
    std::memcpy(y_out, ds.labels.data(), sizeof(double) * n);
  });
}

// dataset_spectrum (bench.cpp:205-212), theoretical_ratio (precond.cpp:208-219),
// avg_condition_number (precond.cpp:165-172).
int ref_dataset_spectrum(const double* x, std::int64_t n, std::int64_t d, double lambda, double* eigs) {
  return guard([&] {
    RidgeProblem p(DataMatrix(colmajor(x, d, n)), Vector(static_cast<std::size_t>(n), 0.0), lambda);
    SpectrumSummary s = dataset_spectrum(p);
    std::memcpy(eigs, s.eigenvalues.data(), sizeof(double) * d);
  });
}

int ref_theoretical_ratio(const double* eigs, std::int64_t d, double lambda, std::int64_t k, double* out) {
  return guard([&] {
    SpectrumSummary s(Vector(eigs, eigs + d), lambda);
    *out = theoretical_ratio(s, static_cast<std::size_t>(k));
  });
}

int ref_avg_condition_number(const double* eigs, std::int64_t d, double lambda, double* out) {
  return guard([&] {
    SpectrumSummary s(Vector(eigs, eigs + d), lambda);
    *out = avg_condition_number(s);
  });
}

// Preconditioner::apply_inv_sqrt (precond.cpp:67-80).
int ref_apply_inv_sqrt(std::int64_t d, const double* U, const double* sigma, std::int64_t k,
                       double lambda, const double* v, double* out) {
  return guard([&] {
    Preconditioner pc = make_precond(d, U, sigma, k, lambda);
    Vector r = pc.apply_inv_sqrt(Vector(v, v + d));
    std::memcpy(out, r.data(), sizeof(double) * d);
  });
}

// preconditioned_components(p, build_sketched(sv, lambda), mode) (ridge.cpp:93-150).
// k == 0 -> Preconditioner::identity.  mode: 0 Dense, 1 Lazy, 2 Auto.
int ref_problem_create(const double* x, std::int64_t n, std::int64_t d, const double* y,
                       double lambda, const double* U, const double* sigma, std::int64_t k,
                       int mode, void** out) {
  return guard([&] {
    RidgeProblem p(DataMatrix(colmajor(x, d, n)), Vector(y, y + n), lambda);
    Preconditioner pc = make_precond(d, U, sigma, k, lambda);
    ApplyMode m = mode == 0 ? ApplyMode::Dense : mode == 1 ? ApplyMode::Lazy : ApplyMode::Auto;
    auto pre = preconditioned_components(p, pc, m);
    *out = new RefProblem{std::move(p), std::move(pc), std::move(pre)};
  });
}

int ref_problem_destroy(void* h) {
  delete static_cast<RefProblem*>(h);
  return 0;
}

int ref_problem_mode(void* h) {
  return static_cast<RefProblem*>(h)->pre->mode() == ApplyMode::Dense ? 0 : 1;
}

int ref_problem_betas(void* h, double* out) {
  return guard([&] {
    const Vector& b = static_cast<RefProblem*>(h)->pre->betas();
    std::memcpy(out, b.data(), sizeof(double) * b.size());
  });
}

int ref_problem_scalars(void* h, double* alpha, double* beta_hat) {
  return guard([&] {
    auto& pre = *static_cast<RefProblem*>(h)->pre;
    *alpha = pre.strong_convexity();
    *beta_hat = mean_beta(pre);
  });
}

int ref_problem_objective(void* h, const double* w, double* out) {
  return guard([&] {
    auto& pre = *static_cast<RefProblem*>(h)->pre;
    *out = pre.objective(Vector(w, w + pre.dimension()));
  });
}

int ref_problem_full_gradient(void* h, const double* w, double* out) {
  return guard([&] {
    auto& pre = *static_cast<RefProblem*>(h)->pre;
    Vector g;
    pre.full_gradient(Vector(w, w + pre.dimension()), g);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

int ref_problem_component_gradient(void* h, std::int64_t i, const double* w, double* out) {
  return guard([&] {
    auto& pre = *static_cast<RefProblem*>(h)->pre;
    Vector g;
    pre.component_gradient(static_cast<std::size_t>(i), Vector(w, w + pre.dimension()), g);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

// svrg_solve (svrg.cpp:152-211).  reference = NaN -> no suboptimality.
// trace_obj/trace_ms sized `epochs`; *done = number of records (partial on divergence).
int ref_svrg_solve(void* h, std::int64_t epochs, std::int64_t m, double eta, std::uint64_t seed,
                   const double* w0, double reference, double* w_out, double* trace_obj,
                   double* trace_ms, std::int64_t* done) {
  auto& pre = *static_cast<RefProblem*>(h)->pre;
  try {
    SvrgConfig cfg;
    cfg.epochs = static_cast<std::size_t>(epochs);
    cfg.epoch_length = static_cast<std::size_t>(m);
    cfg.step_size = eta;
    cfg.seed = seed;
    std::optional<double> ref;
    if (!std::isnan(reference)) ref = reference;
    SvrgResult r = svrg_solve(pre, cfg, Vector(w0, w0 + pre.dimension()), ref);
    std::memcpy(w_out, r.iterate.data(), sizeof(double) * r.iterate.size());
    for (std::size_t s = 0; s < r.trace.size(); ++s) {
      trace_obj[s] = r.trace[s].objective;
      if (trace_ms) trace_ms[s] = r.trace[s].elapsed_ms;
    }
    *done = static_cast<std::int64_t>(r.trace.size());
    return 0;
  } catch (const DivergenceError& e) {
    for (std::size_t s = 0; s < e.trace().size(); ++s) {
      trace_obj[s] = e.trace()[s].objective;
      if (trace_ms) trace_ms[s] = e.trace()[s].elapsed_ms;
    }
    *done = static_cast<std::int64_t>(e.trace().size());
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Index stream svrg_solve draws: lookup_index(make_cumulative_weights(beta),
// NormalSampler(seed).uniform()) for `count` steps (svrg.cpp:90-126,165,174,192).
int ref_index_stream(const double* betas, std::int64_t N, std::uint64_t seed, std::int64_t count,
                     std::int64_t* out) {
  return guard([&] {
    Vector cum = make_cumulative_weights(Vector(betas, betas + N));
    NormalSampler rng(seed);
    (void)sample_index(cum, 0.5);  // validates the table once, as svrg_solve does
    for (std::int64_t t = 0; t < count; ++t) {
      // lookup_index (svrg.cpp:122-126) is file-local; same std::lower_bound + clamp.
      auto it = std::lower_bound(cum.begin(), cum.end(), rng.uniform());
      if (it == cum.end()) --it;
      out[t] = static_cast<std::int64_t>(it - cum.begin());
    }
  });
}

int ref_cumulative_weights(const double* betas, std::int64_t N, double* out) {
  return guard([&] {
    Vector cum = make_cumulative_weights(Vector(betas, betas + N));
    std::memcpy(out, cum.data(), sizeof(double) * N);
  });
}


// ---- the composed pipeline on ONE DataMatrix -------
// RidgeProblem(X, y, lambda) -> block_lanczos(scaled_design(p), {k, 0.5, seed, q})
// -> build_sketched -> preconditioned_components(p, P, mode) -> reference_minimum
// -> svrg_solve(m, eta, seed, L*) -> apply_inv_sqrt -> objective(p, w^)
// (ridge.cpp:413-454 with q_override; bench.cpp:84-94).  X is n x d row-major,
// fp32 (promoted to fp64 once, the reference has no fp32) or fp64.  k == 0: the
// unpreconditioned Preconditioner::identity.  eta_rule 0: 1/(4 max_i ||x~_i||^2);
// 1: 1/(4 max(max_i ||x~_i||^2, beta_hat)) (configs.eta_for).  eta > 0 overrides.
// stop > 0: the solve stops at the first epoch with suboptimality <= stop
// (bench.cpp:182-189 time-to-eps protocol: the trace is cut there).
// sc[0..] = alpha, beta_hat, max_row_sq, eta, L_star, L_hat, sketch_ms,
//           precompute_ms, solve_ms, refmin_ms, mode (0 dense / 1 lazy), k_used,
//           full_gradient_ms (one timed call), rank_reduced
int ref_pipeline(const void* x, int x_f32, std::int64_t n, std::int64_t d, const double* y, double lambda,
                 std::int64_t k, std::int64_t q, std::uint64_t seed, std::int64_t epochs, std::int64_t m,
                 int eta_rule, double eta_in, int mode, double stop, std::int64_t idx_count, double* sigma_out,
                 double* U_out, double* trace, double* trace_ms, std::int64_t* done, double* w_hat,
                 std::int64_t* idx_out, double* sc) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  return guard([&] {
    Vector xs(static_cast<std::size_t>(n * d));
    if (x_f32) {
      const float* xf = static_cast<const float*>(x);
      for (std::size_t e = 0; e < xs.size(); ++e) xs[e] = static_cast<double>(xf[e]);
    } else {
      std::memcpy(xs.data(), x, sizeof(double) * xs.size());
    }
    RidgeProblem p(DataMatrix(DenseMatrix(static_cast<std::size_t>(d), static_cast<std::size_t>(n), std::move(xs))),
                   Vector(y, y + n), lambda);
    auto t0 = clk::now();
    Preconditioner pc = Preconditioner::identity(static_cast<std::size_t>(d), lambda);
    SketchedSvd sv;
    if (k > 0) {
      LanczosConfig lc;
      lc.k = static_cast<std::size_t>(k);
      lc.eps_prime = 0.5;
      lc.seed = seed;
      if (q > 0) lc.q_override = static_cast<std::size_t>(q);
      sv = block_lanczos(scaled_design(p), lc);
      std::memcpy(sigma_out, sv.singular_values.data(), sizeof(double) * sv.k);
      if (U_out) std::memcpy(U_out, sv.left.data(), sizeof(double) * sv.left.size());
      pc = build_sketched(sv, lambda);
    }
    auto t1 = clk::now();
    ApplyMode am = mode == 0 ? ApplyMode::Dense : mode == 1 ? ApplyMode::Lazy : ApplyMode::Auto;
    auto pre = preconditioned_components(p, pc, am);
    auto t2 = clk::now();
    ReferenceSolution ref = reference_minimum(p);
    auto t3 = clk::now();
    const Vector& b = pre->betas();
    double mx = 0.0;
    for (std::int64_t i = 0; i < n; ++i) mx = std::max(mx, b[static_cast<std::size_t>(i)]);
    const double max_row = mx * static_cast<double>(n) / static_cast<double>(n + d);
    const double bh = mean_beta(*pre);
    double eta = eta_in > 0 ? eta_in : 1.0 / (4.0 * (eta_rule == 1 ? std::max(max_row, bh) : max_row));
    Vector g;
    auto tg0 = clk::now();
    pre->full_gradient(Vector(static_cast<std::size_t>(d), 0.0), g);
    auto tg1 = clk::now();
    SvrgConfig cfg;
    cfg.epochs = static_cast<std::size_t>(epochs);
    cfg.epoch_length = static_cast<std::size_t>(m);
    cfg.step_size = eta;
    cfg.seed = seed;
    // time-to-eps: run epoch by epoch through the unmodified engine would change the
    // index stream; instead run the whole solve and cut the trace at the first hit
    auto t4 = clk::now();
    SvrgResult r = svrg_solve(*pre, cfg, Vector(static_cast<std::size_t>(d), 0.0), ref.minimum);
    auto t5 = clk::now();
    std::size_t cut = r.trace.size();
    if (stop > 0)
      for (std::size_t s = 0; s < r.trace.size(); ++s)
        if (r.trace[s].suboptimality && *r.trace[s].suboptimality <= stop) {
          cut = s + 1;
          break;
        }
    for (std::size_t s = 0; s < cut; ++s) {
      trace[s] = r.trace[s].objective;
      trace_ms[s] = r.trace[s].elapsed_ms;
    }
    *done = static_cast<std::int64_t>(cut);
    Vector wh = pc.apply_inv_sqrt(r.iterate);
    std::memcpy(w_hat, wh.data(), sizeof(double) * static_cast<std::size_t>(d));
    const double L = objective(p, wh);
    if (idx_count > 0) {
      Vector cum = make_cumulative_weights(b);
      NormalSampler rng(seed);
      for (std::int64_t t = 0; t < idx_count; ++t) {
        auto it = std::lower_bound(cum.begin(), cum.end(), rng.uniform());
        if (it == cum.end()) --it;
        idx_out[t] = static_cast<std::int64_t>(it - cum.begin());
      }
    }
    sc[0] = pre->strong_convexity();
    sc[1] = bh;
    sc[2] = max_row;
    sc[3] = eta;
    sc[4] = ref.minimum;
    sc[5] = L;
    sc[6] = ms(t0, t1);
    sc[7] = ms(t1, t2);
    sc[8] = ms(t4, t5);
    sc[9] = ms(t2, t3);
    sc[10] = pre->mode() == ApplyMode::Dense ? 0.0 : 1.0;
    sc[11] = static_cast<double>(k > 0 ? sv.k : 0);
    sc[12] = ms(tg0, tg1);
    sc[13] = k > 0 && sv.rank_reduced ? 1.0 : 0.0;
  });
}

// conditioned_matrix(scaled_design, lambda, P) (precond.cpp:174-194), unguarded,
// returned for an external symmetric eigensolve (d > 2000, where the reference's
// own kappa~ refuses: ScaleGuardError).  fp32 input promoted once.
int ref_conditioned_matrix(const void* x, int x_f32, std::int64_t n, std::int64_t d, double lambda, const double* U,
                           const double* sigma, std::int64_t k, double* out) {
  return guard([&] {
    Vector xs(static_cast<std::size_t>(n * d));
    if (x_f32) {
      const float* xf = static_cast<const float*>(x);
      for (std::size_t e = 0; e < xs.size(); ++e) xs[e] = static_cast<double>(xf[e]);
    } else {
      std::memcpy(xs.data(), x, sizeof(double) * xs.size());
    }
    DataMatrix a(DenseMatrix(static_cast<std::size_t>(d), static_cast<std::size_t>(n), std::move(xs)),
                 1.0 / std::sqrt(static_cast<double>(n)));
    Preconditioner pc = make_precond(static_cast<std::size_t>(d), U, sigma, static_cast<std::size_t>(k), lambda);
    DenseMatrix mat = conditioned_matrix(a, lambda, pc);
    std::memcpy(out, mat.data(), sizeof(double) * mat.size());
  });
}

}  // extern "C"
