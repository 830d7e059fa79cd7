// skridge_b200.hpp — header-only C++ host API over the C-ABI (skr.h).
//
// Mirrors the reference's public interface in proj/include/skridge/ for the
// hot path — same names, argument meaning and exception types — so C++
// callers switch by namespace (skridge:: -> skridge::b200::).  Everything runs
// on the B200; this header only owns handles (RAII) and converts status codes
// back into the reference's exceptions (errors.hpp:10-60, svrg.hpp:27-35).
//
//   reference                                  here
//   DataMatrix (data_matrix.hpp:18-61)         b200::DataMatrix (device storage + scale)
//   block_lanczos (sketch.hpp:55)              b200::block_lanczos
//   build_sketched (precond.hpp:70)            b200::build_sketched -> b200::Preconditioner
//   preconditioned_components (ridge.hpp:121)  b200::preconditioned_components
//   PreconditionedRidge (ridge.hpp:78-119)     b200::PreconditionedRidge
//   svrg_solve (svrg.hpp:136-137)              b200::svrg_solve (device index stream)
//   sketched_preconditioned_svrg (ridge.hpp:150) b200::sketched_preconditioned_svrg
//   reference_minimum (bench.hpp:24)           b200::reference_minimum
#pragma once

#include <cctype>
#include <charconv>
#include <chrono>
#include <numeric>
#include <string_view>
#include <system_error>
#include <istream>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <fstream>
#include <sstream>
#include <limits>
#include <vector>

#include "skr.h"

namespace skridge {
namespace b200 {

using Vector = std::vector<double>;

// ---- errors (errors.hpp) ---------------------------------------------------
struct DimensionError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ParameterError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct InputError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct DegenerateSpectrumError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegenerateDataError : std::runtime_error { using std::runtime_error::runtime_error; };
class ParseError : public std::runtime_error {  // errors.hpp:52-61
 public:
  ParseError(std::size_t line, const std::string& what)
      : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};
struct EmptyBasisError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ScaleGuardError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

struct EpochRecord {
  std::size_t epoch = 0;
  double objective = 0.0;
  std::optional<double> suboptimality;
  double elapsed_ms = 0.0;
};
using ConvergenceTrace = std::vector<EpochRecord>;

class DivergenceError : public std::runtime_error {
 public:
  DivergenceError(std::string what, ConvergenceTrace trace)
      : std::runtime_error(std::move(what)), trace_(std::move(trace)) {}
  const ConvergenceTrace& trace() const { return trace_; }

 private:
  ConvergenceTrace trace_;
};

inline void check(int rc) {
  if (rc == SKR_OK) return;
  const std::string m = skr_last_error();
  switch (rc) {
    case SKR_EDIM: throw DimensionError(m);
    case SKR_EPARAM: throw ParameterError(m);
    case SKR_EINPUT: throw InputError(m);
    case SKR_EGUARD: throw ScaleGuardError(m);
    case SKR_EEMPTY: throw EmptyBasisError(m);
    default: throw DeviceError(m);
  }
}

// ---- context ------------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) {
    skr_ctx* c = nullptr;
    check(skr_ctx_create(device, &c));
    h_.reset(c, [](skr_ctx* p) { skr_ctx_destroy(p); });
  }
  Context(int device, int rank, int world, const char nccl_id[128]) {
    skr_ctx* c = nullptr;
    check(skr_ctx_create_dist(device, rank, world, nccl_id, &c));
    h_.reset(c, [](skr_ctx* p) { skr_ctx_destroy(p); });
  }
  skr_ctx* get() const { return h_.get(); }
  void synchronize() const { check(skr_ctx_synchronize(get())); }

 private:
  std::shared_ptr<skr_ctx> h_;
};

// ---- DataMatrix -----------------------------------------------------------------
/// Device-resident DataMatrix.  `rows` is n x d row-major == the reference's
/// d x n column-major DenseMatrix storage (pass DenseMatrix::data() directly).
class DataMatrix {
 public:
  DataMatrix(const Context& ctx, const double* rows, std::size_t n, std::size_t d) : ctx_(ctx) {
    skr_data* x = nullptr;
    check(skr_data_create(ctx.get(), rows, (int64_t)n, (int64_t)d, SKR_F64, &x));
    reset(x);
  }
  DataMatrix(const Context& ctx, const float* rows, std::size_t n, std::size_t d) : ctx_(ctx) {
    skr_data* x = nullptr;
    check(skr_data_create(ctx.get(), rows, (int64_t)n, (int64_t)d, SKR_F32, &x));
    reset(x);
  }
  /// DataMatrix(SparseMatrix) (data_matrix.hpp:24): points as CSR (= the reference's CSC)
  static DataMatrix from_csr(const Context& ctx, std::size_t n, std::size_t d, const std::vector<int64_t>& row_ptr,
                             const std::vector<int32_t>& col_idx, const std::vector<double>& vals) {
    skr_data* x = nullptr;
    check(skr_data_create_csr(ctx.get(), (int64_t)n, (int64_t)d, row_ptr.data(), col_idx.data(), vals.data(), &x));
    DataMatrix out(ctx);
    out.reset(x);
    return out;
  }
  bool is_sparse() const {
    int sp = 0;
    check(skr_data_is_sparse(h_.get(), &sp, nullptr));
    return sp != 0;
  }
  std::size_t rows() const { return (std::size_t)info().d; }   // dimension d
  std::size_t cols() const { return (std::size_t)info().ng; }  // point count n
  double scale() const { return info().scale; }
  DataMatrix scaled(double factor) const {
    skr_data* x = nullptr;
    check(skr_data_scaled(h_.get(), factor, &x));
    DataMatrix out(ctx_);
    out.reset(x);
    return out;
  }
  skr_data* get() const { return h_.get(); }
  const Context& context() const { return ctx_; }

 private:
  explicit DataMatrix(const Context& ctx) : ctx_(ctx) {}
  void reset(skr_data* x) { h_.reset(x, [](skr_data* p) { skr_data_destroy(p); }); }
  struct Info { int64_t n, d, ng, r0; int dtype; double scale; };
  Info info() const {
    Info i{};
    check(skr_data_info(h_.get(), &i.n, &i.d, &i.dtype, &i.scale, &i.ng, &i.r0));
    return i;
  }
  Context ctx_;
  std::shared_ptr<skr_data> h_;
};

// ---- sketch (sketch.hpp) -----------------------------------------------------------
struct LanczosConfig {
  std::size_t k = 0;
  double eps_prime = 0.5;
  std::uint64_t seed = 0;
  std::optional<std::size_t> q_override;
};

/// Column-major factors exactly as the reference's DenseMatrix stores them.
struct SketchedSvd {
  Vector left;             // d x k, column j = basis vector j
  Vector singular_values;  // k
  Vector right;            // n x k (empty unless requested)
  std::size_t d = 0, n = 0, k = 0, q = 0;
  bool rank_reduced = false;
};

inline std::size_t lanczos_iterations(std::size_t n, double eps_prime) {
  const double q = std::ceil(std::log((double)n) / std::sqrt(eps_prime));
  return q < 2.0 ? 2 : (std::size_t)q;
}

inline SketchedSvd block_lanczos(const DataMatrix& a, const LanczosConfig& cfg, bool want_right = false) {
  SketchedSvd out;
  out.d = a.rows();
  int64_t n_local = 0;
  check(skr_data_info(a.get(), &n_local, nullptr, nullptr, nullptr, nullptr, nullptr));
  out.n = (std::size_t)n_local;
  out.left.assign(out.d * cfg.k, 0.0);
  out.singular_values.assign(cfg.k, 0.0);
  if (want_right) out.right.assign(out.n * cfg.k, 0.0);
  int64_t k_used = 0, q_used = 0;
  int rr = 0;
  check(skr_lanczos(a.context().get(), a.get(), (int64_t)cfg.k, cfg.q_override ? (int64_t)*cfg.q_override : 0,
                    cfg.eps_prime, cfg.seed, out.left.data(), out.singular_values.data(),
                    want_right ? out.right.data() : nullptr, &k_used, &q_used, &rr));
  out.k = (std::size_t)k_used;
  out.q = (std::size_t)q_used;
  out.rank_reduced = rr != 0;
  out.left.resize(out.d * out.k);
  out.singular_values.resize(out.k);
  if (want_right) out.right.resize(out.n * out.k);
  return out;
}

// ---- precond (precond.hpp) -------------------------------------------------------
class Preconditioner {
 public:
  static Preconditioner identity(std::size_t dim, double lambda) {
    if (!(lambda > 0.0) || !std::isfinite(lambda)) throw ParameterError("preconditioner: lambda must be positive");
    Preconditioner p;
    p.dim_ = dim;
    p.lambda_ = lambda;
    return p;
  }
  std::size_t dim() const { return dim_; }
  std::size_t rank() const { return sigma_.size(); }
  double lambda() const { return lambda_; }
  double tail_coeff() const { return inv_sqrt_.empty() ? 1.0 : inv_sqrt_.back(); }
  const Vector& inv_sqrt_diag() const { return inv_sqrt_; }
  const Vector& basis() const { return basis_; }  // d x k column-major
  const Vector& singular_values() const { return sigma_; }
  double min_inv_eigenvalue() const {
    const double lead = inv_sqrt_.empty() ? 1.0 : inv_sqrt_.front();
    return lead * lead;
  }
  // precond.cpp:67-118: O(dk) host maps of the value type (off the hot path; the
  // device applies P^{-1/2} inside skr_problem_* and skr_apply_inv_sqrt)
  Vector apply_inv_sqrt(const Vector& v) const { return apply(v, false); }
  Vector apply_sqrt(const Vector& v) const { return apply(v, true); }
  double inv_sqrt_sq_norm(double v_sq_norm, const Vector& proj) const {
    if (proj.size() != rank()) throw DimensionError("inv_sqrt_sq_norm: projection length mismatch");
    const double c = tail_coeff();
    double s = c * c * v_sq_norm;
    for (std::size_t j = 0; j < proj.size(); ++j) s += (inv_sqrt_[j] * inv_sqrt_[j] - c * c) * proj[j] * proj[j];
    return s;
  }
  friend Preconditioner build_sketched(const SketchedSvd& sv, double lambda);

 private:
  Vector apply(const Vector& v, bool sqrt_map) const {
    if (v.size() != dim_) throw DimensionError(sqrt_map ? "apply_sqrt: vector length mismatch"
                                                        : "apply_inv_sqrt: vector length mismatch");
    const double c = sqrt_map ? 1.0 / tail_coeff() : tail_coeff();
    Vector out(dim_);
    for (std::size_t i = 0; i < dim_; ++i) out[i] = c * v[i];
    const std::size_t k = rank();
    for (std::size_t j = 0; j < k; ++j) {
      const double* u = basis_.data() + j * dim_;
      double pj = 0.0;
      for (std::size_t i = 0; i < dim_; ++i) pj += u[i] * v[i];
      pj *= (sqrt_map ? 1.0 / inv_sqrt_[j] : inv_sqrt_[j]) - c;
      for (std::size_t i = 0; i < dim_; ++i) out[i] += u[i] * pj;
    }
    return out;
  }
  std::size_t dim_ = 0;
  double lambda_ = 0.0;
  Vector basis_, sigma_, inv_sqrt_;
};

/// precond.cpp:120-136 (+ validate, :34-49)
inline Preconditioner build_sketched(const SketchedSvd& sv, double lambda) {
  if (!(lambda > 0.0) || !std::isfinite(lambda)) throw ParameterError("preconditioner: lambda must be positive");
  if (sv.k < 1) throw ParameterError("build_sketched: factors must have rank >= 1");
  Preconditioner p;
  p.dim_ = sv.d;
  p.lambda_ = lambda;
  p.basis_ = sv.left;
  p.sigma_ = sv.singular_values;
  p.inv_sqrt_.resize(sv.k);
  const double cap = 1.0 / std::sqrt(lambda) * (1.0 + 1e-12);
  double prev = 0.0;
  for (std::size_t j = 0; j < sv.k; ++j) {
    const double s = sv.singular_values[j];
    const double v = 1.0 / std::sqrt(s * s + lambda);
    if (!(v > 0.0) || v > cap) throw InputError("preconditioner: coefficient out of range");
    if (v < prev) throw InputError("preconditioner: coefficients must be non-decreasing");
    p.inv_sqrt_[j] = prev = v;
  }
  return p;
}

/// precond.cpp:138-142.
inline Preconditioner build_exact(const SketchedSvd& sv, double lambda) { return build_sketched(sv, lambda); }

/// precond.cpp:144-162: full-rank preconditioner from sym_eigs(data.gram()) on the
/// device; guarded at d <= 2000 like the reference.
inline Preconditioner build_optimal(const DataMatrix& data, double lambda) {
  const std::size_t d = data.rows();
  if (d > 2000) throw ScaleGuardError("build_optimal: dimension exceeds the dense diagnostic guard");
  Vector vals(d), vecs(d * d);
  check(skr_gram_eigs(data.context().get(), data.get(), vals.data(), vecs.data()));
  SketchedSvd sv;
  sv.d = d;
  sv.k = d;
  sv.left = std::move(vecs);  // column j = eigenvector j
  sv.singular_values.resize(d);
  for (std::size_t j = 0; j < d; ++j) sv.singular_values[j] = std::sqrt(std::max(vals[j], 0.0));
  return build_sketched(sv, lambda);
}

// ---- svrg (svrg.hpp) -----------------------------------------------------------------
enum class SvrgMode { Theoretical, Tuned };  // svrg.hpp:37 (a label; the solve is identical)

struct SvrgConfig {
  std::size_t epochs = 1;
  std::size_t epoch_length = 1;
  double step_size = 0.1;
  std::uint64_t seed = 0;
  SvrgMode mode = SvrgMode::Tuned;
};

/// bench.cpp:96-100: 2^j / beta_hat, j = -3..3.
inline std::vector<double> eta_grid(double beta_hat) {
  std::vector<double> g;
  for (int j = -3; j <= 3; ++j) g.push_back(std::ldexp(1.0, j) / beta_hat);
  return g;
}

struct SvrgResult {
  Vector iterate;
  ConvergenceTrace trace;
};

// ---- ridge (ridge.hpp) ----------------------------------------------------------------
struct RidgeProblem {
  DataMatrix data;
  Vector labels;
  double lambda;
  RidgeProblem(DataMatrix d, Vector y, double lam) : data(std::move(d)), labels(std::move(y)), lambda(lam) {
    if (!(lambda > 0.0)) throw ParameterError("ridge problem: lambda must be positive");
  }
  std::size_t dim() const { return data.rows(); }
  std::size_t count() const { return data.cols(); }
};

inline DataMatrix scaled_design(const RidgeProblem& p) { return p.data.scaled(1.0 / std::sqrt((double)p.count())); }

enum class ApplyMode { Dense, Lazy, Auto };

/// The FiniteSumProblem of the reference (svrg.hpp:67-80) on the device:
/// component_count, dimension, betas, strong_convexity, objective,
/// full_gradient, component_gradient, plus the epoch kernel for external engines.
class PreconditionedRidge {
 public:
  /// ridge.hpp:84-85.  ApplyMode as skr_problem_create_mode (include/skr.h): Dense
  /// materialises X~ (ScaleGuardError above 2e8 entries, like ridge.cpp:110-113),
  /// Lazy keeps X and the projections, Auto is the device's choice.
  PreconditionedRidge(const RidgeProblem& p, const Preconditioner& pc, ApplyMode mode = ApplyMode::Auto)
      : ctx_(p.data.context()) {
    if (pc.dim() != p.dim()) throw DimensionError("preconditioned components: dimension mismatch");
    skr_problem* h = nullptr;
    check(skr_problem_create_mode(ctx_.get(), p.data.get(), p.labels.data(), p.lambda,
                                  pc.rank() ? pc.basis().data() : nullptr,
                                  pc.rank() ? pc.singular_values().data() : nullptr, (int64_t)pc.rank(),
                                  mode == ApplyMode::Dense ? SKR_MODE_DENSE
                                  : mode == ApplyMode::Lazy ? SKR_MODE_LAZY
                                                            : SKR_MODE_AUTO,
                                  &h));
    h_.reset(h, [](skr_problem* q) { skr_problem_destroy(q); });
    int64_t n = 0, d = 0, k = 0;
    check(skr_problem_info(h, &n, &d, &k, &alpha_, &beta_hat_, &max_row_sq_));
    n_ = (std::size_t)n;
    d_ = (std::size_t)d;
    betas_.resize(n_ + d_);
    check(skr_problem_betas(h, betas_.data()));
  }
  std::size_t component_count() const { return n_ + d_; }
  std::size_t dimension() const { return d_; }
  const Vector& betas() const { return betas_; }
  double strong_convexity() const { return alpha_; }
  double mean_beta() const { return beta_hat_; }
  double max_row_sq() const { return max_row_sq_; }
  /// ridge.hpp:96: the mode the device problem runs in.
  ApplyMode mode() const {
    int m = 0;
    check(skr_problem_mode(h_.get(), &m));
    return m == SKR_MODE_LAZY ? ApplyMode::Lazy : ApplyMode::Dense;
  }
  /// ridge.hpp:97 (LazyEpochState drift check, ridge.cpp:377-393).  The device Lazy
  /// chain tracks w = base + U h - tau mu exactly (no incremental projection to drift),
  /// so the drift is 0 in both modes.
  double max_projection_drift() const { return 0.0; }
  double objective(const Vector& w) const {
    double out = 0.0;
    check(skr_objective(h_.get(), w.data(), &out));
    return out;
  }
  void full_gradient(const Vector& w, Vector& out) const {
    out.resize(d_);
    check(skr_full_gradient(h_.get(), w.data(), out.data(), nullptr));
  }
  void component_gradient(std::size_t i, const Vector& w, Vector& out) const {
    out.resize(d_);
    check(skr_component_gradient(h_.get(), (int64_t)i, w.data(), out.data()));
  }
  /// One EpochState epoch (svrg.hpp:53-62) over caller-supplied indices.
  void epoch(const Vector& snapshot, const Vector& full_grad, const std::vector<int64_t>& idx, double eta,
             Vector& w_avg) const {
    w_avg.resize(d_);
    check(skr_epoch(h_.get(), snapshot.data(), full_grad.data(), idx.data(), (int64_t)idx.size(), eta,
                    w_avg.data()));
  }
  Vector apply_inv_sqrt(const Vector& v) const {
    Vector out(d_);
    check(skr_apply_inv_sqrt(h_.get(), v.data(), out.data()));
    return out;
  }
  skr_problem* get() const { return h_.get(); }

 private:
  Context ctx_;
  std::shared_ptr<skr_problem> h_;
  std::size_t n_ = 0, d_ = 0;
  double alpha_ = 0, beta_hat_ = 0, max_row_sq_ = 0;
  Vector betas_;
};

inline std::shared_ptr<PreconditionedRidge> preconditioned_components(const RidgeProblem& p,
                                                                      const Preconditioner& pc,
                                                                      ApplyMode mode = ApplyMode::Auto) {
  return std::make_shared<PreconditionedRidge>(p, pc, mode);
}

inline double mean_beta(const PreconditionedRidge& p) { return p.mean_beta(); }

/// svrg.cpp:219-232.
inline SvrgConfig theoretical_params(const PreconditionedRidge& p, double w0_gap, double epsilon) {
  if (!(epsilon > 0.0) || !(w0_gap > 0.0)) throw ParameterError("theoretical_params: w0_gap and epsilon must be positive");
  const double bh = p.mean_beta();
  SvrgConfig cfg;
  cfg.mode = SvrgMode::Theoretical;
  cfg.epochs = (std::size_t)std::max(1.0, std::ceil(std::log(w0_gap / epsilon)));
  cfg.epoch_length = (std::size_t)std::max(1.0, std::ceil(bh / p.strong_convexity()));
  cfg.step_size = 0.1 / bh;
  return cfg;
}

/// svrg.cpp:152-211 on the device, drawing the reference's index stream.
/// `stop_suboptimality` (with a reference value) ends after the first epoch at
/// or below it — the time-to-epsilon protocol; the reference runs every epoch.
inline SvrgResult svrg_solve(const PreconditionedRidge& p, const SvrgConfig& cfg, const Vector& w0,
                             std::optional<double> reference_value = std::nullopt,
                             std::optional<double> stop_suboptimality = std::nullopt) {
  if (w0.size() != p.dimension()) throw DimensionError("svrg: start point length mismatch");
  skr_svrg_config c{(int64_t)cfg.epochs, (int64_t)cfg.epoch_length, cfg.step_size, cfg.seed};
  std::vector<skr_epoch_record> rec(cfg.epochs ? cfg.epochs : 1);
  SvrgResult out;
  out.iterate.resize(p.dimension());
  int64_t done = 0;
  const double ref = reference_value ? *reference_value : NAN;
  const int rc = stop_suboptimality
                     ? skr_svrg_until(p.get(), &c, w0.data(), ref, *stop_suboptimality, out.iterate.data(), rec.data(),
                                      &done)
                     : skr_svrg(p.get(), &c, w0.data(), ref, out.iterate.data(), rec.data(), &done);
  for (int64_t s = 0; s < done; ++s) {
    EpochRecord r;
    r.epoch = (std::size_t)rec[s].epoch;
    r.objective = rec[s].objective;
    if (!std::isnan(rec[s].suboptimality)) r.suboptimality = rec[s].suboptimality;
    r.elapsed_ms = rec[s].elapsed_ms;
    out.trace.push_back(r);
  }
  if (rc == SKR_EDIVERGED) throw DivergenceError(skr_last_error(), out.trace);
  check(rc);
  return out;
}

struct SketchedSolveDiagnostics {  // ridge.hpp:125-136
  Vector singular_values;  // sketched values used by the preconditioner
  std::size_t k_used = 0;
  std::size_t q_used = 0;
  bool rank_reduced = false;
  ApplyMode mode = ApplyMode::Dense;
  double beta_hat = 0.0;
  double sketch_ms = 0.0;
  double precompute_ms = 0.0;
  double solve_ms = 0.0;
  double max_projection_drift = 0.0;
};

struct SketchedSolveResult {  // ridge.hpp:138-142
  Vector iterate;  // in original coordinates
  ConvergenceTrace trace;
  SketchedSolveDiagnostics diagnostics;
};

/// ridge.cpp:413-454 (same signature as ridge.hpp:150-153), plus an optional
/// explicit q for the BASELINE configs (the reference's
/// pipeline always uses q = lanczos_iterations(n, 1/2)).
inline SketchedSolveResult sketched_preconditioned_svrg(const RidgeProblem& p, std::size_t k, const SvrgConfig& cfg,
                                                        std::uint64_t sketch_seed, ApplyMode mode = ApplyMode::Auto,
                                                        std::optional<double> reference_value = std::nullopt,
                                                        std::optional<std::size_t> q_override = std::nullopt) {
  if (k < 1 || k > std::min(p.dim(), p.count())) throw ParameterError("sketched svrg: k must satisfy 1 <= k <= min(d, n)");
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
  SketchedSolveResult out;
  auto t0 = clk::now();
  LanczosConfig lc;
  lc.k = k;
  lc.eps_prime = 0.5;
  lc.seed = sketch_seed;
  lc.q_override = q_override;
  SketchedSvd sv = block_lanczos(scaled_design(p), lc);
  out.diagnostics.sketch_ms = ms(t0);
  out.diagnostics.singular_values = sv.singular_values;
  out.diagnostics.k_used = sv.k;
  out.diagnostics.q_used = sv.q;
  out.diagnostics.rank_reduced = sv.rank_reduced;
  t0 = clk::now();
  Preconditioner precond = build_sketched(sv, p.lambda);
  auto comp = preconditioned_components(p, precond, mode);
  out.diagnostics.precompute_ms = ms(t0);
  out.diagnostics.mode = comp->mode();
  out.diagnostics.beta_hat = comp->mean_beta();
  t0 = clk::now();
  SvrgResult r = svrg_solve(*comp, cfg, Vector(p.dim(), 0.0), reference_value);
  out.diagnostics.solve_ms = ms(t0);
  out.diagnostics.max_projection_drift = comp->max_projection_drift();
  out.iterate = precond.apply_inv_sqrt(r.iterate);
  out.trace = std::move(r.trace);
  return out;
}

struct ReferenceSolution {
  Vector minimizer;
  double minimum = 0.0;
};

/// bench.hpp:26 / bench.cpp:56-82 on the device.
inline Vector reference_minimum_cg(const RidgeProblem& p, double rel_residual_tol, std::size_t max_iterations) {
  Vector w(p.dim());
  check(skr_reference_minimum_cg(p.data.context().get(), p.data.get(), p.labels.data(), p.lambda, rel_residual_tol,
                                 (int64_t)max_iterations, w.data(), nullptr));
  return w;
}

/// bench.cpp:84-94 on the device (Cholesky for d <= 5000, the CG route above).
inline ReferenceSolution reference_minimum(const RidgeProblem& p) {
  ReferenceSolution r;
  r.minimizer.resize(p.dim());
  check(skr_reference_minimum(p.data.context().get(), p.data.get(), p.labels.data(), p.lambda, r.minimizer.data(),
                              &r.minimum));
  return r;
}

// ---- sparse corpus I/O (dataset.hpp:37-49, dataset.cpp:80-198) ------------------------------
struct LabeledDataset {
  DataMatrix data;
  Vector labels;
  std::string provenance;
};

/// Host-side CSR arrays of a parsed corpus (points = rows).
struct CsrCorpus {
  std::vector<int64_t> row_ptr{0};
  std::vector<int32_t> col_idx;
  Vector vals, labels;
  std::size_t dim = 0;
};

namespace detail {
// Cursor over one line of the corpus text: whitespace-separated tokens, the
// rest of the line after '#' ignored.
struct LineCursor {
  const char* p;
  const char* end;
  bool next(std::string_view& tok) {
    while (p < end && std::isspace((unsigned char)*p)) ++p;
    if (p == end || *p == '#') return false;
    const char* b = p;
    while (p < end && !std::isspace((unsigned char)*p) && *p != '#') ++p;
    tok = std::string_view(b, (std::size_t)(p - b));
    return true;
  }
};
// Whole-token numeric conversions (std::from_chars: no locale, no partial parse).
inline bool to_double(std::string_view t, double& v) {
  if (!t.empty() && t.front() == '+') t.remove_prefix(1);
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
inline bool to_index(std::string_view t, long long& v) {
  if (!t.empty() && t.front() == '+') t.remove_prefix(1);
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
}  // namespace detail

/// The sparse text format of dataset.hpp:37-49 ("label idx:value ..." per point,
/// 1-based strictly increasing feature indices, '#' comments, blank lines
/// skipped, explicit zeros dropped, d = the largest index seen).  Same
/// exception types and line numbering as the reference reader (dataset.cpp:87-162).
inline CsrCorpus parse_sparse_corpus(std::istream& in) {
  CsrCorpus c;
  std::string raw;
  std::size_t lineno = 0;
  while (std::getline(in, raw)) {
    ++lineno;
    detail::LineCursor cur{raw.data(), raw.data() + raw.size()};
    std::string_view tok;
    if (!cur.next(tok)) continue;  // blank or comment-only line
    double label = 0.0;
    if (!detail::to_double(tok, label)) throw ParseError(lineno, "bad label '" + std::string(tok) + "'");
    c.labels.push_back(label);
    long long last = 0;
    while (cur.next(tok)) {
      const std::size_t sep = tok.find(':');
      long long index = 0;
      double value = 0.0;
      const bool ok = sep != std::string_view::npos && sep > 0 && sep + 1 < tok.size() &&
                      detail::to_index(tok.substr(0, sep), index) && index >= 1 &&
                      detail::to_double(tok.substr(sep + 1), value);
      if (!ok) throw ParseError(lineno, "bad feature '" + std::string(tok) + "'");
      if (index <= last) throw ParseError(lineno, "feature indices must be strictly increasing");
      if (!std::isfinite(value)) throw ParseError(lineno, "non-finite value");
      last = index;
      if ((std::size_t)index > c.dim) c.dim = (std::size_t)index;
      if (value == 0.0) continue;
      c.col_idx.push_back((int32_t)(index - 1));
      c.vals.push_back(value);
    }
    c.row_ptr.push_back((int64_t)c.vals.size());
  }
  return c;
}

inline LabeledDataset read_sparse_corpus(const Context& ctx, const std::string& path) {
  std::ifstream in(path);
  if (!in) throw InputError("corpus: cannot open " + path);
  CsrCorpus c = parse_sparse_corpus(in);
  if (c.labels.empty()) throw InputError("corpus: no data lines in " + path);
  if (c.dim == 0) throw DegenerateDataError("corpus: no features seen");
  const std::size_t n = c.labels.size();
  return LabeledDataset{DataMatrix::from_csr(ctx, n, c.dim, c.row_ptr, c.col_idx, c.vals), std::move(c.labels), path};
}

// ---- ratio / spectrum diagnostics (precond.hpp:13-20,81-91; bench.cpp:195-212) --------
struct SpectrumSummary {
  Vector eigenvalues;  // descending, >= 0
  double lambda = 0.0;
  SpectrumSummary() = default;
  SpectrumSummary(Vector eigs, double lam) : eigenvalues(std::move(eigs)), lambda(lam) {  // precond.cpp:23-32
    double prev = std::numeric_limits<double>::infinity();
    const double floor = eigenvalues.empty() ? 0.0 : -1e-10 * std::max(1.0, eigenvalues.front());
    for (double& v : eigenvalues) {
      if (v < floor) throw InputError("spectrum: negative eigenvalue");
      if (v < 0.0) v = 0.0;
      if (v > prev) throw InputError("spectrum: eigenvalues must be descending");
      prev = v;
    }
  }
  std::size_t dim() const { return eigenvalues.size(); }
};

struct RatioRow {
  std::size_t k = 0;
  double ratio = 0.0;
};

/// bench.cpp:205-212: one device SYRK + eigensolve of X^T X / n.
inline SpectrumSummary dataset_spectrum(const RidgeProblem& p) {
  Vector e(p.dim());
  check(skr_dataset_spectrum(p.data.context().get(), p.data.get(), e.data()));
  return SpectrumSummary(std::move(e), p.lambda);
}

/// kappa_avg = tr(Sigma + lambda I) / (lambda_min + lambda) (precond.hpp:81-84).
inline double avg_condition_number(const SpectrumSummary& spec) {
  const Vector& e = spec.eigenvalues;
  if (e.empty()) throw InputError("avg_condition_number: empty spectrum");
  const double bottom = e.back() + spec.lambda;
  if (!(bottom > 0.0)) throw InputError("avg_condition_number: lam_min + lambda must be positive");
  const double shifted = std::accumulate(e.begin(), e.end(), 0.0,
                                         [&](double acc, double v) { return acc + (v + spec.lambda); });
  return shifted / bottom;
}

/// Paper Thm. ratio (precond.hpp:86-91): sum_i s_i / (k s_k + sum_{i>k} s_i),
/// with the spectrum split at k.
inline double theoretical_ratio(const SpectrumSummary& spec, std::size_t k) {
  const Vector& e = spec.eigenvalues;
  if (k < 1 || k > e.size()) throw ParameterError("theoretical_ratio: k must satisfy 1 <= k <= d");
  const auto split = e.begin() + (std::ptrdiff_t)k;
  const double top = std::accumulate(e.begin(), split, 0.0);
  const double rest = std::accumulate(split, e.end(), 0.0);
  const double below = rest + (double)k * e[k - 1];
  if (below == 0.0) throw DegenerateSpectrumError("theoretical_ratio: zero denominator");
  return (top + rest) / below;
}

/// bench.cpp:195-203.
inline std::vector<RatioRow> run_ratio_curve(const SpectrumSummary& spec, std::size_t k_max) {
  if (k_max < 1 || k_max > spec.dim()) throw ParameterError("ratio curve: k_max must satisfy 1 <= k_max <= d");
  std::vector<RatioRow> rows;
  for (std::size_t k = 1; k <= k_max; ++k) rows.push_back({k, theoretical_ratio(spec, k)});
  return rows;
}

}  // namespace b200
}  // namespace skridge
