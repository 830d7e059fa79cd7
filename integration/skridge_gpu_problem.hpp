// skridge_gpu_problem.hpp — the drop-in plugin for the reference engine.
//
// Compiles against the REFERENCE headers (proj/include/skridge/svrg.hpp) and
// include/skridge_b200.hpp.  GpuPreconditionedRidge is a sibling of the
// reference's PreconditionedRidge (which is `final`, ridge.hpp:78) implementing
// the same FiniteSumProblem virtuals (svrg.hpp:67-80) on the B200, so the
// reference's own svrg_solve (svrg.cpp:152-211) drives it unchanged:
//   * betas / strong_convexity / objective / full_gradient / component_gradient
//     are device calls through the C-ABI;
//   * make_epoch_state returns GpuEpochState, whose step(i, eta, inv_nq) only
//     records i (the engine draws i from its own NormalSampler stream,
//     svrg.cpp:174,192, so the index sequence is the reference's by
//     construction) and whose epoch_average runs the whole epoch as one
//     persistent inner-loop kernel (K10).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include <cmath>
#include <optional>

#include "skridge/data_matrix.hpp"
#include "skridge/precond.hpp"
#include "skridge/ridge.hpp"
#include "skridge/sketch.hpp"
#include "skridge/svrg.hpp"
#include "skridge_b200.hpp"

namespace skridge_gpu {

class GpuEpochState final : public skridge::EpochState {
 public:
  explicit GpuEpochState(const skridge::b200::PreconditionedRidge& p) : p_(p) {}
  void begin_epoch(const skridge::Vector& snapshot, const skridge::Vector& full_grad) override {
    snapshot_ = snapshot;
    mu_ = full_grad;
    idx_.clear();
  }
  void step(std::size_t index, double eta, double /*inv_nq: recomputed on the device*/) override {
    idx_.push_back(static_cast<int64_t>(index));
    eta_ = eta;
  }
  void epoch_average(skridge::Vector& out) override { p_.epoch(snapshot_, mu_, idx_, eta_, out); }

 private:
  const skridge::b200::PreconditionedRidge& p_;
  skridge::Vector snapshot_, mu_;
  std::vector<int64_t> idx_;
  double eta_ = 0.0;
};

class GpuPreconditionedRidge final : public skridge::FiniteSumProblem {
 public:
  explicit GpuPreconditionedRidge(std::shared_ptr<skridge::b200::PreconditionedRidge> p) : p_(std::move(p)) {}
  std::size_t component_count() const override { return p_->component_count(); }
  std::size_t dimension() const override { return p_->dimension(); }
  const skridge::Vector& betas() const override { return p_->betas(); }
  double strong_convexity() const override { return p_->strong_convexity(); }
  double objective(const skridge::Vector& w) const override { return p_->objective(w); }
  void full_gradient(const skridge::Vector& w, skridge::Vector& out) const override { p_->full_gradient(w, out); }
  void component_gradient(std::size_t i, const skridge::Vector& w, skridge::Vector& out) const override {
    p_->component_gradient(i, w, out);
  }
  std::unique_ptr<skridge::EpochState> make_epoch_state() const override {
    return std::make_unique<GpuEpochState>(*p_);
  }
  const skridge::b200::PreconditionedRidge& device() const { return *p_; }

 private:
  std::shared_ptr<skridge::b200::PreconditionedRidge> p_;
};

// ---- reference-typed drop-ins ------------------------------------
// Same signatures and value types as the reference's sketch.hpp:55, ridge.hpp:121-123
// and ridge.hpp:150-153, computed on the B200 through the C-ABI.  Callers keep the
// reference's DataMatrix / RidgeProblem / SketchedSvd / Preconditioner / SvrgConfig.

/// The device context the drop-ins use (one per process; device 0).
inline const skridge::b200::Context& device_context() {
  static const skridge::b200::Context ctx(0);
  return ctx;
}

/// skridge::DataMatrix (dense d x n column-major == n x d rows, or CSC over points
/// == CSR over points) -> device DataMatrix with the same logical entries.
/// fold_scale: upload scale * stored (a problem's data handle must be unscaled);
/// otherwise keep the scale on the handle, as scaled_design does (ridge.cpp:54-56).
inline skridge::b200::DataMatrix to_device(const skridge::DataMatrix& a,
                                           const skridge::b200::Context& ctx = device_context(),
                                           bool fold_scale = false) {
  namespace b = skridge::b200;
  const std::size_t d = a.rows(), n = a.cols();
  const double s = a.scale();
  const bool fold = fold_scale && s != 1.0;
  if (const skridge::DenseMatrix* m = a.dense()) {
    if (fold) {
      std::vector<double> v(m->entries());
      for (double& e : v) e *= s;
      return b::DataMatrix(ctx, v.data(), n, d);
    }
    b::DataMatrix x(ctx, m->data(), n, d);
    return s == 1.0 ? x : x.scaled(s);
  }
  const skridge::SparseMatrix* sp = a.sparse();
  std::vector<int64_t> rp(sp->col_ptr().begin(), sp->col_ptr().end());
  std::vector<int32_t> ci(sp->row_idx().begin(), sp->row_idx().end());
  std::vector<double> vals(sp->values());
  if (fold)
    for (double& e : vals) e *= s;
  b::DataMatrix x = b::DataMatrix::from_csr(ctx, n, d, rp, ci, vals);
  return (s == 1.0 || fold) ? x : x.scaled(s);
}

inline skridge::SketchedSvd to_reference(const skridge::b200::SketchedSvd& sv) {
  skridge::SketchedSvd out;
  out.left = skridge::DenseMatrix(sv.d, sv.k, sv.left);  // both column-major d x k
  out.singular_values = sv.singular_values;
  if (!sv.right.empty()) out.right = skridge::DenseMatrix(sv.n, sv.k, sv.right);
  out.k = sv.k;
  out.q = sv.q;
  out.rank_reduced = sv.rank_reduced;
  return out;
}

inline skridge::b200::SketchedSvd from_reference(const skridge::SketchedSvd& sv) {
  skridge::b200::SketchedSvd out;
  out.d = sv.left.rows();
  out.k = sv.k;
  out.n = sv.right.rows();
  out.q = sv.q;
  out.left = sv.left.entries();
  out.singular_values = sv.singular_values;
  out.right = sv.right.entries();
  out.rank_reduced = sv.rank_reduced;
  return out;
}

/// Device Preconditioner carrying the same map as a reference Preconditioner: the
/// basis is copied and sigma~_j recovered from the coefficients,
/// sigma~_j^2 = 1/D_j^2 - lambda (the device rebuilds D_j = 1/sqrt(sigma~_j^2 + lambda)).
inline skridge::b200::Preconditioner from_reference(const skridge::Preconditioner& pc) {
  if (pc.rank() == 0) return skridge::b200::Preconditioner::identity(pc.dim(), pc.lambda());
  skridge::b200::SketchedSvd sv;
  sv.d = pc.dim();
  sv.k = pc.rank();
  sv.left = pc.basis().entries();
  sv.singular_values.resize(sv.k);
  for (std::size_t j = 0; j < sv.k; ++j) {
    const double Dj = pc.inv_sqrt_diag()[j];
    sv.singular_values[j] = std::sqrt(std::max(1.0 / (Dj * Dj) - pc.lambda(), 0.0));
  }
  return skridge::b200::build_sketched(sv, pc.lambda());
}

inline skridge::b200::RidgeProblem to_device(const skridge::RidgeProblem& p,
                                             const skridge::b200::Context& ctx = device_context()) {
  return skridge::b200::RidgeProblem(to_device(p.data, ctx, /*fold_scale=*/true), p.labels, p.lambda);
}

inline skridge::b200::ApplyMode to_device(skridge::ApplyMode m) {
  return m == skridge::ApplyMode::Dense  ? skridge::b200::ApplyMode::Dense
         : m == skridge::ApplyMode::Lazy ? skridge::b200::ApplyMode::Lazy
                                         : skridge::b200::ApplyMode::Auto;
}

/// sketch.hpp:55 on the device (right factors included, as the reference returns them).
inline skridge::SketchedSvd block_lanczos(const skridge::DataMatrix& a, const skridge::LanczosConfig& cfg) {
  skridge::b200::LanczosConfig lc;
  lc.k = cfg.k;
  lc.eps_prime = cfg.eps_prime;
  lc.seed = cfg.seed;
  lc.q_override = cfg.q_override;
  return to_reference(skridge::b200::block_lanczos(to_device(a), lc, /*want_right=*/true));
}

/// ridge.hpp:121-123 on the device: a FiniteSumProblem the reference's svrg_solve drives.
inline std::shared_ptr<GpuPreconditionedRidge> preconditioned_components(const skridge::RidgeProblem& p,
                                                                         const skridge::Preconditioner& pc,
                                                                         skridge::ApplyMode mode = skridge::ApplyMode::Auto) {
  return std::make_shared<GpuPreconditionedRidge>(
      skridge::b200::preconditioned_components(to_device(p), from_reference(pc), to_device(mode)));
}

/// ridge.hpp:150-153 on the device, returning the reference's SketchedSolveResult.
inline skridge::SketchedSolveResult sketched_preconditioned_svrg(const skridge::RidgeProblem& p, std::size_t k,
                                                                 const skridge::SvrgConfig& cfg,
                                                                 std::uint64_t sketch_seed,
                                                                 skridge::ApplyMode mode = skridge::ApplyMode::Auto,
                                                                 std::optional<double> reference_value = std::nullopt) {
  skridge::b200::SvrgConfig c;
  c.epochs = cfg.epochs;
  c.epoch_length = cfg.epoch_length;
  c.step_size = cfg.step_size;
  c.seed = cfg.seed;
  const auto r = skridge::b200::sketched_preconditioned_svrg(to_device(p), k, c, sketch_seed, to_device(mode),
                                                             reference_value);
  skridge::SketchedSolveResult out;
  out.iterate = r.iterate;
  for (const auto& e : r.trace) {
    skridge::EpochRecord x;
    x.epoch = e.epoch;
    x.objective = e.objective;
    x.suboptimality = e.suboptimality;
    x.elapsed_ms = e.elapsed_ms;
    out.trace.push_back(x);
  }
  auto& dg = out.diagnostics;
  dg.singular_values = r.diagnostics.singular_values;
  dg.k_used = r.diagnostics.k_used;
  dg.q_used = r.diagnostics.q_used;
  dg.rank_reduced = r.diagnostics.rank_reduced;
  dg.mode = r.diagnostics.mode == skridge::b200::ApplyMode::Lazy ? skridge::ApplyMode::Lazy : skridge::ApplyMode::Dense;
  dg.beta_hat = r.diagnostics.beta_hat;
  dg.sketch_ms = r.diagnostics.sketch_ms;
  dg.precompute_ms = r.diagnostics.precompute_ms;
  dg.solve_ms = r.diagnostics.solve_ms;
  dg.max_projection_drift = r.diagnostics.max_projection_drift;
  return out;
}

}  // namespace skridge_gpu
