// TEST: the reference-typed drop-ins of integration/skridge_gpu_problem.hpp
// against the UNMODIFIED reference (oracle/_ref) on one instance built with the
// reference's own types:
//   * skridge_gpu::block_lanczos            vs skridge::block_lanczos (sketch.hpp:55)
//   * skridge_gpu::sketched_preconditioned_svrg vs skridge::sketched_preconditioned_svrg
//     (ridge.hpp:150-153): iterate, trace and every diagnostics field
//   * skridge_gpu::preconditioned_components(p, P, Lazy) driven by the reference's
//     svrg_solve vs the reference's own Lazy components (ridge.cpp:283-400).
// Prints the largest relative differences; exit 0 iff all gates hold.
#include <cmath>
#include <cstdio>

#include "skridge/bench.hpp"
#include "skridge/random.hpp"
#include "skridge/ridge.hpp"
#include "skridge/sketch.hpp"
#include "skridge_gpu_problem.hpp"

static double rel(const skridge::Vector& a, const skridge::Vector& b) {
  double m = 0.0, s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, std::fabs(a[i] - b[i]));
    s = std::max(s, std::fabs(b[i]));
  }
  return s > 0 ? m / s : m;
}

int main() {
  using namespace skridge;
  const std::size_t d = 40, n = 700, k = 6;
  DenseMatrix x = gaussian_matrix(d, n, 11);  // d x n column-major == n x d rows
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < d; ++j) x(j, i) /= std::pow(double(j + 1), 1.2);
  NormalSampler s(12);
  Vector y(n);
  for (double& v : y) v = s.normal();
  const double lambda = 1e-3;
  RidgeProblem p(DataMatrix(x), y, lambda);
  int bad = 0;
  auto gate = [&](bool ok, const char* what, double v) {
    std::printf("%-44s %.3e %s\n", what, v, ok ? "ok" : "FAIL");
    bad += !ok;
  };

  // block_lanczos (default q = lanczos_iterations(n, 1/2))
  LanczosConfig lc;
  lc.k = k;
  lc.seed = 5;
  SketchedSvd ref_sv = block_lanczos(scaled_design(p), lc);
  SketchedSvd gpu_sv = skridge_gpu::block_lanczos(scaled_design(p), lc);
  gate(gpu_sv.k == ref_sv.k && gpu_sv.q == ref_sv.q && gpu_sv.rank_reduced == ref_sv.rank_reduced,
       "block_lanczos k / q / rank_reduced", 0.0);
  gate(rel(gpu_sv.singular_values, ref_sv.singular_values) < 1e-10, "block_lanczos sigma~ (rel)",
       rel(gpu_sv.singular_values, ref_sv.singular_values));
  gate(rel(gpu_sv.left.entries(), ref_sv.left.entries()) < 1e-8, "block_lanczos U (sign-normalised, rel)",
       rel(gpu_sv.left.entries(), ref_sv.left.entries()));
  gate(rel(gpu_sv.right.entries(), ref_sv.right.entries()) < 1e-8, "block_lanczos V (rel)",
       rel(gpu_sv.right.entries(), ref_sv.right.entries()));

  // the composed pipeline
  Preconditioner pc = build_sketched(ref_sv, lambda);
  auto comp = preconditioned_components(p, pc, ApplyMode::Dense);
  double mx = 0.0;
  for (std::size_t i = 0; i < n; ++i) mx = std::max(mx, comp->betas()[i]);
  SvrgConfig cfg;
  cfg.epochs = 6;
  cfg.epoch_length = 2 * n;
  cfg.step_size = 1.0 / (4.0 * mx * double(n) / double(n + d));
  cfg.seed = 9;
  const double L_star = reference_minimum(p).minimum;
  SketchedSolveResult a = sketched_preconditioned_svrg(p, k, cfg, 5, ApplyMode::Auto, L_star);
  SketchedSolveResult b = skridge_gpu::sketched_preconditioned_svrg(p, k, cfg, 5, ApplyMode::Auto, L_star);
  Vector ta, tb;
  for (auto& r : a.trace) ta.push_back(r.objective);
  for (auto& r : b.trace) tb.push_back(r.objective);
  gate(ta.size() == tb.size() && rel(tb, ta) < 1e-8, "pipeline trace objectives (rel)", rel(tb, ta));
  gate(rel(b.iterate, a.iterate) < 1e-8, "pipeline iterate w^ (rel)", rel(b.iterate, a.iterate));
  gate(rel(b.diagnostics.singular_values, a.diagnostics.singular_values) < 1e-10, "diagnostics sigma~",
       rel(b.diagnostics.singular_values, a.diagnostics.singular_values));
  gate(b.diagnostics.k_used == a.diagnostics.k_used && b.diagnostics.q_used == a.diagnostics.q_used &&
           b.diagnostics.rank_reduced == a.diagnostics.rank_reduced && b.diagnostics.mode == a.diagnostics.mode,
       "diagnostics k_used / q_used / rank_reduced / mode", 0.0);
  gate(std::fabs(b.diagnostics.beta_hat - a.diagnostics.beta_hat) <= 1e-10 * a.diagnostics.beta_hat,
       "diagnostics beta_hat (rel)", std::fabs(b.diagnostics.beta_hat - a.diagnostics.beta_hat) / a.diagnostics.beta_hat);
  gate(b.diagnostics.max_projection_drift == 0.0 && a.diagnostics.max_projection_drift == 0.0,
       "diagnostics max_projection_drift (Dense: 0)", b.diagnostics.max_projection_drift);
  bool sub = true;
  for (std::size_t e = 0; e < a.trace.size() && e < b.trace.size(); ++e)
    sub = sub && a.trace[e].suboptimality.has_value() == b.trace[e].suboptimality.has_value();
  gate(sub, "trace suboptimality presence", 0.0);

  // Lazy mode through the device Lazy chain, driven by the reference engine
  auto ref_lazy = preconditioned_components(p, pc, ApplyMode::Lazy);
  auto gpu_lazy = skridge_gpu::preconditioned_components(p, pc, ApplyMode::Lazy);
  gate(gpu_lazy->device().mode() == b200::ApplyMode::Lazy, "device mode() == Lazy", 0.0);
  gate(rel(gpu_lazy->betas(), ref_lazy->betas()) < 1e-12, "Lazy betas (rel)", rel(gpu_lazy->betas(), ref_lazy->betas()));
  SvrgResult rl = svrg_solve(*ref_lazy, cfg, Vector(d, 0.0), L_star);
  SvrgResult gl = svrg_solve(*gpu_lazy, cfg, Vector(d, 0.0), L_star);
  Vector tl, tg;
  for (auto& r : rl.trace) tl.push_back(r.objective);
  for (auto& r : gl.trace) tg.push_back(r.objective);
  gate(rel(tg, tl) < 1e-8, "Lazy traces, reference engine (rel)", rel(tg, tl));
  std::printf("%d gate(s) failed\n", bad);
  return bad == 0 ? 0 : 1;
}
