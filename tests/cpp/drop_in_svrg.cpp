// TEST: the reference's own engine drives the GPU problem (drop-in check).
//
// Builds one instance with the reference's types, runs the UNMODIFIED
// reference svrg_solve (oracle/_ref) twice — on its own PreconditionedRidge
// (Dense) and on skridge_gpu::GpuPreconditionedRidge (B200) — with the same
// sketch, seed and step size, and prints both traces plus the maximum
// relative difference.  Exit 0 iff traces agree to 1e-10 relative.
#include <cmath>
#include <cstdio>

#include "skridge/random.hpp"
#include "skridge/ridge.hpp"
#include "skridge/sketch.hpp"
#include "skridge_gpu_problem.hpp"

int main() {
  using namespace skridge;
  const std::size_t d = 48, n = 600, k = 6;
  DenseMatrix x = gaussian_matrix(d, n, 3);  // d x n column-major == n x d rows
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < d; ++j) x(j, i) /= std::pow(double(j + 1), 1.1);
  NormalSampler s(4);
  Vector y(n);
  for (double& v : y) v = s.normal();
  const double lambda = 1e-3;
  RidgeProblem p(DataMatrix(x), y, lambda);
  LanczosConfig lc;
  lc.k = k;
  lc.seed = 5;
  lc.q_override = 3;
  SketchedSvd sv = block_lanczos(scaled_design(p), lc);
  auto cpu = preconditioned_components(p, build_sketched(sv, lambda), ApplyMode::Dense);

  b200::Context ctx(0);
  b200::RidgeProblem gp(b200::DataMatrix(ctx, x.data(), n, d), y, lambda);
  b200::SketchedSvd gsv;
  gsv.left = sv.left.entries();
  gsv.singular_values = sv.singular_values;
  gsv.d = d;
  gsv.k = sv.k;
  skridge_gpu::GpuPreconditionedRidge gpu(b200::preconditioned_components(gp, b200::build_sketched(gsv, lambda)));

  SvrgConfig cfg;
  cfg.epochs = 5;
  cfg.epoch_length = 2 * n;
  cfg.seed = 9;
  cfg.step_size = 0.25 / mean_beta(*cpu);
  Vector w0(d, 0.0);
  SvrgResult a = svrg_solve(*cpu, cfg, w0);
  SvrgResult b = svrg_solve(gpu, cfg, w0);
  double worst = 0.0;
  for (std::size_t e = 0; e < a.trace.size(); ++e) {
    const double r = std::abs(a.trace[e].objective - b.trace[e].objective) / std::abs(a.trace[e].objective);
    worst = std::max(worst, r);
    std::printf("epoch %zu  reference-cpu %.17g  reference-engine-on-b200 %.17g\n", e + 1, a.trace[e].objective,
                b.trace[e].objective);
  }
  double wi = 0.0;
  for (std::size_t j = 0; j < d; ++j) wi = std::max(wi, std::abs(a.iterate[j] - b.iterate[j]));
  std::printf("max_rel_trace_diff %.3e  max_abs_iterate_diff %.3e\n", worst, wi);
  return worst < 1e-10 ? 0 : 1;
}
