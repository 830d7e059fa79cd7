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

}  // namespace skridge_gpu
