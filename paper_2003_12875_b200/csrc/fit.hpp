// Fit drivers on top of the GPU likelihood.
//
//  * fit_nelder_mead: the reference minimiser (proj/src/fit.cpp:86-251, Nelder-Mead
//    in sine-transformed space, central-difference Hessian) with every batch of
//    independent points -- the initial simplex, a shrink, the 1+2d+2d(d-1) Hessian
//    points -- issued as ONE multi-point launch.
//  * fit_gradient: Minuit-style quasi-Newton (BFGS).  Gradients from the fused NLL +
//    gradient pass (one point per iteration) when the model's
//    layout fits it, else central finite differences (one launch of 2d+1 points per
//    iteration).
#pragma once

#include <string>
#include <vector>

#include "engine.hpp"

namespace ffb {

struct FitOptions {
  double tolerance = 1e-8;  // NM: simplex NLL spread; gradient: EDM threshold
  int max_iterations = 10000;
  bool record_trace = false;
  double fd_step = 1e-4;    // u-space step for gradients / Hessian
  bool analytic_gradient = true;  // fit_gradient: the fused NLL + gradient pass when available
};

struct FittedParameter {
  std::string name;
  double value = 0.0;
  double uncertainty = 0.0;
};

struct FitResult {
  bool converged = false;
  double nll_min = 0.0;
  std::vector<FittedParameter> parameters;
  unsigned long long n_nll_calls = 0;   // parameter points evaluated
  unsigned long long n_launches = 0;    // multi-point launches (batches)
  unsigned long long kernel_launches = 0;
  int iterations = 0;
  double wall_seconds = 0.0;
  bool uncertainties_valid = true;
  bool analytic_gradient = false;  // fit_gradient used the fused gradient pass
  double edm = 0.0;                // fit_gradient: last estimated distance to minimum
  std::vector<double> trace;
};

double bound_transform(double u, double lower, double upper);
double bound_transform_inverse(double p, double lower, double upper);

// What a fit driver evaluates: the NLL (and, where the model's layout allows, its analytic
// gradient) at a batch of parameter points, as ONE launch per batch.  EngineSource is one
// device; ShardGroup (shard.hpp) an event-sharded likelihood over several GPUs whose batches
// cost one collective each.
class LikelihoodSource {
 public:
  virtual ~LikelihoodSource() = default;
  virtual NllResult nll_points(const double* thetas, int P) = 0;
  virtual NllGradResult nll_grad_points(const double* thetas, int P) = 0;
  virtual bool grad_ok() = 0;
  // device buffers for batches of up to P_nll likelihood / P_grad gradient points
  virtual void reserve(int P_nll, int P_grad) = 0;
};

class EngineSource : public LikelihoodSource {
 public:
  EngineSource(Engine& e, const DeviceDataset& ds) : e_(e), ds_(ds) {}
  NllResult nll_points(const double* thetas, int P) override { return e_.nll_points(ds_, thetas, P); }
  NllGradResult nll_grad_points(const double* thetas, int P) override { return e_.nll_grad_points(ds_, thetas, P); }
  bool grad_ok() override { return e_.grad_plan().ok; }
  void reserve(int P_nll, int P_grad) override { e_.reserve(ds_, P_nll, P_grad); }

 private:
  Engine& e_;
  const DeviceDataset& ds_;
};

FitResult fit_nelder_mead(Model& m, LikelihoodSource& src, const FitOptions& o);
FitResult fit_gradient(Model& m, LikelihoodSource& src, const FitOptions& o);

inline FitResult fit_nelder_mead(Model& m, Engine& e, const DeviceDataset& ds, const FitOptions& o) {
  EngineSource src(e, ds);
  return fit_nelder_mead(m, src, o);
}
inline FitResult fit_gradient(Model& m, Engine& e, const DeviceDataset& ds, const FitOptions& o) {
  EngineSource src(e, ds);
  return fit_gradient(m, src, o);
}

// Central-difference Hessian in u-space at the model's current values (one
// launch of 1+2d+2d(d-1) points) -> uncertainties written into the model.
bool hessian_uncertainties(Model& m, LikelihoodSource& src, double h, FitResult& r);

}  // namespace ffb
