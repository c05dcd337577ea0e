// Host side of the evaluation plan: flattening (once per model) and the per-point
// constant builder (once per parameter point, vectorised over the P points of a
// launch).  See plan.hpp for the canonical form.
#pragma once

#include <vector>

#include "model.hpp"
#include "plan.hpp"

namespace ffb {

struct HostPlan {
  DevPlan dev{};
  int pdf = -1;            // the pdf this plan evaluates
  bool normalized = true;  // true: p = unnorm / N (the likelihood); false: eval_batch
  std::vector<int> col_obs;  // compact column slot -> observable index
};

// Flattens `pdf` (the model root for the likelihood).  Throws Usage for trees
// outside the canonical form (e.g. a ProdPdf nested in a 1-D sum).
HostPlan compile_plan(const Model& m, int pdf, bool normalized);

// Writes one row of `plan.dev.stride` constants for parameter vector theta
// (all model parameters, declaration order).  Validates the point first
// (check_params, proj/src/pdfs.cpp:127-176) and computes every normalisation.
// `extra_scale` multiplies the whole density (the likelihood kernel passes
// 2^kPScaleLog2, see plan.hpp; exact, a power of two).
void build_constants(const HostPlan& plan, const Model& m, const double* theta, double* row,
                     double extra_scale = 1.0);

}  // namespace ffb
