// Host side of the evaluation plan: flattening (once per model) and the per-point
// constant builder (once per parameter point, vectorised over the P points of a
// launch).  See plan.hpp for the canonical form.
#pragma once

#include <string>
#include <vector>

#include "model.hpp"
#include "plan.hpp"

namespace ffb {

struct HostPlan {
  DevPlan dev{};
  int pdf = -1;            // the pdf this plan evaluates
  bool normalized = true;  // true: p = unnorm / N (the likelihood); false: eval_batch
  std::vector<int> col_obs;  // compact column slot -> observable index
  std::vector<int> term_pdf; // leaf pdf of each term
  std::vector<ExprInstr> programs;  // Expression leaves' device programs (DevPlan::prog)
};

// Slot layout of the fused NLL + gradient pass (plan.hpp DevGradPlan) for the
// model's free parameters.  `ok` false (with the reason) when the layout exceeds the
// device limits; then only finite-difference gradients are available.
struct GradPlan {
  bool ok = false;
  std::string why;
  DevGradPlan dev{};
  std::vector<int> slot_param;  // B slot -> parameter index (-1 for slot 0 / A slots)
  std::vector<int> a_slot;      // term -> its A slot
};

GradPlan compile_grad_plan(const HostPlan& plan, const Model& m);

// d coef_c / d theta_j for every term of the plan (the coefficients exactly as
// build_constants writes them, extra_scale included): the constant builder's
// traversal differentiated forward, with the normalisation derivatives of
// model_grad.cpp.
std::vector<double> coef_derivatives(const HostPlan& plan, const Model& m, const double* theta, int j,
                                     double extra_scale);

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
