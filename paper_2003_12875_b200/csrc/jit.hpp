// Formula-specialised builds of the likelihood kernels for plans with Expression leaves
// (second stage).  The device interpreter (kernels_device.cuh
// expr_eval) runs any formula but pays a local-memory stack and an opcode switch per
// operation; here each formula of the plan becomes straight-line device code
// (`ffb_expr_batch`), the fused kernels of kernels_device.cuh are compiled around it at
// run time with NVRTC (sm_100a SASS), loaded through the driver API and launched with the
// same shapes as the static builds.  Modules are cached per (device, source).
//
// NVRTC and the driver are reached through dlopen / cudaGetDriverEntryPoint, so the
// library has no link-time dependency on either; when NVRTC is absent or a compile fails
// the engine keeps the interpreter (jit_status() says why).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kernels.cuh"
#include "plan_build.hpp"

namespace ffb {

// Launch-constant formula subtrees: a maximal subtree of an Expression term whose only
// inputs are x, constants and parameters bitwise identical over every point of the
// launch is computed once per staged tile into a shared-memory column (the tile kernel's
// launch-constant builds) and read by every point; values bit-identical to the
// uncached formula.  ArgusBG spelled as the reference's formula, m0 fixed:
// x*sqrt(1-(x/m0)^2) and 1-(x/m0)^2 are cached, each point computes exp(c*t) and a product.
struct HoistSlot {
  int term;        // plan term
  int prog;        // program offset (DevPlan::prog)
  int begin, end;  // instruction range of the subtree (inclusive), absolute indices
  int col;         // shared-memory column of the cached value
  int xcol;        // the term's data column
  int coff;        // the term's constant-row offset
};
struct ExprHoist {
  std::vector<HoistSlot> slots;
};
// The cacheable subtrees of a launch of P points (host constant rows `rows`, P x stride).
ExprHoist analyse_expr_hoist(const HostPlan& plan, const double* rows, int P);

// The generated formula functions for `plan` (prepended to kernels_device.cuh), with
// the cached-subtree variants when `hoist` lists any.
std::string jit_expression_source(const HostPlan& plan, const ExprHoist* hoist = nullptr);

// Whether the JIT path is switched on (default: on; FFB_NO_EXPR_JIT=1 or
// ffcu_expression_jit(0) turns it off).
bool jit_enabled();
void jit_enable(bool on);

// Compiles (or fetches from the cache) the kernels for `plan` on the current device;
// false (with the reason in jit_status()) when that is not possible.
bool jit_prepare(const HostPlan& plan);
std::string jit_status();

// As launch_nll, through the plan's formula-specialised kernels (jit_prepare first).
// h_rows: the launch's host constant rows (P x stride), for the launch-constant subtrees.
NllLaunchInfo launch_nll_jit(const HostPlan& plan, const ColPtrs& cols, long long n, const double* d_consts, int P,
                             void* scratch, SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream,
                             const double* h_rows, cudaEvent_t ev_start = nullptr, cudaEvent_t ev_stop = nullptr);

// Plan-specialised gradient pass (kernels_device.cuh nll_grad_spec_kernel): one point,
// single-column single-sum plans without Expression leaves, aligned column.
bool grad_spec_applies(const HostPlan& plan, const GradPlan& gp, const ColPtrs& cols, int P);
bool grad_spec_prepare(const HostPlan& plan, const GradPlan& gp, int ks);  // compile / cache
std::string grad_spec_text(const HostPlan& plan, const GradPlan& gp);
bool grad_spec_compile_only(const HostPlan& plan, const GradPlan& gp, int ks, std::string* log);
NllLaunchInfo launch_nll_grad_spec(const HostPlan& plan, const GradPlan& gp, const ColPtrs& cols, long long n,
                                   const double* d_consts, void* scratch, SumPair* d_out,
                                   unsigned long long* d_bad, cudaStream_t stream, int ks,
                                   cudaEvent_t ev_start = nullptr, cudaEvent_t ev_stop = nullptr);

// Plan-specialised likelihood builds (kernels_device.cuh eval_plan_spec): the tile
// kernel compiled at run time around the launch's term list (kinds, columns, flags,
// constant offsets as compile-time constants; the launch-constant rewrite included), and
// for single-column single-sum plans the few-point streaming kernel the same way; for
// launches of at least FFB_PLAN_SPEC_MIN (default 5e7) event-points of models without
// Expression leaves.  FFB_NO_PLAN_SPEC=1 turns it off.
std::string plan_spec_source(const DevPlan& launch);
// Sets the event-point threshold (v >= 0; -1 turns the builds off; other negatives only
// query); returns the previous setting.
double plan_spec_min_work(double v);
bool plan_spec_applies(const HostPlan& plan, const DevPlan& launch, long long n, int P);
bool plan_spec_prepare(const DevPlan& launch, int ks);  // compile / cache
bool plan_spec_compile_only(const DevPlan& launch, int ks, std::string* log);
NllLaunchInfo launch_nll_spec(const DevPlan& launch, const ColPtrs& cols, long long n, const double* d_consts, int P,
                              void* scratch, SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream, int ks,
                              int waves, cudaEvent_t ev_start = nullptr, cudaEvent_t ev_stop = nullptr);

// Compiles the plan's kernels (the generated formulas + kernels_device.cuh, both kernel
// instantiations) to sm_100a SASS without loading them: the CPU-side check of the
// generated code (NVRTC needs no GPU).
bool jit_compile_only(const HostPlan& plan, std::string* log, const ExprHoist* hoist = nullptr);

}  // namespace ffb
