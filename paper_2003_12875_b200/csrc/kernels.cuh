// Launch interface of the sm_100a kernels (kernels.cu).  All launches are
// asynchronous on the given stream and return the number of kernels launched
// (the reference's batch-mode call accounting, proj/include/ffit/eval.hpp:14-21:
// independent of the number of events).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace ffb {


struct NllLaunchInfo {
  int threads = 0;
  int events_per_thread = 0;
  int tile = 0;
  int ntiles = 0;
  int nchunks = 0;
  int grid = 0;
  int launches = 0;
  int jit = 0;  // 1: the formula-specialised (NVRTC) build ran
  int cached = 0;  // terms served by the launch-constant branch cache
};

// Bytes of scratch the fused NLL launch needs for (n events, P points).
std::size_t nll_scratch_bytes(long long n, int P, int ncols);

// Fused likelihood: for every point p in [0, P) and every event i in [0, n):
//   v = -log(plan(x_i; consts[p])) summed with compensated (Neumaier) block
//   partials, then a deterministic fixed-order pass over the partials.
// out[p] = (s, c) with NLL_events(p) = s + c; bad[p] = smallest event index with
// p <= 0 or non-finite (kNoInvalid if none).  `scratch` holds nll_scratch_bytes.
// `ks` selects the kernel build by the leaf kinds it contains (plan_kind_set);
// ev_start / ev_stop (may be null) are recorded around the fused kernel alone.
NllLaunchInfo launch_nll(const DevPlan& plan, const ColPtrs& cols, long long n,
                         const double* d_consts, int P, void* scratch, SumPair* d_out,
                         unsigned long long* d_bad, cudaStream_t stream, int ks,
                         cudaEvent_t ev_start = nullptr, cudaEvent_t ev_stop = nullptr);

// Fused likelihood + analytic gradient accumulators (plan.hpp DevGradPlan): for each
// point p and slot q, out[p * gp.nslots + q] = (s, c); bad as launch_nll.
NllLaunchInfo launch_nll_grad(const DevPlan& plan, const DevGradPlan& gp, const ColPtrs& cols,
                              long long n, const double* d_consts, int P, void* scratch,
                              SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream, int ks,
                              cudaEvent_t ev_start = nullptr, cudaEvent_t ev_stop = nullptr);
std::size_t nll_grad_scratch_bytes(long long n, int P, const DevPlan& plan, const DevGradPlan& gp);
// Whether the gradient pass's shared-memory layout fits a CTA.
bool grad_layout_fits(const DevPlan& plan, const DevGradPlan& gp);

// The smallest kernel build that covers the plan: 0 = Gaussian / Exponential /
// ArgusBG (p = 1/2, |c| <= 700), 1 = + Chebychev / Polynomial, 2 = everything
// (ChiSquare, JohnsonSU, general ArgusBG).  host_consts: the P rows about to launch.
int plan_kind_set(const DevPlan& plan, const double* host_consts, int P);

// Launch-constant branch cache (plan.hpp DevDerive): rewrites, in `plan`, the ArgusBG
// terms whose m0 and p = 1/2 are bitwise identical over the P rows about to launch
// into LK_ARGUS_CACHED terms whose data-only part the tile kernel computes once per
// tile.  Values are bit-identical to the uncached plan.  Returns the terms rewritten
// (0 when P is small enough for the streaming build, or FFB_NO_CONST_CACHE is set).
// A majority m0 (at least half the points and more than kStreamMaxP) makes the term
// LK_ARGUS_HYBRID instead: the rows of the points sharing it get the cache flag (c[5] = 1).
int cache_launch_constants(DevPlan& plan, double* host_consts, int P);

// Per-event values of the plan for one point (probabilities() when the plan is
// normalised, PdfSpec::eval_batch when not).
// h_row (the point's constant row on the host) selects the build per leaf-kind set; without it
// the generic kernel runs.
int launch_eval(const DevPlan& plan, const ColPtrs& cols, long long n, const double* d_consts,
                double* d_out, cudaStream_t stream, const double* h_row = nullptr);

// Combine R per-rank Neumaier pairs per point in fixed rank order (multi-GPU
// exchange step after an all-gather): in = R x P pairs, out = P pairs.
int launch_combine_ranks(const SumPair* d_in, int R, int P, SumPair* d_out, cudaStream_t stream);

// The sharded likelihood's exchange step (shard.cpp): d_in = R rank blocks of
// [rows pairs | P local first-invalid indices] (2 rows + P words each), gathered by one
// collective; d_out = rows pairs combined in rank order, d_bad = P global indices
// (d_offsets[r] = rank r's first global row).
int launch_combine_shards(const double* d_in, int R, int rows, int P, const long long* d_offsets, SumPair* d_out,
                          unsigned long long* d_bad, cudaStream_t stream);

// Fixed-order fold of `ntiles` partial pairs per row into one pair per row.
int launch_reduce(const SumPair* partial, int ntiles, int rows, SumPair* out, cudaStream_t stream);

// Target waves of the tile kernel's (tile x point-chunk) grid (FFB_NLL_WAVES).
int nll_waves();

// The tile kernel's grid for `items` work items on `slots` resident CTAs (FFB_NLL_PERSIST).
long long nll_grid(long long items, long long slots);

// Streaming multiprocessors of the current device (cached).
int device_sm_count();

// Test hook: which = 0 -> the kernel's exp, 1 -> its log, over n device doubles.
int launch_math_probe(int which, const double* d_in, double* d_out, long long n, cudaStream_t stream);

// DFMA-chain microbenchmark: returns FP64 FMA instructions per second measured
// with CUDA events on `stream` (the FP64 roofline denominator).
// Device-side numeric normalisation: the reference's adaptive Simpson of `plan` (an unnormalised
// sub-pdf plan, one row of constants per point) over [lo, hi] for P points; d_out[p] = integral,
// d_status[p] != 0 where the integrand was not finite.  Returns the launch count.
int launch_simpson(const DevPlan& plan, const double* d_rows, int P, double lo, double hi, double abs_tol,
                   double rel_tol, int max_depth, double* d_out, int* d_status, cudaStream_t stream);
double fp64_peak(cudaStream_t stream, float* ms_out);
double fp64_issue_probe(int others, cudaStream_t stream);

}  // namespace ffb
