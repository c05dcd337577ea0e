// Host orchestration of the GPU likelihood: HBM-resident SoA datasets and the
// per-model engine that builds per-point constants, uploads them and launches
// the fused kernels.  This is where the reference's nll_batch / probabilities /
// eval_batch (proj/src/eval.cpp:119-192, proj/src/pdfs.cpp:212-269) cross to the
// device.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "model.hpp"
#include "plan_build.hpp"

namespace ffb {

// Immutable SoA event table resident in HBM: one contiguous fp64 column per
// observable (the reference's DataSet, proj/include/ffit/dataset.hpp:20-51).
struct DeviceDataset {
  int device = 0;
  long long n = 0;
  std::vector<std::string> names;
  std::vector<double*> cols;
  bool owns = true;
  std::shared_ptr<DeviceDataset> parent;  // keeps the storage of a view alive

  DeviceDataset() = default;
  DeviceDataset(const DeviceDataset&) = delete;
  DeviceDataset& operator=(const DeviceDataset&) = delete;
  ~DeviceDataset();

  int column_index(const std::string& name) const;  // -1 if absent

  // Owned, uninitialised columns of n rows (padded to whole 2048-event tiles).
  static std::shared_ptr<DeviceDataset> allocate(const std::vector<std::string>& names, long long n);
  static std::shared_ptr<DeviceDataset> upload(const std::vector<std::string>& names,
                                               const std::vector<const double*>& host_cols,
                                               long long n);
  static std::shared_ptr<DeviceDataset> view(const std::vector<std::string>& names,
                                             const std::vector<const double*>& dev_cols,
                                             long long n, int device);
  void copy_from_host(const std::vector<const double*>& host_cols);
  void copy_from_host_async(const std::vector<const double*>& host_cols, cudaStream_t stream);
  void download(int col, double* host_out) const;
};

void cuda_check(cudaError_t e, const char* what);

class DeviceGuard {
 public:
  explicit DeviceGuard(int device);
  ~DeviceGuard();

 private:
  int prev_ = 0;
  bool switched_ = false;
};

// Parameter points per device launch (larger batches are split into launches of this size).
constexpr int kMaxPointsPerLaunch = 512;

struct NllResult {
  std::vector<double> value;         // s + c + extended term; +inf if an event is invalid
  std::vector<SumPair> pairs;        // the raw per-point Neumaier pairs (events only)
  std::vector<long long> first_invalid;
  unsigned long long launches = 0;
};

// Fused NLL + gradient: value[p] as NllResult; grad[p * npar + j] = dNLL/dtheta_j
// for the free parameters (0 for constant ones); NaN gradients with +inf values.
struct NllGradResult {
  std::vector<double> value;
  std::vector<double> grad;
  std::vector<long long> first_invalid;
  unsigned long long launches = 0;
  int nslots = 0;
  std::vector<SumPair> slots;  // raw per-point accumulators (P x nslots, events only)
};

class Engine {
 public:
  explicit Engine(const Model& m);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Synchronous: P points (rows of all model parameters, declaration order).
  NllResult nll_points(const DeviceDataset& ds, const double* thetas, int P);

  // Asynchronous on `stream`: results stay on the device (d_pairs: P pairs,
  // d_bad: P indices, kNoInvalid if none).  Host-side constant building and the
  // constant upload are part of the call.  Returns kernels launched.
  // upload_stream (optional): where the constant rows are copied (a caller's copy stream).
  int nll_points_device(const DeviceDataset& ds, const double* thetas, int P, SumPair* d_pairs,
                        unsigned long long* d_bad, cudaStream_t stream, cudaStream_t upload_stream = nullptr);

  // Analytic gradient in the same pass over the events (plan.hpp DevGradPlan):
  // P points, one launch pair per <= 512 points.  Throws Usage when the model's
  // gradient layout does not fit the device pass (grad_plan().why).
  NllGradResult nll_grad_points(const DeviceDataset& ds, const double* thetas, int P);

  // Host finish of the gradient from the (rank-combined) slot sums: P x nslots
  // values in `slot_sums`, n_events the global event count.
  void grad_finish(const double* thetas, int P, const double* slot_sums, double n_events,
                   double* values, double* grads);

  // Sizes the device buffers for launches of up to P_nll likelihood points and P_grad
  // gradient points on `ds` (fits call it before their clock starts).
  void reserve(const DeviceDataset& ds, int P_nll, int P_grad);

  // Current gradient layout (recompiled when parameters change constness).
  const GradPlan& grad_plan();
  bool last_grad_jit() const { return last_grad_jit_ != 0; }

  // probabilities() (proj/src/eval.cpp:174-192): normalised per-event values.
  void probabilities(const DeviceDataset& ds, const double* theta, double* out, bool out_on_device,
                     cudaStream_t stream = nullptr);

  // PdfSpec::eval_batch (proj/src/pdfs.cpp:212-269): unnormalised values of a
  // (sub-)pdf of the model.
  void eval_batch(int pdf, const DeviceDataset& ds, const double* theta, double* out,
                  bool out_on_device, cudaStream_t stream = nullptr);

  // Device-side numeric normalisation.  Off (the default): every Simpson
  // normalisation is the host's, bit-identical to the reference's.  On: the nodes of a launch's
  // plan whose normalisation has no closed form (Expression, ChiSquare, JohnsonSU, ArgusBG with
  // p != 1/2, sums over them) are integrated on the GPU for all P points at once -- the
  // reference's own adaptive rule, one warp per point (kernels_device.cuh simpson_kernel) --
  // and the host builds the constant rows from those values.  FFB_DEVICE_NORM=1 switches it
  // on for every engine.
  void set_device_normalization(bool on) { device_norm_ = on; }
  bool device_normalization() const { return device_norm_; }
  // The normalisation integral of `pdf` at P points by the device quadrature (children's
  // normalisations included, bottom-up); out[P].  On the current device (or the engine's).
  void device_normalization_of(int pdf, const double* thetas, int P, double* out);
  unsigned long long device_norm_launches() const { return norm_launches_; }

  const HostPlan& likelihood_plan() const { return plan_; }
  NllLaunchInfo last_launch() const { return last_; }
  cudaStream_t stream(int device);

 private:
  static constexpr int kGraphMaxPoints = 8;  // few-point synchronous calls replay a CUDA graph
  NllResult nll_points_graph(const DeviceDataset& ds, const double* thetas, int P);
  NllResult nll_points_stream(const DeviceDataset& ds, const double* thetas, int P);
  // the kernel build and plan rewrite a launch of these rows takes (may flag rows for the
  // partly shared ArgusBG cache, so it runs between building and copying them)
  struct LaunchChoice {
    DevPlan lp{};
    int cached = 0, ks = 0;
    bool jit = false, spec = false;
  };
  LaunchChoice choose_launch(double* h_rows, int P, long long n);
  int build_rows(const HostPlan& plan, const double* thetas, int P, double extra_scale);  // -> slot
  const double* copy_rows(const HostPlan& plan, int slot, int P, cudaStream_t s);
  void mark_consumed(int slot, cudaStream_t s);
  int launch_device(const DeviceDataset& ds, int P, const double* d_consts, const double* h_rows,
                    const LaunchChoice& c, SumPair* d_pairs, unsigned long long* d_bad, cudaStream_t s,
                    cudaEvent_t ea, cudaEvent_t eb);
  std::string launch_signature(const DeviceDataset& ds, int P, const LaunchChoice& c, const double* h_rows) const;
  void drop_graph();
  void ensure_gslots(std::size_t need);  // gradient slot buffers (device + pinned host)
  void bind_columns(const HostPlan& plan, const DeviceDataset& ds, ColPtrs& cols) const;
  void ensure(int device, int P, std::size_t scratch);
  const double* upload_constants(const HostPlan& plan, const double* thetas, int P, cudaStream_t s,
                                 double extra_scale = 1.0);

  // fills norm_cache_ (P x pdfs, NaN = not computed) for the Simpson-normalised nodes under
  // `pdf`; false when there are none (or the device path is off)
  bool device_norms(int pdf, const double* thetas, int P);
  struct NormJob {
    HostPlan plan;
    ExprInstr* d_prog = nullptr;
  };
  std::map<int, NormJob> norm_jobs_;
  std::vector<double> norm_cache_;
  bool device_norm_ = false;
  cudaStream_t norm_stream_ = nullptr;
  double* d_nrows_ = nullptr;
  double* d_nout_ = nullptr;
  int* d_nstatus_ = nullptr;
  std::size_t cap_nrows_ = 0;
  int cap_nout_ = 0;
  unsigned long long norm_launches_ = 0;

  const Model& m_;
  HostPlan plan_;
  int device_ = -1;
  cudaStream_t stream_ = nullptr;
  int cap_points_ = 0;
  std::size_t cap_scratch_ = 0;
  // double-buffered constant rows: host builds slot k while the GPU may still
  // be copying / reading slot k^1
  double* d_consts_[2] = {nullptr, nullptr};
  double* h_consts_[2] = {nullptr, nullptr};  // pinned
  cudaEvent_t staged_[2] = {nullptr, nullptr};
  cudaEvent_t consumed_[2] = {nullptr, nullptr};  // the last launch reading slot k's device rows
  int slot_ = 0;
  void* d_scratch_ = nullptr;
  SumPair* d_pairs_ = nullptr;
  unsigned long long* d_bad_ = nullptr;
  SumPair* h_pairs_ = nullptr;             // pinned
  unsigned long long* h_bad_ = nullptr;    // pinned
  NllLaunchInfo last_{};
  GradPlan grad_{};
  std::vector<bool> grad_const_;  // constness the layout was compiled for
  ExprInstr* d_prog_ = nullptr;  // device copy of plan_.programs
  int last_grad_jit_ = 0;
  SumPair* d_gslots_ = nullptr;
  SumPair* h_gslots_ = nullptr;  // pinned
  std::size_t cap_gslots_ = 0;
  cudaGraphExec_t graph_exec_ = nullptr;  // the captured few-point call (nll_points_graph)
  std::string graph_key_;
  int graph_launches_ = 0;
  NllLaunchInfo graph_last_{};
};

// Optional per-launch timing of the fused NLL kernel (CUDA events on the
// launching stream), for the live roofline in bench.py.
void kernel_timer_enable(bool on);
// Synchronises on the recorded events; returns summed ms and count, then clears.
double kernel_timer_read(unsigned long long* count);

// Process-wide count of kernels this library launched.
unsigned long long kernel_launches();
void count_launches(unsigned long long k);

}  // namespace ffb
