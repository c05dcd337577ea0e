#include "engine.hpp"

#include "jit.hpp"
#include "parallel.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <optional>
#include <sstream>
#include <utility>

namespace ffb {

namespace {

std::atomic<unsigned long long> g_launches{0};

}  // namespace

namespace {
std::mutex g_timer_mu;
bool g_timer_on = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timer_events;
}  // namespace

void kernel_timer_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  g_timer_on = on;
}

double kernel_timer_read(unsigned long long* count) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  double total = 0.0;
  for (auto& [a, b] : g_timer_events) {
    cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize(timer)");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
    total += ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  if (count) *count = g_timer_events.size();
  g_timer_events.clear();
  return total;
}

unsigned long long kernel_launches() { return g_launches.load(); }
void count_launches(unsigned long long k) { g_launches += k; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(ErrorCode::Numeric, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

DeviceGuard::DeviceGuard(int device) {
  cuda_check(cudaGetDevice(&prev_), "cudaGetDevice");
  if (prev_ != device) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    switched_ = true;
  }
}

DeviceGuard::~DeviceGuard() {
  if (switched_) cudaSetDevice(prev_);
}

// ---------------------------------------------------------------------------
// DeviceDataset

DeviceDataset::~DeviceDataset() {
  if (owns) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (double* c : cols) cudaFree(c);
    cudaSetDevice(prev);
  }
}

int DeviceDataset::column_index(const std::string& name) const {
  for (std::size_t i = 0; i < names.size(); ++i) {
    if (names[i] == name) return static_cast<int>(i);
  }
  return -1;
}

std::shared_ptr<DeviceDataset> DeviceDataset::upload(const std::vector<std::string>& names,
                                                     const std::vector<const double*>& host_cols,
                                                     long long n) {
  if (names.size() != host_cols.size()) usage_error("dataset: names/columns length mismatch");
  auto ds = allocate(names, n);
  ds->copy_from_host(host_cols);
  return ds;
}

std::shared_ptr<DeviceDataset> DeviceDataset::allocate(const std::vector<std::string>& names, long long n) {
  if (n < 0) usage_error("dataset: negative row count");
  for (std::size_t i = 0; i < names.size(); ++i) {
    for (std::size_t j = 0; j < i; ++j) {
      if (names[i] == names[j]) data_error("duplicate column name: " + names[i]);
    }
  }
  auto ds = std::make_shared<DeviceDataset>();
  cuda_check(cudaGetDevice(&ds->device), "cudaGetDevice");
  ds->n = n;
  ds->names = names;
  // Columns are padded to a whole number of 2048-event tiles (16-byte aligned
  // bulk copies of full tiles; cudaMalloc gives 256-byte alignment).
  const long long padded = ((n + 2047) / 2048) * 2048 + 2048;
  for (std::size_t i = 0; i < names.size(); ++i) {
    double* d = nullptr;
    cuda_check(cudaMalloc(&d, static_cast<std::size_t>(padded) * sizeof(double)), "cudaMalloc(column)");
    ds->cols.push_back(d);
  }
  return ds;
}

std::shared_ptr<DeviceDataset> DeviceDataset::view(const std::vector<std::string>& names,
                                                   const std::vector<const double*>& dev_cols,
                                                   long long n, int device) {
  if (names.size() != dev_cols.size()) usage_error("dataset: names/columns length mismatch");
  auto ds = std::make_shared<DeviceDataset>();
  ds->device = device;
  ds->n = n;
  ds->names = names;
  ds->owns = false;
  for (const double* c : dev_cols) {
    if (!c && n > 0) usage_error("dataset view: null device column");
    if (reinterpret_cast<uintptr_t>(c) % 8 != 0) usage_error("dataset view: columns must be 8-byte aligned");
    ds->cols.push_back(const_cast<double*>(c));
  }
  return ds;
}

void DeviceDataset::copy_from_host(const std::vector<const double*>& host_cols) {
  if (host_cols.size() != cols.size()) usage_error("dataset: column count mismatch");
  if (n == 0) return;
  DeviceGuard g(device);
  for (std::size_t i = 0; i < cols.size(); ++i) {
    if (!host_cols[i]) usage_error("dataset: null host column");
    cuda_check(cudaMemcpy(cols[i], host_cols[i], static_cast<std::size_t>(n) * sizeof(double),
                          cudaMemcpyHostToDevice),
               "cudaMemcpy(H2D column)");
  }
}

void DeviceDataset::copy_from_host_async(const std::vector<const double*>& host_cols, cudaStream_t stream) {
  if (host_cols.size() != cols.size()) usage_error("dataset: column count mismatch");
  if (n == 0) return;
  DeviceGuard g(device);
  for (std::size_t i = 0; i < cols.size(); ++i) {
    if (!host_cols[i]) usage_error("dataset: null host column");
    cuda_check(cudaMemcpyAsync(cols[i], host_cols[i], static_cast<std::size_t>(n) * sizeof(double),
                               cudaMemcpyHostToDevice, stream),
               "cudaMemcpyAsync(H2D column)");
  }
}

void DeviceDataset::download(int col, double* host_out) const {
  if (col < 0 || col >= static_cast<int>(cols.size())) usage_error("dataset: column index out of range");
  if (n == 0) return;
  DeviceGuard g(device);
  cuda_check(cudaMemcpy(host_out, cols[col], static_cast<std::size_t>(n) * sizeof(double),
                        cudaMemcpyDeviceToHost),
             "cudaMemcpy(D2H column)");
}

// ---------------------------------------------------------------------------
// Engine

Engine::Engine(const Model& m) : m_(m), plan_(compile_plan(m, m.root, true)) {
  const char* e = std::getenv("FFB_DEVICE_NORM");
  device_norm_ = e != nullptr && e[0] == '1';
}

Engine::~Engine() {
  if (device_ >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    drop_graph();
    for (int k = 0; k < 2; ++k) {
      cudaFree(d_consts_[k]);
      cudaFreeHost(h_consts_[k]);
      if (staged_[k]) cudaEventDestroy(staged_[k]);
      if (consumed_[k]) cudaEventDestroy(consumed_[k]);
    }
    cudaFree(d_scratch_);
    cudaFree(d_pairs_);
    cudaFree(d_bad_);
    cudaFreeHost(h_pairs_);
    cudaFreeHost(h_bad_);
    cudaFree(d_gslots_);
    cudaFreeHost(h_gslots_);
    cudaFree(d_prog_);
    cudaFree(d_nrows_);
    cudaFree(d_nout_);
    cudaFree(d_nstatus_);
    for (auto& j : norm_jobs_) cudaFree(j.second.d_prog);
    if (norm_stream_) cudaStreamDestroy(norm_stream_);
    if (stream_) cudaStreamDestroy(stream_);
    cudaSetDevice(prev);
  }
}

cudaStream_t Engine::stream(int device) {
  ensure(device, 1, 0);
  return stream_;
}

void Engine::ensure(int device, int P, std::size_t scratch) {
  if (device_ != device) {
    if (device_ >= 0) usage_error("a model's GPU engine is bound to one device; use one model per device");
    device_ = device;
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaEventCreateWithFlags(&staged_[k], cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaEventCreateWithFlags(&consumed_[k], cudaEventDisableTiming), "cudaEventCreate");
    }
    if (!plan_.programs.empty()) {  // Expression programs: once per engine and device
      const std::size_t bytes = plan_.programs.size() * sizeof(ExprInstr);
      cuda_check(cudaMalloc(&d_prog_, bytes), "cudaMalloc(programs)");
      cuda_check(cudaMemcpy(d_prog_, plan_.programs.data(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy(programs)");
      plan_.dev.prog = d_prog_;
    }
  }
  if (P > cap_points_) {
    drop_graph();  // the captured call reads the buffers replaced here
    const int cap = std::max(P, 16);
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaEventSynchronize(staged_[k]), "cudaEventSynchronize");
      cudaFree(d_consts_[k]);
      cudaFreeHost(h_consts_[k]);
    }
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    cudaFree(d_pairs_);
    cudaFree(d_bad_);
    cudaFreeHost(h_pairs_);
    cudaFreeHost(h_bad_);
    const std::size_t cbytes = static_cast<std::size_t>(cap) * std::max(1, plan_.dev.stride) * sizeof(double);
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaMalloc(&d_consts_[k], cbytes), "cudaMalloc(consts)");
      cuda_check(cudaHostAlloc(&h_consts_[k], cbytes, cudaHostAllocDefault), "cudaHostAlloc(consts)");
    }
    cuda_check(cudaMalloc(&d_pairs_, cap * sizeof(SumPair)), "cudaMalloc(pairs)");
    cuda_check(cudaMalloc(&d_bad_, cap * sizeof(unsigned long long)), "cudaMalloc(bad)");
    cuda_check(cudaHostAlloc(&h_pairs_, cap * sizeof(SumPair), cudaHostAllocDefault), "cudaHostAlloc");
    cuda_check(cudaHostAlloc(&h_bad_, cap * sizeof(unsigned long long), cudaHostAllocDefault), "cudaHostAlloc");
    cap_points_ = cap;
  }
  if (scratch > cap_scratch_) {
    drop_graph();
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    cudaFree(d_scratch_);
    cuda_check(cudaMalloc(&d_scratch_, scratch), "cudaMalloc(scratch)");
    cap_scratch_ = scratch;
  }
}

void Engine::bind_columns(const HostPlan& plan, const DeviceDataset& ds, ColPtrs& cols) const {
  std::memset(&cols, 0, sizeof(cols));
  for (std::size_t s = 0; s < plan.col_obs.size(); ++s) {
    const std::string& name = m_.observables[plan.col_obs[s]].name;
    const int ci = ds.column_index(name);
    if (ci < 0) data_error("unknown column: " + name);
    cols.c[s] = ds.cols[ci];
  }
}

const double* Engine::upload_constants(const HostPlan& plan, const double* thetas, int P,
                                       cudaStream_t s, double extra_scale) {
  const int k = build_rows(plan, thetas, P, extra_scale);
  return copy_rows(plan, k, P, s);
}

// Every launch that reads slot k's device rows records consumed_[k] on its stream right
// after it is queued; copy_rows makes the next copy into that slot wait for it.
void Engine::mark_consumed(int k, cudaStream_t s) {
  cuda_check(cudaEventRecord(consumed_[k], s), "cudaEventRecord");
}

const double* Engine::copy_rows(const HostPlan& plan, int k, int P, cudaStream_t s) {
  // the launch that last read this slot's device rows may run on another stream
  cuda_check(cudaStreamWaitEvent(s, consumed_[k], 0), "cudaStreamWaitEvent");
  cuda_check(cudaMemcpyAsync(d_consts_[k], h_consts_[k],
                             static_cast<std::size_t>(P) * plan.dev.stride * sizeof(double),
                             cudaMemcpyHostToDevice, s),
             "cudaMemcpyAsync(consts)");
  cuda_check(cudaEventRecord(staged_[k], s), "cudaEventRecord");
  return d_consts_[k];
}

bool Engine::device_norms(int pdf, const double* thetas, int P) {
  if (!device_norm_ || device_ < 0 || P <= 0) return false;
  const int npar = static_cast<int>(m_.params.size());
  const int npdf = static_cast<int>(m_.pdfs.size());
  // which nodes take the Simpson route is decided at the first point (it depends on the
  // parameters only through ArgusBG's p == 1/2); a node that needs a quadrature at a later
  // point only falls back to the host's
  const std::vector<int> nodes = m_.simpson_nodes(pdf, thetas);
  if (nodes.empty()) return false;
  norm_cache_.assign(static_cast<std::size_t>(P) * npdf, std::numeric_limits<double>::quiet_NaN());
  if (!norm_stream_) cuda_check(cudaStreamCreateWithFlags(&norm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  if (P > cap_nout_) {
    cudaFree(d_nout_);
    cudaFree(d_nstatus_);
    cap_nout_ = std::max(P, 64);
    cuda_check(cudaMalloc(&d_nout_, cap_nout_ * sizeof(double)), "cudaMalloc(norms)");
    cuda_check(cudaMalloc(&d_nstatus_, cap_nout_ * sizeof(int)), "cudaMalloc(norm status)");
  }
  std::vector<double> rows, vals(P);
  std::vector<int> status(P);
  for (const int id : nodes) {  // children before parents
    auto it = norm_jobs_.find(id);
    if (it == norm_jobs_.end()) {
      NormJob job;
      try {
        job.plan = compile_plan(m_, id, false);
      } catch (const Error&) {
        // a subtree outside the plan's canonical form: its quadrature stays on the host (the
        // cache keeps NaN for it, so normalization() integrates it as before)
        job.plan.pdf = -1;
      }
      if (!job.plan.programs.empty()) {
        const std::size_t bytes = job.plan.programs.size() * sizeof(ExprInstr);
        cuda_check(cudaMalloc(&job.d_prog, bytes), "cudaMalloc(programs)");
        cuda_check(cudaMemcpy(job.d_prog, job.plan.programs.data(), bytes, cudaMemcpyHostToDevice),
                   "cudaMemcpy(programs)");
        job.plan.dev.prog = job.d_prog;
      }
      it = norm_jobs_.emplace(id, std::move(job)).first;
    }
    const HostPlan& plan = it->second.plan;
    if (plan.pdf < 0) continue;
    const int stride = std::max(1, plan.dev.stride);
    rows.assign(static_cast<std::size_t>(P) * stride, 0.0);
    // the sub-pdf's unnormalised rows: its children's normalisations are already in the cache
    for (int p = 0; p < P; ++p) {
      NormOverride ov(&norm_cache_[static_cast<std::size_t>(p) * npdf]);
      build_constants(plan, m_, thetas + static_cast<std::size_t>(p) * npar, &rows[static_cast<std::size_t>(p) * stride],
                      1.0);
    }
    if (rows.size() > cap_nrows_) {
      cudaFree(d_nrows_);
      cap_nrows_ = rows.size();
      cuda_check(cudaMalloc(&d_nrows_, cap_nrows_ * sizeof(double)), "cudaMalloc(norm rows)");
    }
    cuda_check(cudaMemcpyAsync(d_nrows_, rows.data(), rows.size() * sizeof(double), cudaMemcpyHostToDevice, norm_stream_),
               "cudaMemcpyAsync(norm rows)");
    const Observable& o = m_.obs_of(id);
    const int launches = launch_simpson(plan.dev, d_nrows_, P, o.lo, o.hi, 1e-10 * (o.hi - o.lo), 1e-10, 60, d_nout_,
                                        d_nstatus_, norm_stream_);
    cuda_check(cudaGetLastError(), "launch_simpson");
    cuda_check(cudaMemcpyAsync(vals.data(), d_nout_, P * sizeof(double), cudaMemcpyDeviceToHost, norm_stream_),
               "cudaMemcpyAsync(norms)");
    cuda_check(cudaMemcpyAsync(status.data(), d_nstatus_, P * sizeof(int), cudaMemcpyDeviceToHost, norm_stream_),
               "cudaMemcpyAsync(norm status)");
    cuda_check(cudaStreamSynchronize(norm_stream_), "device normalisation");
    count_launches(launches);
    norm_launches_ += launches;
    for (int p = 0; p < P; ++p) {
      if (status[p]) numeric_error("non-finite integrand in the normalisation of '" + m_.pdfs[id].name + "'");
      norm_cache_[static_cast<std::size_t>(p) * npdf + id] = vals[p];
    }
  }
  return true;
}

void Engine::device_normalization_of(int pdf, const double* thetas, int P, double* out) {
  if (P <= 0) return;
  int dev = device_;
  if (dev < 0) cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  DeviceGuard g(dev);
  ensure(dev, 1, 0);
  const int npar = static_cast<int>(m_.params.size());
  const int npdf = static_cast<int>(m_.pdfs.size());
  for (int p = 0; p < P; ++p) m_.check_params(pdf, thetas + static_cast<std::size_t>(p) * npar);
  const bool was = device_norm_;
  device_norm_ = true;
  bool have = false;
  try {
    have = device_norms(pdf, thetas, P);
  } catch (...) {
    device_norm_ = was;
    throw;
  }
  device_norm_ = was;
  for (int p = 0; p < P; ++p) {
    if (have) {
      NormOverride ov(&norm_cache_[static_cast<std::size_t>(p) * npdf]);
      out[p] = m_.normalization(pdf, thetas + static_cast<std::size_t>(p) * npar);
    } else {
      out[p] = m_.normalization(pdf, thetas + static_cast<std::size_t>(p) * npar);
    }
  }
}

int Engine::build_rows(const HostPlan& plan, const double* thetas, int P, double extra_scale) {
  const int k = slot_ ^= 1;
  // slot k fed the copy two calls ago; that copy must be done before reuse
  cuda_check(cudaEventSynchronize(staged_[k]), "cudaEventSynchronize");
  const int npar = static_cast<int>(m_.params.size());
  const int stride = plan.dev.stride;
  // the points' constant rows are independent: spread them over the host pool when the
  // rows are expensive (Simpson normalisations: Expression / ChiSquare / JohnsonSU), else
  // build them here -- analytic rows take ~0.2-1 us, less than waking the pool (each row
  // is validated; the first invalid point's error is raised)
  // (device-side numeric normalisation, when on: the Simpson-normalised nodes of all P points
  // first, in a few launches; the rows then read those values)
  const bool dn = device_norms(plan.pdf, thetas, P);
  const int npdf = static_cast<int>(m_.pdfs.size());
  auto row = [&](int p) {
    std::optional<NormOverride> ov;
    if (dn) ov.emplace(&norm_cache_[static_cast<std::size_t>(p) * npdf]);
    build_constants(plan, m_, thetas + static_cast<std::size_t>(p) * npar,
                    h_consts_[k] + static_cast<std::size_t>(p) * stride, extra_scale);
  };
  const auto t0 = std::chrono::steady_clock::now();
  row(0);
  const double first_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  if (P > 1 && first_us * (P - 1) > 100.0) {
    ThreadPool::instance().parallel_for(P - 1, [&](int p) { row(p + 1); });
  } else {
    for (int p = 1; p < P; ++p) row(p);
  }
  return k;
}

int Engine::nll_points_device(const DeviceDataset& ds, const double* thetas, int P,
                              SumPair* d_pairs, unsigned long long* d_bad, cudaStream_t stream,
                              cudaStream_t upload_stream) {
  if (P <= 0) return 0;
  if (P > kMaxPointsPerLaunch) usage_error("nll_points_device: at most 512 points per call");
  DeviceGuard g(ds.device);
  const std::size_t scratch = ds.n > 0 ? nll_scratch_bytes(ds.n, P, plan_.dev.ncols) : 0;
  ensure(ds.device, P, scratch);
  cudaStream_t s = stream ? stream : stream_;
  if (s != stream_) {
    // order this call after the engine's previous work and vice versa
    cudaEvent_t ev;
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    cudaEventRecord(ev, stream_);
    cudaStreamWaitEvent(s, ev, 0);
    cudaEventDestroy(ev);
  }
  // the likelihood kernel evaluates p * 2^kPScaleLog2 (plan.hpp); the launch decisions
  // (launch-constant caches may flag rows) come between building the rows and their copy
  const int slot = build_rows(plan_, thetas, P, std::ldexp(1.0, kPScaleLog2));
  const LaunchChoice choice = choose_launch(h_consts_[slot], P, ds.n);
  const double* d_consts = nullptr;
  if (upload_stream && upload_stream != s) {
    // the rows' copy on the caller's upload stream (beside its input copies: no copy-engine
    // queueing behind this stream's running kernels), the launch after it
    d_consts = copy_rows(plan_, slot, P, upload_stream);
    cuda_check(cudaStreamWaitEvent(s, staged_[slot], 0), "cudaStreamWaitEvent");
  } else {
    d_consts = copy_rows(plan_, slot, P, s);
  }
  cudaEvent_t ea = nullptr, eb = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_timer_mu);
    if (g_timer_on && ds.n > 0) {
      cuda_check(cudaEventCreate(&ea), "cudaEventCreate");
      cuda_check(cudaEventCreate(&eb), "cudaEventCreate");
      g_timer_events.emplace_back(ea, eb);
    }
  }
  const int launches = launch_device(ds, P, d_consts, h_consts_[slot], choice, d_pairs, d_bad, s, ea, eb);
  mark_consumed(slot, s);
  if (s != stream_) {
    cudaEvent_t ev;
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(stream_, ev, 0);
    cudaEventDestroy(ev);
  }
  count_launches(launches);
  return launches;
}

Engine::LaunchChoice Engine::choose_launch(double* h_rows, int P, long long n) {
  LaunchChoice c;
  c.lp = plan_.dev;
  if (!plan_.programs.empty() && jit_prepare(plan_)) {
    c.jit = true;  // Expression leaves: the formula-specialised build (jit.cpp)
    return c;
  }
  // launch-constant branches (leaves / ArgusBG data parts fixed over the launch) cached per
  // tile; a partly shared ArgusBG m0 flags the rows that use the cache
  c.cached = cache_launch_constants(c.lp, h_rows, P);
  c.ks = plan_kind_set(c.lp, h_rows, P);
  c.spec = plan_spec_applies(plan_, c.lp, n, P) && plan_spec_prepare(c.lp, c.ks);
  return c;
}

int Engine::launch_device(const DeviceDataset& ds, int P, const double* d_consts, const double* h_rows,
                          const LaunchChoice& c, SumPair* d_pairs, unsigned long long* d_bad, cudaStream_t s,
                          cudaEvent_t ea, cudaEvent_t eb) {
  if (ds.n == 0) {
    cuda_check(cudaMemsetAsync(d_pairs, 0, P * sizeof(SumPair), s), "cudaMemsetAsync");
    cuda_check(cudaMemsetAsync(d_bad, 0xff, P * sizeof(unsigned long long), s), "cudaMemsetAsync");
    return 0;
  }
  ColPtrs cols;
  bind_columns(plan_, ds, cols);
  if (c.jit) {
    last_ = launch_nll_jit(plan_, cols, ds.n, d_consts, P, d_scratch_, d_pairs, d_bad, s, h_rows, ea, eb);
  } else {
    if (c.spec) {
      // the tile kernel compiled around this launch's term list (jit.cpp; cached)
      last_ = launch_nll_spec(c.lp, cols, ds.n, d_consts, P, d_scratch_, d_pairs, d_bad, s, c.ks, nll_waves(), ea,
                              eb);
    } else {
      last_ = launch_nll(c.lp, cols, ds.n, d_consts, P, d_scratch_, d_pairs, d_bad, s, c.ks, ea, eb);
    }
    last_.cached = c.cached;
  }
  cuda_check(cudaGetLastError(), "launch_nll");
  return last_.launches;
}

// What launch_device would run for these rows: the key under which a captured graph of
// the launch stays valid (the dataset's columns and size, P, and every launch decision).
std::string Engine::launch_signature(const DeviceDataset& ds, int P, const LaunchChoice& c,
                                     const double* h_rows) const {
  std::ostringstream o;
  o << ds.n << ':' << P;
  for (const double* col : ds.cols) o << ':' << static_cast<const void*>(col);
  if (c.jit) {
    const ExprHoist h = analyse_expr_hoist(plan_, h_rows, P);
    o << "|jit";
    for (const HoistSlot& v : h.slots) o << ',' << v.col << '/' << v.begin << '/' << v.end;
  } else {
    o << "|c" << c.cached << "|k" << c.ks << "|s" << c.spec;
    for (int i = 0; i < c.lp.nterms; ++i) o << ',' << c.lp.t[i].kind << '/' << c.lp.t[i].order;
    for (int d = 0; d < c.lp.nderived; ++d) o << ",d" << c.lp.dv[d].row << '/' << c.lp.dv[d].dst;
  }
  return o.str();
}

void Engine::ensure_gslots(std::size_t need) {
  if (need <= cap_gslots_) return;
  cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
  cudaFree(d_gslots_);
  cudaFreeHost(h_gslots_);
  cuda_check(cudaMalloc(&d_gslots_, need * sizeof(SumPair)), "cudaMalloc(gslots)");
  cuda_check(cudaHostAlloc(&h_gslots_, need * sizeof(SumPair), cudaHostAllocDefault), "cudaHostAlloc");
  cap_gslots_ = need;
}

void Engine::reserve(const DeviceDataset& ds, int P_nll, int P_grad) {
  DeviceGuard g(ds.device);
  std::size_t scratch = 0;
  if (ds.n > 0 && P_nll > 0) scratch = nll_scratch_bytes(ds.n, P_nll, plan_.dev.ncols);
  if (ds.n > 0 && P_grad > 0) {
    const GradPlan& gp = grad_plan();
    if (gp.ok) scratch = std::max(scratch, nll_grad_scratch_bytes(ds.n, P_grad, plan_.dev, gp.dev));
  }
  ensure(ds.device, std::max(P_nll, P_grad), scratch);
  if (P_grad > 0 && grad_plan().ok) ensure_gslots(static_cast<std::size_t>(P_grad) * grad_plan().dev.nslots);
}

void Engine::drop_graph() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  graph_exec_ = nullptr;
  graph_key_.clear();
}

NllResult Engine::nll_points(const DeviceDataset& ds, const double* thetas, int P) {
  static const bool no_graphs = std::getenv("FFB_NO_GRAPHS") != nullptr;
  bool timing;
  {
    std::lock_guard<std::mutex> lk(g_timer_mu);
    timing = g_timer_on;
  }
  if (!no_graphs && !timing && P <= kGraphMaxPoints && ds.n > 0) return nll_points_graph(ds, thetas, P);
  return nll_points_stream(ds, thetas, P);
}

// Few-point synchronous calls (a minimiser's function evaluations): the constant-row
// upload, the launch sequence and the result read-back are one CUDA graph, captured on the
// second call with the same launch signature and replayed while it holds -- one graph
// launch instead of six API calls per evaluation.  The graph's H2D node reads the pinned
// row buffer at execution, so each call only rewrites the rows.
NllResult Engine::nll_points_graph(const DeviceDataset& ds, const double* thetas, int P) {
  NllResult r;
  r.value.resize(P);
  r.pairs.resize(P);
  r.first_invalid.resize(P);
  const int npar = static_cast<int>(m_.params.size());
  DeviceGuard g(ds.device);
  ensure(ds.device, P, nll_scratch_bytes(ds.n, P, plan_.dev.ncols));
  // rows into slot 0 (any earlier asynchronous copy out of it has completed)
  cuda_check(cudaEventSynchronize(staged_[0]), "cudaEventSynchronize");
  const int stride = plan_.dev.stride;
  const bool dn = device_norms(plan_.pdf, thetas, P);  // (the quadrature stays outside the graph)
  const int npdf = static_cast<int>(m_.pdfs.size());
  for (int p = 0; p < P; ++p) {
    std::optional<NormOverride> ov;
    if (dn) ov.emplace(&norm_cache_[static_cast<std::size_t>(p) * npdf]);
    build_constants(plan_, m_, thetas + static_cast<std::size_t>(p) * npar,
                    h_consts_[0] + static_cast<std::size_t>(p) * stride, std::ldexp(1.0, kPScaleLog2));
  }
  const LaunchChoice choice = choose_launch(h_consts_[0], P, ds.n);
  const std::string key = launch_signature(ds, P, choice, h_consts_[0]);
  const std::size_t bytes = static_cast<std::size_t>(P) * stride * sizeof(double);
  auto sequence = [&] {
    cuda_check(cudaMemcpyAsync(d_consts_[0], h_consts_[0], bytes, cudaMemcpyHostToDevice, stream_),
               "cudaMemcpyAsync(consts)");
    launch_device(ds, P, d_consts_[0], h_consts_[0], choice, d_pairs_, d_bad_, stream_, nullptr, nullptr);
    cuda_check(cudaMemcpyAsync(h_pairs_, d_pairs_, P * sizeof(SumPair), cudaMemcpyDeviceToHost, stream_),
               "cudaMemcpyAsync(pairs)");
    cuda_check(cudaMemcpyAsync(h_bad_, d_bad_, P * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_),
               "cudaMemcpyAsync(bad)");
  };
  int launches = 0;
  if (graph_exec_ && key == graph_key_) {
    cuda_check(cudaGraphLaunch(graph_exec_, stream_), "cudaGraphLaunch");
    launches = graph_launches_;
    last_ = graph_last_;
  } else if (key == graph_key_) {  // second call with this signature: capture, then replay
    cudaGraph_t graph = nullptr;
    cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
      sequence();
    } catch (...) {
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    cuda_check(cudaStreamEndCapture(stream_, &graph), "cudaStreamEndCapture");
    const cudaError_t e = cudaGraphInstantiate(&graph_exec_, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(e, "cudaGraphInstantiate");
    graph_launches_ = last_.launches;
    graph_last_ = last_;
    cuda_check(cudaGraphLaunch(graph_exec_, stream_), "cudaGraphLaunch");
    launches = graph_launches_;
  } else {  // a new signature: the plain sequence (it also compiles / loads any build)
    drop_graph();
    sequence();
    graph_key_ = key;
    launches = last_.launches;
  }
  cuda_check(cudaStreamSynchronize(stream_), "nll kernels");
  count_launches(launches);
  r.launches = launches;
  for (int i = 0; i < P; ++i) {
    r.pairs[i] = h_pairs_[i];
    const bool bad = h_bad_[i] != kNoInvalid;
    r.first_invalid[i] = bad ? static_cast<long long>(h_bad_[i]) : -1;
    r.value[i] = bad ? std::numeric_limits<double>::infinity()
                     : (h_pairs_[i].s + h_pairs_[i].c) +
                           m_.extended_term(thetas + static_cast<std::size_t>(i) * npar, static_cast<double>(ds.n));
  }
  return r;
}

NllResult Engine::nll_points_stream(const DeviceDataset& ds, const double* thetas, int P) {
  NllResult r;
  r.value.resize(P);
  r.pairs.resize(P);
  r.first_invalid.resize(P);
  const int npar = static_cast<int>(m_.params.size());
  DeviceGuard g(ds.device);
  for (int p0 = 0; p0 < P; p0 += kMaxPointsPerLaunch) {
    const int np = std::min(kMaxPointsPerLaunch, P - p0);
    const double* th = thetas + static_cast<std::size_t>(p0) * npar;
    ensure(ds.device, np, 0);
    r.launches += nll_points_device(ds, th, np, d_pairs_, d_bad_, stream_);
    cuda_check(cudaMemcpyAsync(h_pairs_, d_pairs_, np * sizeof(SumPair), cudaMemcpyDeviceToHost, stream_),
               "cudaMemcpyAsync(pairs)");
    cuda_check(cudaMemcpyAsync(h_bad_, d_bad_, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               stream_),
               "cudaMemcpyAsync(bad)");
    cuda_check(cudaStreamSynchronize(stream_), "nll kernels");
    for (int i = 0; i < np; ++i) {
      const int p = p0 + i;
      r.pairs[p] = h_pairs_[i];
      const bool bad = h_bad_[i] != kNoInvalid;
      r.first_invalid[p] = bad ? static_cast<long long>(h_bad_[i]) : -1;
      r.value[p] = bad ? std::numeric_limits<double>::infinity()
                       : (h_pairs_[i].s + h_pairs_[i].c) +
                             m_.extended_term(th + static_cast<std::size_t>(i) * npar,
                                              static_cast<double>(ds.n));
    }
  }
  return r;
}

const GradPlan& Engine::grad_plan() {
  std::vector<bool> cst(m_.params.size());
  for (std::size_t i = 0; i < cst.size(); ++i) cst[i] = m_.params[i].constant;
  if (grad_const_.empty() || cst != grad_const_) {
    grad_ = compile_grad_plan(plan_, m_);
    if (grad_.ok && !grad_layout_fits(plan_.dev, grad_.dev)) {
      grad_.ok = false;
      grad_.why = "gradient accumulators do not fit one CTA's shared memory";
    }
    grad_const_ = cst;
  }
  return grad_;
}

void Engine::grad_finish(const double* thetas, int P, const double* slot_sums, double n_events,
                         double* values, double* grads) {
  const GradPlan& gp = grad_plan();
  if (!gp.ok) usage_error("analytic gradient unavailable for this model: " + gp.why);
  const int npar = static_cast<int>(m_.params.size());
  const int S = gp.dev.nslots;
  const int nt = plan_.dev.nterms;
  std::vector<double> dc;
  for (int p = 0; p < P; ++p) {
    const double* th = thetas + static_cast<std::size_t>(p) * npar;
    const double* q = slot_sums + static_cast<std::size_t>(p) * S;
    double* g = grads + static_cast<std::size_t>(p) * npar;
    values[p] = q[0] + m_.extended_term(th, n_events);
    for (int j = 0; j < npar; ++j) g[j] = 0.0;
    m_.check_params(plan_.pdf, th);
    for (int j = 0; j < npar; ++j) {
      if (m_.params[j].constant) continue;
      dc = coef_derivatives(plan_, m_, th, j, std::ldexp(1.0, kPScaleLog2));
      double a = 0.0;
      for (int i = 0; i < nt; ++i) a += q[gp.a_slot[i]] * dc[i];
      g[j] = -a;
    }
    for (int k = 1; k < S; ++k) {
      const int j = gp.slot_param[k];
      if (j >= 0) g[j] -= q[k];
    }
    if (m_.extended()) {  // d(nu - N log nu)/d y_k = 1 - N / nu
      double nu = 0.0;
      for (const int k : m_.pdfs[m_.root].params) nu += th[k];
      for (const int k : m_.pdfs[m_.root].params) {
        if (!m_.params[k].constant) g[k] += 1.0 - n_events / nu;
      }
    }
  }
}

NllGradResult Engine::nll_grad_points(const DeviceDataset& ds, const double* thetas, int P) {
  const GradPlan& gp = grad_plan();
  if (!gp.ok) usage_error("analytic gradient unavailable for this model: " + gp.why);
  NllGradResult r;
  const int npar = static_cast<int>(m_.params.size());
  const int S = gp.dev.nslots;
  r.nslots = S;
  r.value.resize(P);
  r.grad.resize(static_cast<std::size_t>(P) * npar);
  r.first_invalid.resize(P);
  r.slots.resize(static_cast<std::size_t>(P) * S);
  DeviceGuard guard(ds.device);
  std::vector<double> sums;
  for (int p0 = 0; p0 < P; p0 += kMaxPointsPerLaunch) {
    const int np = std::min(kMaxPointsPerLaunch, P - p0);
    const double* th = thetas + static_cast<std::size_t>(p0) * npar;
    const std::size_t scratch = ds.n > 0 ? nll_grad_scratch_bytes(ds.n, np, plan_.dev, gp.dev) : 0;
    ensure(ds.device, np, scratch);
    const std::size_t need = static_cast<std::size_t>(np) * S;
    ensure_gslots(need);
    const double* d_consts = upload_constants(plan_, th, np, stream_, std::ldexp(1.0, kPScaleLog2));
    if (ds.n == 0) {
      cuda_check(cudaMemsetAsync(d_gslots_, 0, need * sizeof(SumPair), stream_), "cudaMemsetAsync");
      cuda_check(cudaMemsetAsync(d_bad_, 0xff, np * sizeof(unsigned long long), stream_), "cudaMemsetAsync");
    } else {
      ColPtrs cols;
      bind_columns(plan_, ds, cols);
      const int ks = plan_kind_set(plan_.dev, h_consts_[slot_], np);
      cudaEvent_t ea = nullptr, eb = nullptr;
      {
        std::lock_guard<std::mutex> lk(g_timer_mu);
        if (g_timer_on) {
          cuda_check(cudaEventCreate(&ea), "cudaEventCreate");
          cuda_check(cudaEventCreate(&eb), "cudaEventCreate");
          g_timer_events.emplace_back(ea, eb);
        }
      }
      const bool spec = grad_spec_applies(plan_, gp, cols, np) && grad_spec_prepare(plan_, gp, ks);
      const NllLaunchInfo li =
          spec ? launch_nll_grad_spec(plan_, gp, cols, ds.n, d_consts, d_scratch_, d_gslots_, d_bad_, stream_, ks, ea,
                                      eb)
               : launch_nll_grad(plan_.dev, gp.dev, cols, ds.n, d_consts, np, d_scratch_, d_gslots_, d_bad_, stream_,
                                 ks, ea, eb);
      last_grad_jit_ = li.jit;
      cuda_check(cudaGetLastError(), "launch_nll_grad");
      mark_consumed(slot_, stream_);
      r.launches += li.launches;
      count_launches(li.launches);
    }
    cuda_check(cudaMemcpyAsync(h_gslots_, d_gslots_, need * sizeof(SumPair), cudaMemcpyDeviceToHost, stream_),
               "cudaMemcpyAsync(gslots)");
    cuda_check(cudaMemcpyAsync(h_bad_, d_bad_, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_),
               "cudaMemcpyAsync(bad)");
    cuda_check(cudaStreamSynchronize(stream_), "nll_grad kernels");
    sums.resize(need);
    for (std::size_t k = 0; k < need; ++k) {
      r.slots[static_cast<std::size_t>(p0) * S + k] = h_gslots_[k];
      sums[k] = h_gslots_[k].s + h_gslots_[k].c;
    }
    grad_finish(th, np, sums.data(), static_cast<double>(ds.n), r.value.data() + p0,
                r.grad.data() + static_cast<std::size_t>(p0) * npar);
    for (int i = 0; i < np; ++i) {
      const int p = p0 + i;
      const bool bad = h_bad_[i] != kNoInvalid;
      r.first_invalid[p] = bad ? static_cast<long long>(h_bad_[i]) : -1;
      if (bad) {
        r.value[p] = std::numeric_limits<double>::infinity();
        for (int j = 0; j < npar; ++j) {
          r.grad[static_cast<std::size_t>(p) * npar + j] = std::numeric_limits<double>::quiet_NaN();
        }
      }
    }
  }
  return r;
}

void Engine::probabilities(const DeviceDataset& ds, const double* theta, double* out,
                           bool out_on_device, cudaStream_t stream) {
  eval_batch(-1, ds, theta, out, out_on_device, stream);
}

void Engine::eval_batch(int pdf, const DeviceDataset& ds, const double* theta, double* out,
                        bool out_on_device, cudaStream_t stream) {
  HostPlan plan = pdf < 0 ? plan_ : compile_plan(m_, pdf, false);
  m_.check_params(plan.pdf, theta);
  if (ds.n == 0) return;
  DeviceGuard g(ds.device);
  ensure(ds.device, 1, 0);
  if (pdf < 0) plan.dev.prog = plan_.dev.prog;
  ExprInstr* d_sub_prog = nullptr;  // a sub-pdf's own Expression programs (freed below)
  if (pdf >= 0 && !plan.programs.empty()) {
    const std::size_t bytes = plan.programs.size() * sizeof(ExprInstr);
    cuda_check(cudaMalloc(&d_sub_prog, bytes), "cudaMalloc(programs)");
    cuda_check(cudaMemcpy(d_sub_prog, plan.programs.data(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy(programs)");
    plan.dev.prog = d_sub_prog;
  }
  cudaStream_t s = stream ? stream : stream_;
  ColPtrs cols;
  bind_columns(plan, ds, cols);
  if (s != stream_) cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
  const double* d_consts = upload_constants(plan, theta, 1, s);
  double* d_out = out;
  if (!out_on_device) {
    cuda_check(cudaMalloc(&d_out, static_cast<std::size_t>(ds.n) * sizeof(double)), "cudaMalloc(out)");
  }
  const int slot = slot_;  // upload_constants filled this slot
  count_launches(launch_eval(plan.dev, cols, ds.n, d_consts, d_out, s, h_consts_[slot]));
  cuda_check(cudaGetLastError(), "launch_eval");
  mark_consumed(slot, s);  // a later copy into this slot (any stream) waits for the kernel
  if (!out_on_device) {
    cuda_check(cudaMemcpyAsync(out, d_out, static_cast<std::size_t>(ds.n) * sizeof(double),
                               cudaMemcpyDeviceToHost, s),
               "cudaMemcpyAsync(out)");
    cuda_check(cudaStreamSynchronize(s), "eval kernel");
    cudaFree(d_out);
  } else if (s != stream_) {
    cudaEvent_t ev;
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(stream_, ev, 0);
    cudaEventDestroy(ev);
  }
  if (d_sub_prog) {
    cuda_check(cudaStreamSynchronize(s), "eval kernel");
    cudaFree(d_sub_prog);
  }
}

}  // namespace ffb
