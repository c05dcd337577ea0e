#include "shard.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "common.hpp"

namespace ffb {

namespace {

void cuda_free_all(std::initializer_list<void*> ps) {
  for (void* p : ps)
    if (p) cudaFree(p);
}

}  // namespace

std::unique_ptr<ShardGroup> ShardGroup::create_rank(const Model& m, std::shared_ptr<DeviceDataset> shard,
                                                    long long n_total, long long offset, const ncclUniqueId& id,
                                                    int world, int rank) {
  if (!shard) usage_error("shard group: null dataset");
  if (world < 1 || rank < 0 || rank >= world) usage_error("shard group: bad rank / world");
  if (offset < 0 || offset + shard->n > n_total) usage_error("shard group: shard outside [0, n_total)");
  const NcclApi& api = nccl();
  std::unique_ptr<ShardGroup> g(new ShardGroup(m, n_total, world));
  Local L;
  L.device = shard->device;
  L.rank = rank;
  L.offset = offset;
  L.ds = std::move(shard);
  L.engine = std::make_unique<Engine>(m);
  DeviceGuard dg(L.device);
  cuda_check(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking), "cudaStreamCreate");
  g->local_.push_back(std::move(L));
  Local& l = g->local_.back();
  nccl_check(api.comm_init_rank(&l.comm, world, id, rank), "ncclCommInitRank");
  // every rank's (first row, rows), once: the offsets of the first-invalid translation and
  // the check that the shards tile [0, n_total) in rank order
  long long* d = nullptr;
  cuda_check(cudaMalloc(&d, sizeof(long long) * 2 * (1 + world)), "cudaMalloc");
  const long long mine[2] = {l.offset, l.ds->n};
  // (on the group's stream: a pageable cudaMemcpy on the legacy stream may return before its
  // DMA lands, and l.stream -- non-blocking -- does not order behind it)
  cuda_check(cudaMemcpyAsync(d, mine, sizeof(mine), cudaMemcpyHostToDevice, l.stream), "cudaMemcpyAsync");
  nccl_check(api.all_gather(d, d + 2, 2, ncclInt64, l.comm, l.stream), "ncclAllGather(offsets)");
  std::vector<long long> all(2 * world);
  cuda_check(cudaMemcpyAsync(all.data(), d + 2, sizeof(long long) * 2 * world, cudaMemcpyDeviceToHost, l.stream),
             "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(l.stream), "offsets exchange");
  cudaFree(d);
  long long next = 0;
  for (int r = 0; r < world; ++r) {
    if (all[2 * r] != next) {
      usage_error("shard group: rank " + std::to_string(r) + " starts at row " + std::to_string(all[2 * r]) +
                  ", expected " + std::to_string(next) + " (ranks must own contiguous ranges in rank order)");
    }
    g->offsets_.push_back(all[2 * r]);
    next += all[2 * r + 1];
  }
  if (next != n_total) {
    usage_error("shard group: the shards hold " + std::to_string(next) + " rows, n_total is " +
                std::to_string(n_total));
  }
  g->finish_setup();
  return g;
}

std::unique_ptr<ShardGroup> ShardGroup::create_local(const Model& m, const std::vector<std::string>& names,
                                                     const std::vector<const double*>& host_cols, long long n_total,
                                                     const std::vector<int>& devices) {
  const int G = static_cast<int>(devices.size());
  if (G < 1) usage_error("shard group: no devices");
  if (names.size() != host_cols.size() || names.empty()) usage_error("shard group: names / columns mismatch");
  const NcclApi& api = nccl();
  std::unique_ptr<ShardGroup> g(new ShardGroup(m, n_total, G));
  for (int r = 0; r < G; ++r) {
    const long long b = n_total * r / G, e = n_total * (r + 1) / G;
    Local L;
    L.device = devices[r];
    L.rank = r;
    L.offset = b;
    DeviceGuard dg(L.device);
    std::vector<const double*> part;
    for (const double* c : host_cols) part.push_back(c + b);
    L.ds = DeviceDataset::upload(names, part, e - b);
    L.engine = std::make_unique<Engine>(m);
    cuda_check(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    g->offsets_.push_back(b);
    g->local_.push_back(std::move(L));
  }
  std::vector<ncclComm_t> comms(G);
  nccl_check(api.comm_init_all(comms.data(), G, devices.data()), "ncclCommInitAll");
  for (int r = 0; r < G; ++r) g->local_[r].comm = comms[r];
  g->finish_setup();
  return g;
}

void ShardGroup::finish_setup() {
  for (Local& L : local_) {
    DeviceGuard dg(L.device);
    cuda_check(cudaMalloc(&L.d_offsets, sizeof(long long) * world_), "cudaMalloc(offsets)");
    cuda_check(cudaMemcpyAsync(L.d_offsets, offsets_.data(), sizeof(long long) * world_, cudaMemcpyHostToDevice,
                               L.stream),
               "cudaMemcpyAsync(offsets)");
    cuda_check(cudaStreamSynchronize(L.stream), "offsets upload");
  }
}

ShardGroup::~ShardGroup() {
  for (Local& L : local_) {
    DeviceGuard dg(L.device);
    if (L.stream) cudaStreamSynchronize(L.stream);
    if (L.comm) nccl().comm_destroy(L.comm);
    cuda_free_all({L.d_send, L.d_recv, L.d_pairs, L.d_bad, L.d_offsets});
    L.engine.reset();
    if (L.stream) cudaStreamDestroy(L.stream);
  }
  if (h_pairs_) cudaFreeHost(h_pairs_);
  if (h_bad_) cudaFreeHost(h_bad_);
}

void ShardGroup::ensure_words(Local& L, std::size_t words, int rows) {
  if (words <= L.cap_words && static_cast<std::size_t>(rows) * 2 <= L.cap_words) return;
  const std::size_t cap = std::max<std::size_t>(words, 3 * 64);
  DeviceGuard dg(L.device);
  cuda_check(cudaStreamSynchronize(L.stream), "cudaStreamSynchronize");
  cuda_free_all({L.d_send, L.d_recv, L.d_pairs, L.d_bad});
  cuda_check(cudaMalloc(&L.d_send, cap * sizeof(double)), "cudaMalloc(send)");
  cuda_check(cudaMalloc(&L.d_recv, cap * world_ * sizeof(double)), "cudaMalloc(recv)");
  // rows <= words / 2 and P <= words: both outputs fit cap entries
  cuda_check(cudaMalloc(&L.d_pairs, cap * sizeof(SumPair)), "cudaMalloc(pairs)");
  cuda_check(cudaMalloc(&L.d_bad, cap * sizeof(unsigned long long)), "cudaMalloc(bad)");
  L.cap_words = cap;
}

void ShardGroup::exchange(std::size_t words, int rows, int P) {
  const NcclApi& api = nccl();
  nccl_check(api.group_start(), "ncclGroupStart");
  for (Local& L : local_) {
    nccl_check(api.all_gather(L.d_send, L.d_recv, words, ncclUint64, L.comm, L.stream), "ncclAllGather");
  }
  nccl_check(api.group_end(), "ncclGroupEnd");
  for (Local& L : local_) {
    DeviceGuard dg(L.device);
    count_launches(launch_combine_shards(L.d_recv, world_, rows, P, L.d_offsets, L.d_pairs, L.d_bad, L.stream));
    cuda_check(cudaGetLastError(), "combine_shards");
  }
}

NllResult ShardGroup::nll_points(const double* thetas, int P) {
  NllResult r;
  r.value.resize(P);
  r.pairs.resize(P);
  r.first_invalid.resize(P);
  const int npar = static_cast<int>(m_.params.size());
  for (int p0 = 0; p0 < P; p0 += kMaxPointsPerLaunch) {
    const int np = std::min(kMaxPointsPerLaunch, P - p0);
    const double* th = thetas + static_cast<std::size_t>(p0) * npar;
    const std::size_t words = 3 * static_cast<std::size_t>(np);
    for (Local& L : local_) {
      ensure_words(L, words, np);
      // the reduce kernel writes the pairs and the first-invalid indices straight into the
      // send buffer: [np pairs | np indices]
      r.launches += L.engine->nll_points_device(*L.ds, th, np, reinterpret_cast<SumPair*>(L.d_send),
                                                reinterpret_cast<unsigned long long*>(L.d_send + 2 * np), L.stream);
    }
    exchange(words, np, np);
    r.launches += 1;
    Local& L0 = local_[0];
    if (static_cast<std::size_t>(np) > cap_host_) {
      if (h_pairs_) cudaFreeHost(h_pairs_);
      if (h_bad_) cudaFreeHost(h_bad_);
      cap_host_ = std::max<std::size_t>(np, 64);
      cuda_check(cudaHostAlloc(&h_pairs_, cap_host_ * sizeof(SumPair), cudaHostAllocDefault), "cudaHostAlloc");
      cuda_check(cudaHostAlloc(&h_bad_, cap_host_ * sizeof(unsigned long long), cudaHostAllocDefault),
                 "cudaHostAlloc");
    }
    DeviceGuard dg(L0.device);
    cuda_check(cudaMemcpyAsync(h_pairs_, L0.d_pairs, np * sizeof(SumPair), cudaMemcpyDeviceToHost, L0.stream),
               "cudaMemcpyAsync(pairs)");
    cuda_check(cudaMemcpyAsync(h_bad_, L0.d_bad, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, L0.stream),
               "cudaMemcpyAsync(bad)");
    for (Local& L : local_) {
      DeviceGuard g2(L.device);
      cuda_check(cudaStreamSynchronize(L.stream), "sharded nll");
    }
    for (int i = 0; i < np; ++i) {
      const int p = p0 + i;
      r.pairs[p] = h_pairs_[i];
      const bool bad = h_bad_[i] != kNoInvalid;
      r.first_invalid[p] = bad ? static_cast<long long>(h_bad_[i]) : -1;
      r.value[p] = bad ? std::numeric_limits<double>::infinity()
                       : h_pairs_[i].s + h_pairs_[i].c +
                             m_.extended_term(th + static_cast<std::size_t>(i) * npar, static_cast<double>(n_total_));
    }
  }
  return r;
}

int ShardGroup::nll_points_device(const double* thetas, int P, SumPair* d_pairs, unsigned long long* d_bad,
                                  cudaStream_t stream, cudaStream_t upload_stream) {
  if (local_.size() != 1) usage_error("nll_points_device: one local device per group (create_rank)");
  if (P <= 0) return 0;
  if (P > kMaxPointsPerLaunch) usage_error("nll_points_device: at most 512 points per call");
  Local& L = local_[0];
  DeviceGuard dg(L.device);
  cudaStream_t s = stream ? stream : L.stream;
  const std::size_t words = 3 * static_cast<std::size_t>(P);
  ensure_words(L, words, P);
  int launches = L.engine->nll_points_device(*L.ds, thetas, P, reinterpret_cast<SumPair*>(L.d_send),
                                             reinterpret_cast<unsigned long long*>(L.d_send + 2 * P), s,
                                             upload_stream);
  nccl_check(nccl().all_gather(L.d_send, L.d_recv, words, ncclUint64, L.comm, s), "ncclAllGather");
  launches += launch_combine_shards(L.d_recv, world_, P, P, L.d_offsets, d_pairs, d_bad, s);
  count_launches(1);
  cuda_check(cudaGetLastError(), "combine_shards");
  return launches;
}

bool ShardGroup::grad_ok() { return local_[0].engine->grad_plan().ok; }

void ShardGroup::reserve(int P_nll, int P_grad) {
  int S = 0;
  if (P_grad > 0 && grad_ok()) S = local_[0].engine->grad_plan().dev.nslots;
  for (Local& L : local_) {
    L.engine->reserve(*L.ds, P_nll, P_grad);
    const int pn = std::min(P_nll, kMaxPointsPerLaunch), pg = std::min(P_grad, kMaxPointsPerLaunch);
    const std::size_t words = std::max<std::size_t>(3 * static_cast<std::size_t>(pn),
                                                    static_cast<std::size_t>(pg) * (2 * S + 1));
    ensure_words(L, words, std::max(pn, pg * std::max(S, 1)));
  }
}

NllGradResult ShardGroup::nll_grad_points(const double* thetas, int P) {
  Engine& e0 = *local_[0].engine;
  const GradPlan& gp = e0.grad_plan();
  if (!gp.ok) usage_error("analytic gradient unavailable for this model: " + gp.why);
  const int npar = static_cast<int>(m_.params.size());
  const int S = gp.dev.nslots;
  NllGradResult r;
  r.nslots = S;
  r.value.resize(P);
  r.grad.resize(static_cast<std::size_t>(P) * npar);
  r.first_invalid.resize(P);
  r.slots.resize(static_cast<std::size_t>(P) * S);
  std::vector<double> stage, sums;
  std::vector<SumPair> hp;
  std::vector<unsigned long long> hb;
  for (int p0 = 0; p0 < P; p0 += kMaxPointsPerLaunch) {
    const int np = std::min(kMaxPointsPerLaunch, P - p0);
    const double* th = thetas + static_cast<std::size_t>(p0) * npar;
    const int rows = np * S;
    const std::size_t words = 2 * static_cast<std::size_t>(rows) + np;
    for (Local& L : local_) {
      // this rank's slot pairs (events of its shard) and local first-invalid indices
      const NllGradResult lr = L.engine->nll_grad_points(*L.ds, th, np);
      r.launches += lr.launches;
      stage.resize(words);
      std::memcpy(stage.data(), lr.slots.data(), sizeof(SumPair) * rows);
      for (int i = 0; i < np; ++i) {
        const unsigned long long b = lr.first_invalid[i] < 0 ? kNoInvalid : static_cast<unsigned long long>(lr.first_invalid[i]);
        std::memcpy(&stage[2 * static_cast<std::size_t>(rows) + i], &b, sizeof(b));
      }
      ensure_words(L, words, rows);
      DeviceGuard dg(L.device);
      cuda_check(cudaMemcpyAsync(L.d_send, stage.data(), words * sizeof(double), cudaMemcpyHostToDevice, L.stream),
                 "cudaMemcpyAsync(send)");
    }
    exchange(words, rows, np);
    r.launches += 1;
    Local& L0 = local_[0];
    hp.resize(rows);
    hb.resize(np);
    {
      DeviceGuard dg(L0.device);
      cuda_check(cudaMemcpyAsync(hp.data(), L0.d_pairs, rows * sizeof(SumPair), cudaMemcpyDeviceToHost, L0.stream),
                 "cudaMemcpyAsync(slots)");
      cuda_check(cudaMemcpyAsync(hb.data(), L0.d_bad, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 L0.stream),
                 "cudaMemcpyAsync(bad)");
    }
    for (Local& L : local_) {
      DeviceGuard g2(L.device);
      cuda_check(cudaStreamSynchronize(L.stream), "sharded gradient");
    }
    sums.resize(rows);
    for (int k = 0; k < rows; ++k) {
      r.slots[static_cast<std::size_t>(p0) * S + k] = hp[k];
      sums[k] = hp[k].s + hp[k].c;
    }
    e0.grad_finish(th, np, sums.data(), static_cast<double>(n_total_), r.value.data() + p0,
                   r.grad.data() + static_cast<std::size_t>(p0) * npar);
    for (int i = 0; i < np; ++i) {
      const int p = p0 + i;
      const bool bad = hb[i] != kNoInvalid;
      r.first_invalid[p] = bad ? static_cast<long long>(hb[i]) : -1;
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

}  // namespace ffb
