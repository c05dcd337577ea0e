// Event-sharded likelihood over several GPUs: every rank owns a
// contiguous range of the events of every column, resident in its HBM for the whole fit;
// a batch of P parameter points is ONE fused launch per rank plus ONE collective:
//
//   rank r:  nll launch -> [P Neumaier pairs | P local first-invalid indices]  (3P words,
//            written by the reduce kernel straight into the send buffer)
//   all:     ncclAllGather of the 3P words            (NVLink / NVSwitch; 24P bytes per rank)
//   rank r:  combine_shards_kernel: pairs combined in rank order (bitwise independent of
//            NCCL's algorithm, identical on every rank), first invalid = lowest rank's,
//            shifted by that rank's first global row
//   host:    value = s + c + the extended term with the GLOBAL event count
//
// Gradients (the fused NLL + gradient pass) exchange their P x nslots slot pairs the same
// way and finish on the host with the global N.  Two topologies share the code:
//   * create_rank: one process per GPU (torchrun / MPI-style), the caller distributes an
//     ncclUniqueId (ffcu_nccl_unique_id on rank 0);
//   * create_local: one process driving G devices (ncclCommInitAll), the host columns cut
//     into G contiguous shards and uploaded.
// A ShardGroup is a LikelihoodSource, so the fit drivers (fit.hpp) run on it unchanged:
// BASELINE config 5's sharded fit.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "fit.hpp"
#include "nccl_dl.hpp"

namespace ffb {

class ShardGroup : public LikelihoodSource {
 public:
  static std::unique_ptr<ShardGroup> create_rank(const Model& m, std::shared_ptr<DeviceDataset> shard,
                                                 long long n_total, long long offset, const ncclUniqueId& id,
                                                 int world, int rank);
  static std::unique_ptr<ShardGroup> create_local(const Model& m, const std::vector<std::string>& names,
                                                  const std::vector<const double*>& host_cols, long long n_total,
                                                  const std::vector<int>& devices);
  ~ShardGroup() override;
  ShardGroup(const ShardGroup&) = delete;
  ShardGroup& operator=(const ShardGroup&) = delete;

  // LikelihoodSource: synchronous, combined over all ranks, identical on every rank
  NllResult nll_points(const double* thetas, int P) override;
  NllGradResult nll_grad_points(const double* thetas, int P) override;
  bool grad_ok() override;
  void reserve(int P_nll, int P_grad) override;

  // Asynchronous on `stream` (single local device): the combined pairs (events only, no
  // extended term) and global first-invalid indices of P <= 512 points stay on the device.
  // upload_stream (optional): where the constant rows are copied (a pipeline's copy stream).
  int nll_points_device(const double* thetas, int P, SumPair* d_pairs, unsigned long long* d_bad,
                        cudaStream_t stream, cudaStream_t upload_stream = nullptr);

  int world() const { return world_; }
  int local_count() const { return static_cast<int>(local_.size()); }
  long long n_total() const { return n_total_; }
  long long local_rows(int i) const { return local_[i].ds->n; }
  long long local_offset(int i) const { return local_[i].offset; }
  int local_rank(int i) const { return local_[i].rank; }
  const std::vector<long long>& offsets() const { return offsets_; }
  Engine& engine(int i) { return *local_[i].engine; }

 private:
  struct Local {
    int device = 0;
    int rank = 0;
    long long offset = 0;
    std::shared_ptr<DeviceDataset> ds;
    std::unique_ptr<Engine> engine;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    double* d_send = nullptr;   // one rank block
    double* d_recv = nullptr;   // world rank blocks
    SumPair* d_pairs = nullptr;  // combined
    unsigned long long* d_bad = nullptr;
    long long* d_offsets = nullptr;
    std::size_t cap_words = 0;  // of d_send (rows * 2 + P)
  };
  ShardGroup(const Model& m, long long n_total, int world) : m_(m), n_total_(n_total), world_(world) {}
  void finish_setup();                       // offsets on every local device
  void ensure_words(Local& L, std::size_t words, int rows);
  // the all-gather of `words` per rank + the combine, on every local device's stream
  void exchange(std::size_t words, int rows, int P);

  const Model& m_;
  long long n_total_;
  int world_;
  std::vector<long long> offsets_;  // every rank's first global row
  std::vector<Local> local_;
  SumPair* h_pairs_ = nullptr;  // pinned read-back of local device 0
  unsigned long long* h_bad_ = nullptr;
  std::size_t cap_host_ = 0;
};

}  // namespace ffb
