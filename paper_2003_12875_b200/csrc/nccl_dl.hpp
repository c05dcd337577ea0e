// NCCL, loaded at run time (dlopen) for the event-sharded likelihood (shard.cpp).
//
// The library does not link NCCL: a process that already holds one (PyTorch loads its
// bundled libnccl.so.2) shares it -- two NCCL builds under one soname in one process would
// collide -- and a C caller gets the system's.  Only the entry points the exchange step
// needs are bound.  nccl.h supplies the types.
#pragma once

#include <nccl.h>

#include <string>

namespace ffb {

struct NcclApi {
  bool ok = false;
  std::string why;      // when !ok: what failed to load
  std::string version;  // "major.minor.patch" of the library actually bound
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

// Binds on first use; throws Numeric (with the loader's message) if NCCL is unavailable.
const NcclApi& nccl();

// Throws Numeric with NCCL's message when r is not ncclSuccess.
void nccl_check(ncclResult_t r, const char* what);

}  // namespace ffb
