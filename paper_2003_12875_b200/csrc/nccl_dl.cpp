#include "nccl_dl.hpp"

#include <dlfcn.h>

#include <mutex>

#include "common.hpp"

namespace ffb {

namespace {

template <class F>
bool bind(void* h, const char* name, F& f, std::string& why) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) why = std::string("NCCL: missing symbol ") + name;
  return f != nullptr;
}

NcclApi load() {
  NcclApi a;
  // a copy already in the process (PyTorch's) first, then the loader's search path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW);
  if (!h) {
    const char* e = dlerror();
    a.why = std::string("NCCL not loadable: ") + (e ? e : "libnccl.so.2 not found");
    return a;
  }
  bool ok = bind(h, "ncclGetUniqueId", a.get_unique_id, a.why) &&
            bind(h, "ncclCommInitRank", a.comm_init_rank, a.why) &&
            bind(h, "ncclCommInitAll", a.comm_init_all, a.why) &&
            bind(h, "ncclCommDestroy", a.comm_destroy, a.why) &&
            bind(h, "ncclAllGather", a.all_gather, a.why) && bind(h, "ncclGroupStart", a.group_start, a.why) &&
            bind(h, "ncclGroupEnd", a.group_end, a.why) && bind(h, "ncclGetErrorString", a.error_string, a.why) &&
            bind(h, "ncclGetVersion", a.get_version, a.why);
  if (!ok) return a;
  int v = 0;
  if (a.get_version(&v) == ncclSuccess) {
    // NCCL >= 2.9: major * 10000 + minor * 100 + patch
    a.version = std::to_string(v / 10000) + "." + std::to_string((v / 100) % 100) + "." + std::to_string(v % 100);
  }
  a.ok = true;
  return a;
}

}  // namespace

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  std::call_once(once, [] { api = load(); });
  if (!api.ok) numeric_error(api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclApi& a = nccl();
  numeric_error(std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
}

}  // namespace ffb
