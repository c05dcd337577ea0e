#include "jit.hpp"

#include <cuda.h>  // driver API types only: the functions come from cudaGetDriverEntryPoint
#include <dlfcn.h>
#include <nvrtc.h>  // NVRTC types only: the library is dlopen'ed

#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <vector>

namespace ffb {

namespace {

#include "jit_sources.inc"  // kJitHeaders: the device headers as strings (embed_sources.py)

// ---------------------------------------------------------------------------
// NVRTC, loaded at run time

struct NvrtcApi {
  bool ok = false;
  std::string why;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcAddNameExpression) add_name = nullptr;
  decltype(&nvrtcGetLoweredName) lowered = nullptr;
  decltype(&nvrtcGetErrorString) error = nullptr;
};

NvrtcApi& nvrtc() {
  static NvrtcApi api = [] {
    NvrtcApi a;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      a.why = std::string("libnvrtc not found (") + dlerror() + ")";
      return a;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f) a.why = std::string("libnvrtc lacks ") + name;
      return f != nullptr;
    };
    a.ok = sym(a.create, "nvrtcCreateProgram") && sym(a.destroy, "nvrtcDestroyProgram") &&
           sym(a.compile, "nvrtcCompileProgram") && sym(a.log_size, "nvrtcGetProgramLogSize") &&
           sym(a.log, "nvrtcGetProgramLog") && sym(a.cubin_size, "nvrtcGetCUBINSize") &&
           sym(a.cubin, "nvrtcGetCUBIN") && sym(a.add_name, "nvrtcAddNameExpression") &&
           sym(a.lowered, "nvrtcGetLoweredName") && sym(a.error, "nvrtcGetErrorString");
    return a;
  }();
  return api;
}

// ---------------------------------------------------------------------------
// driver entry points (through cudart: no link-time libcuda dependency)

struct DriverApi {
  bool ok = false;
  std::string why;
  CUresult (*module_load)(CUmodule*, const void*) = nullptr;
  CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
};

DriverApi& driver() {
  static DriverApi api = [] {
    DriverApi a;
    auto get = [&](auto& f, const char* name) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
        a.why = std::string("driver entry point ") + name + " unavailable";
        return false;
      }
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(p);
      return true;
    };
    a.ok = get(a.module_load, "cuModuleLoadData") && get(a.get_function, "cuModuleGetFunction") &&
           get(a.launch, "cuLaunchKernel") && get(a.set_attribute, "cuFuncSetAttribute") &&
           get(a.occupancy, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    return a;
  }();
  return api;
}

// ---------------------------------------------------------------------------

std::atomic<bool> g_enabled{std::getenv("FFB_NO_EXPR_JIT") == nullptr};
std::mutex g_mu;
std::string g_status = "not used yet";

constexpr int kJitThreads = 256;
constexpr int kJitE = 8;
constexpr int kJitTile = kJitThreads * kJitE;
constexpr int kJitStages = 3;   // kernels_device.cuh kStreamStages
constexpr int kJitStreamMaxP = 8;
constexpr int kModeAll = 2;     // kernels_device.cuh kKsAll

struct Module {
  CUmodule mod = nullptr;
  CUfunction tile = nullptr;
  CUfunction stream = nullptr;  // single-column single-sum plans only
  int tile_occ = 1, stream_occ = 1;
};
std::map<std::pair<int, std::string>, Module> g_modules;  // (device, source)

std::string hexbits(double v) {
  unsigned long long b;
  std::memcpy(&b, &v, 8);
  char buf[48];
  std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxll)", b);
  return buf;
}

// The smallest kind set covering the plan's other leaves (the formulas are in every
// set of a formula-specialised build): ArgusBG may meet p != 1/2 at run time, so it
// takes the full set, as ChiSquare / JohnsonSU do.
int jit_kind_set(const HostPlan& plan) {
  int ks = 0;
  for (int i = 0; i < plan.dev.nterms; ++i) {
    const int k = plan.dev.t[i].kind;
    if (k == LK_CHISQ || k == LK_JOHNSON || k == LK_ARGUS) return kModeAll;
    if (k == LK_CHEB || k == LK_POLY) ks = 1;
  }
  return ks;
}

std::string tile_name(const HostPlan& plan) {
  const bool onecol = plan.dev.ncols == 1;
  const int mode = jit_kind_set(plan) + (plan.dev.simple ? 0 : 3);
  return "&ffb::nll_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(kJitE) + ", " +
         (onecol ? "true" : "false") + ", 2, " + std::to_string(mode) + ">";
}
std::string stream_name(const HostPlan& plan) {
  return "&ffb::nll_stream_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(kJitE) + ", 2, " +
         std::to_string(jit_kind_set(plan)) + ">";
}
bool has_stream(const HostPlan& plan) { return plan.dev.ncols == 1 && plan.dev.simple; }

// Compiles source to sm_100a SASS; the lowered names of `names` in `lowered`.
bool compile(const std::string& source, const std::vector<std::string>& names, std::vector<char>* cubin,
             std::vector<std::string>* lowered, std::string* log) {
  NvrtcApi& api = nvrtc();
  if (!api.ok) {
    *log = api.why;
    return false;
  }
  std::vector<const char*> hdr_src, hdr_name;
  for (const auto& h : kJitHeaders) {
    hdr_name.push_back(h.name);
    hdr_src.push_back(h.text);
  }
  nvrtcProgram prog = nullptr;
  if (api.create(&prog, source.c_str(), "ffb_expr_jit.cu", static_cast<int>(hdr_src.size()), hdr_src.data(),
                 hdr_name.data()) != NVRTC_SUCCESS) {
    *log = "nvrtcCreateProgram failed";
    return false;
  }
  for (const auto& n : names) api.add_name(prog, n.c_str());
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                        "--device-as-default-execution-space", "-diag-suppress=128"};
  const nvrtcResult rc = api.compile(prog, 5, opts);
  std::size_t ls = 0;
  api.log_size(prog, &ls);
  std::string l(ls, '\0');
  if (ls) api.log(prog, l.data());
  *log = l;
  bool ok = rc == NVRTC_SUCCESS;
  if (ok && cubin) {
    std::size_t cs = 0;
    api.cubin_size(prog, &cs);
    cubin->resize(cs);
    api.cubin(prog, cubin->data());
    for (const auto& n : names) {
      const char* low = nullptr;
      if (api.lowered(prog, n.c_str(), &low) != NVRTC_SUCCESS || !low) {
        ok = false;
        *log += "\nno lowered name for " + n;
        break;
      }
      lowered->push_back(low);
    }
  } else if (!ok) {
    *log = std::string(api.error(rc)) + "\n" + l;
  }
  api.destroy(&prog);
  return ok;
}

std::string full_source(const HostPlan& plan) {
  return jit_expression_source(plan) + "#include \"kernels_device.cuh\"\n";
}

}  // namespace

std::string jit_expression_source(const HostPlan& plan) {
  std::ostringstream o;
  // exp / log / sqrt take the kernels' table-driven, branch-free forms on their safe
  // domains (<= 2 ulp, fastmath.cuh) and libdevice outside them, so NaN / inf / zero /
  // negative arguments keep the IEEE results the reference would see
  o << "// generated by jit.cpp: the model's Expression formulas as straight-line device code\n"
       "#define FFB_EXPR_JIT 1\n"
       "#include \"fastmath.cuh\"\n"
       "namespace ffb {\n"
       "__device__ __forceinline__ double ffb_pow(double a, double b) {\n"
       "  if (b == 2.0) return __dmul_rn(a, a);\n"
       "  if (b == 3.0) return __dmul_rn(__dmul_rn(a, a), a);\n"
       "  if (b == 4.0) { const double a2 = __dmul_rn(a, a); return __dmul_rn(a2, a2); }\n"
       "  return pow(a, b);\n"
       "}\n"
       // branch-free: the special cases are selected, not branched to, so the compiler
       // keeps interleaving the E independent events of a thread
       "__device__ __forceinline__ double ffb_exp(double a, const MathTables* __restrict__ tb) {\n"
       "  const double r = fast_exp(a == a ? a : 0.0, tb);\n"
       "  return a == a ? r : a;\n"
       "}\n"
       "__device__ __forceinline__ double ffb_log(double a, const MathTables* __restrict__ tb) {\n"
       "  const double inf = __longlong_as_double(0x7ff0000000000000LL);\n"
       "  const bool ok = a > 0.0 && a < inf;\n"
       "  const double r = fast_log(ok ? a : 1.0, tb);\n"
       "  return ok ? r : (a == 0.0 ? -inf : (a == inf ? inf : __longlong_as_double(0x7ff8000000000000LL)));\n"
       "}\n"
       "__device__ __forceinline__ double ffb_sqrt(double a) {\n"
       "  const double inf = __longlong_as_double(0x7ff0000000000000LL);\n"
       "  const bool ok = a > 0.0 && a < inf;\n"
       "  const bool tiny = a < 0x1p-1000;\n"
       "  double r = fast_sqrt_unit(ok ? (tiny ? a * 0x1p108 : a) : 1.0);\n"
       "  r = tiny ? r * 0x1p-54 : r;\n"
       "  return ok ? r : ((a == 0.0 || a == inf) ? a : __longlong_as_double(0x7ff8000000000000LL));\n"
       "}\n"
       // division by a point-uniform divisor: RN(1/d) hoisted by the compiler across the
       // events, one correction step (div_by: the IEEE quotient bar rare 1-ulp cases)
       "__device__ __forceinline__ double ffb_div_uniform(double a, double d) {\n"
       "  return div_by(a, d, __drcp_rn(d));\n"
       "}\n";
  std::vector<int> offsets;
  for (int i = 0; i < plan.dev.nterms; ++i) {
    if (plan.dev.t[i].kind != LK_EXPR) continue;
    const int off = plan.dev.t[i].order;
    bool seen = false;
    for (const int s : offsets) seen = seen || s == off;
    if (seen) continue;
    offsets.push_back(off);
    // stack slots are named by depth: the postfix program is straight-line code
    int depth = 0, max_depth = 0;
    std::ostringstream body;
    std::vector<bool> uni(kExprMaxDepth + 1, false);  // the slot depends on constants / parameters only
    for (std::size_t j = static_cast<std::size_t>(off); plan.programs[j].op != EX_END; ++j) {
      const ExprInstr& in = plan.programs[j];
      auto s = [](int d) { return "s" + std::to_string(d); };
      switch (in.op) {
        case EX_CONST: body << "  " << s(depth) << " = " << hexbits(in.c) << ";\n"; uni[depth] = true; ++depth; break;
        case EX_VAR: body << "  " << s(depth) << " = k[" << 1 + in.slot << "];\n"; uni[depth] = true; ++depth; break;
        case EX_X: body << "  " << s(depth) << " = x;\n"; uni[depth] = false; ++depth; break;
        case EX_ADD: --depth; body << "  " << s(depth - 1) << " = __dadd_rn(" << s(depth - 1) << ", " << s(depth) << ");\n"; break;
        case EX_SUB: --depth; body << "  " << s(depth - 1) << " = __dsub_rn(" << s(depth - 1) << ", " << s(depth) << ");\n"; break;
        case EX_MUL: --depth; body << "  " << s(depth - 1) << " = __dmul_rn(" << s(depth - 1) << ", " << s(depth) << ");\n"; break;
        case EX_DIV:
          --depth;
          body << "  " << s(depth - 1) << " = " << (uni[depth] && !uni[depth - 1] ? "ffb_div_uniform(" : "__ddiv_rn(")
               << s(depth - 1) << ", " << s(depth) << ");\n";
          break;
        case EX_POW: --depth; body << "  " << s(depth - 1) << " = ffb_pow(" << s(depth - 1) << ", " << s(depth) << ");\n"; break;
        case EX_NEG: body << "  " << s(depth - 1) << " = -" << s(depth - 1) << ";\n"; break;
        case EX_SQUARE: body << "  " << s(depth - 1) << " = __dmul_rn(" << s(depth - 1) << ", " << s(depth - 1) << ");\n"; break;
        case EX_CUBE:
          body << "  " << s(depth - 1) << " = __dmul_rn(__dmul_rn(" << s(depth - 1) << ", " << s(depth - 1) << "), "
               << s(depth - 1) << ");\n";
          break;
        case EX_FOURTH:
          body << "  { const double t = __dmul_rn(" << s(depth - 1) << ", " << s(depth - 1) << "); " << s(depth - 1)
               << " = __dmul_rn(t, t); }\n";
          break;
        default: {
          const bool tab = in.op == EX_EXP || in.op == EX_LOG;
          const char* f = in.op == EX_EXP ? "ffb_exp" : in.op == EX_LOG ? "ffb_log" : in.op == EX_SIN ? "sin"
                        : in.op == EX_COS ? "cos" : in.op == EX_SQRT ? "ffb_sqrt" : in.op == EX_ABS ? "fabs"
                        : in.op == EX_SINH ? "sinh" : "asinh";
          body << "  " << s(depth - 1) << " = " << f << "(" << s(depth - 1) << (tab ? ", tb" : "") << ");\n";
          break;
        }
      }
      switch (in.op) {  // binary operators: the result is uniform iff both operands were
        case EX_ADD: case EX_SUB: case EX_MUL: case EX_DIV: case EX_POW:
          uni[depth - 1] = uni[depth - 1] && uni[depth];
          break;
        default:
          break;
      }
      if (depth > max_depth) max_depth = depth;
    }
    o << "__device__ __forceinline__ double ffb_expr_" << off
      << "(double x, const double* __restrict__ k, const MathTables* __restrict__ tb) {\n";
    o << "  (void)x; (void)k; (void)tb;\n";
    for (int d = 0; d < max_depth; ++d) o << "  double s" << d << ";\n";
    o << body.str() << "  return s0;\n}\n";
  }
  o << "template <int E>\n"
       "__device__ __forceinline__ void ffb_expr_batch(int off, const double* __restrict__ k, const double (&x)[E],\n"
       "                                               double (&v)[E], const MathTables* __restrict__ tb) {\n"
       "  switch (off) {\n";
  for (const int off : offsets) {
    o << "    case " << off << ":\n#pragma unroll\n      for (int e = 0; e < E; ++e) v[e] = ffb_expr_" << off
      << "(x[e], k, tb);\n      break;\n";
  }
  o << "    default:\n      break;\n  }\n}\n}  // namespace ffb\n";
  return o.str();
}

bool jit_enabled() { return g_enabled.load(); }
void jit_enable(bool on) { g_enabled.store(on); }

std::string jit_status() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_status;
}

bool jit_compile_only(const HostPlan& plan, std::string* log) {
  std::vector<std::string> names = {tile_name(plan)};
  if (has_stream(plan)) names.push_back(stream_name(plan));
  std::vector<char> cubin;
  std::vector<std::string> low;
  return compile(full_source(plan), names, &cubin, &low, log);
}

namespace {

Module* module_for(const HostPlan& plan) {
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string src = full_source(plan);
  const auto key = std::make_pair(dev, src);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_modules.find(key);
  if (it != g_modules.end()) return it->second.mod ? &it->second : nullptr;
  Module m;  // a failed compile is cached too (mod stays null): no retry per launch
  DriverApi& drv = driver();
  std::vector<std::string> names = {tile_name(plan)};
  if (has_stream(plan)) names.push_back(stream_name(plan));
  std::vector<char> cubin;
  std::vector<std::string> lowered;
  std::string log;
  if (!drv.ok) {
    g_status = "interpreter: " + drv.why;
  } else if (!compile(src, names, &cubin, &lowered, &log)) {
    g_status = "interpreter: NVRTC compile failed: " + log.substr(0, 2000);
  } else {
    cudaFree(nullptr);  // the runtime's primary context is current before the driver call
    if (drv.module_load(&m.mod, cubin.data()) != CUDA_SUCCESS ||
        drv.get_function(&m.tile, m.mod, lowered[0].c_str()) != CUDA_SUCCESS ||
        (has_stream(plan) && drv.get_function(&m.stream, m.mod, lowered[1].c_str()) != CUDA_SUCCESS)) {
      m.mod = nullptr;
      g_status = "interpreter: loading the NVRTC module failed";
    } else {
      const int tile_smem = kMaxCols * kJitTile * static_cast<int>(sizeof(double));
      drv.set_attribute(m.tile, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, tile_smem);
      drv.occupancy(&m.tile_occ, m.tile, kJitThreads, plan.dev.ncols * kJitTile * sizeof(double));
      if (m.tile_occ < 1) m.tile_occ = 1;
      if (m.stream) {
        const int ss = kJitStages * kJitTile * static_cast<int>(sizeof(double));
        drv.set_attribute(m.stream, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, ss);
        drv.occupancy(&m.stream_occ, m.stream, kJitThreads, ss);
        if (m.stream_occ < 1) m.stream_occ = 1;
      }
      g_status = "jit: formula-specialised kernels (NVRTC, sm_100a)";
    }
  }
  auto& slot = g_modules[key];
  slot = m;
  return slot.mod ? &slot : nullptr;
}

}  // namespace

bool jit_prepare(const HostPlan& plan) {
  if (!jit_enabled() || plan.programs.empty()) return false;
  return module_for(plan) != nullptr;
}

NllLaunchInfo launch_nll_jit(const HostPlan& plan, const ColPtrs& cols, long long n, const double* d_consts, int P,
                             void* scratch, SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream,
                             cudaEvent_t ev_start, cudaEvent_t ev_stop) {
  NllLaunchInfo info;
  if (P <= 0) return info;
  Module* m = module_for(plan);
  if (!m) usage_error("internal: launch_nll_jit without a module");
  DriverApi& drv = driver();
  const int sms = device_sm_count();
  DevPlan dp = plan.dev;
  ColPtrs cp = cols;
  long long nn = n;
  const double* kc = d_consts;
  int PP = P;
  SumPair* partial = static_cast<SumPair*>(scratch);
  unsigned long long* bad = d_bad;
  cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long) * P, stream);
  const long long ntl = (n + kJitTile - 1) / kJitTile;
  bool aligned = true;
  for (int c = 0; c < plan.dev.ncols; ++c) aligned = aligned && (reinterpret_cast<uintptr_t>(cols.c[c]) & 15) == 0;
  CUresult rc;
  int rows;
  if (m->stream && P <= kJitStreamMaxP && aligned && std::getenv("FFB_NO_STREAM") == nullptr) {
    long long G = static_cast<long long>(sms) * m->stream_occ;
    if (G > ntl) G = ntl;
    int ntiles = static_cast<int>(ntl);
    void* args[] = {&dp, &cp, &nn, &kc, &PP, &ntiles, &partial, &bad};
    if (ev_start) cudaEventRecord(ev_start, stream);
    rc = drv.launch(m->stream, static_cast<unsigned>(G), 1, 1, kJitThreads, 1, 1,
                    kJitStages * kJitTile * sizeof(double), reinterpret_cast<CUstream>(stream), args, nullptr);
    if (ev_stop) cudaEventRecord(ev_stop, stream);
    rows = static_cast<int>(G);
    info.nchunks = 0;
    info.grid = static_cast<int>(G);
  } else {
    int ntiles = static_cast<int>(ntl < 1 ? 1 : ntl);
    const long long slots = static_cast<long long>(sms) * m->tile_occ;
    long long want = (8 * slots + ntiles - 1) / ntiles;
    if (want < 1) want = 1;
    if (want > P) want = P;
    int pchunk = static_cast<int>((P + want - 1) / want);
    const int nchunks = (P + pchunk - 1) / pchunk;
    void* args[] = {&dp, &cp, &nn, &kc, &PP, &pchunk, &ntiles, &partial, &bad};
    if (ev_start) cudaEventRecord(ev_start, stream);
    rc = drv.launch(m->tile, static_cast<unsigned>(static_cast<long long>(ntiles) * nchunks), 1, 1, kJitThreads, 1, 1,
                    plan.dev.ncols * kJitTile * sizeof(double), reinterpret_cast<CUstream>(stream), args, nullptr);
    if (ev_stop) cudaEventRecord(ev_stop, stream);
    rows = ntiles;
    info.nchunks = nchunks;
    info.grid = ntiles * nchunks;
  }
  if (rc != CUDA_SUCCESS) numeric_error("cuLaunchKernel (formula-specialised likelihood) failed: " + std::to_string(rc));
  launch_reduce(partial, rows, P, d_out, stream);
  info.threads = kJitThreads;
  info.events_per_thread = kJitE;
  info.tile = kJitTile;
  info.ntiles = static_cast<int>(ntl);
  info.launches = 2;
  info.jit = 1;
  return info;
}

}  // namespace ffb
