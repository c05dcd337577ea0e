#include "jit.hpp"

#include <cuda.h>  // driver API types only: the functions come from cudaGetDriverEntryPoint
#include <dlfcn.h>
#include <nvrtc.h>  // NVRTC types only: the library is dlopen'ed

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <sstream>
#include <vector>

namespace ffb {

std::string plan_spec_struct(const DevPlan& d);

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

// FFB_JIT_OPTS (extra NVRTC options, read at every compile) is part of every build cache key:
// a process can hold a build and its A/B variant side by side (bench.py's per-event-log line).
std::string opts_key() {
  const char* e = std::getenv("FFB_JIT_OPTS");
  return e ? std::string("\n// opts: ") + e : std::string();
}
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
  int smem_cols = 1;  // data columns + cached formula subtrees
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

// formula builds are plan-specialised too (PlanSpec); MODE + 6 (the launch-constant
// builds) when the launch caches formula subtrees
std::string tile_name(const HostPlan& plan, bool hoisted) {
  const bool onecol = plan.dev.ncols == 1;
  const int mode = jit_kind_set(plan) + (plan.dev.simple ? 0 : 3) + (hoisted ? 6 : 0);
  return "&ffb::nll_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(kJitE) + ", " +
         (onecol ? "true" : "false") + ", 2, " + std::to_string(mode) + ", ffb::PlanSpec>";
}
std::string stream_name(const HostPlan& plan) {
  return "&ffb::nll_stream_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(kJitE) + ", 2, " +
         std::to_string(jit_kind_set(plan)) + ", ffb::PlanSpec>";
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
  std::vector<std::string> extra;  // FFB_JIT_OPTS: extra NVRTC options (A/B builds, e.g. -DFFB_CONST_BANK)
  if (const char* e = std::getenv("FFB_JIT_OPTS")) {
    std::istringstream is(e);
    for (std::string w; is >> w;) extra.push_back(w);
  }
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                                   "--device-as-default-execution-space", "-diag-suppress=128"};
  for (const auto& w : extra) opts.push_back(w.c_str());
  const nvrtcResult rc = api.compile(prog, static_cast<int>(opts.size()), opts.data());
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
    if (const char* dump = std::getenv("FFB_JIT_DUMP")) {  // debugging: cuobjdump the generated builds
      static std::atomic<int> seq{0};
      const std::string path = std::string(dump) + "." + std::to_string(seq++) + ".cubin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(cubin->data(), 1, cs, f);
        std::fclose(f);
      }
    }
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

// ---------------------------------------------------------------------------
// formula code generation (jit_expression_source)

// Emits the stack code of program instructions [b, e) as a scoped block whose value ends
// in the E-array `result`.  Ranges listed in `hoisted` (launch-constant subtrees) push
// their cached shared-memory column instead of being computed.
void emit_block(std::ostream& o, const std::vector<ExprInstr>& prog, int b, int e,
                const std::vector<const HoistSlot*>* hoisted, const std::string& result) {
  int depth = 0, max_depth = 0;
  std::ostringstream body;
  std::vector<bool> uni(kExprMaxDepth + 2, false);  // the slot holds one value for every event
  auto S = [](int d) { return "s" + std::to_string(d); };
  // a uniform slot is a scalar u<d>; the others are arrays s<d>[E]
  auto U = [](int d) { return "u" + std::to_string(d); };
  auto elem = [&](int d) { return uni[d] ? U(d) : S(d) + "[e]"; };
  auto loop = [&](const std::string& stmt) {
    body << "#pragma unroll\n  for (int e = 0; e < E; ++e) " << stmt << "\n";
  };
  auto widen = [&](int d) {  // make slot d an array (before a per-event op writes it)
    if (uni[d]) {
      loop(S(d) + "[e] = " + U(d) + ";");
      uni[d] = false;
    }
  };
  for (int j = b; j < e; ++j) {
    const HoistSlot* h = nullptr;
    if (hoisted) {
      for (const HoistSlot* c : *hoisted) h = c->begin == j ? c : h;
    }
    if (h) {  // the whole subtree [begin, end] from the tile's cache
      loop(S(depth) + "[e] = dsm[" + std::to_string(h->col) + " * (T * E) + e * T];");
      uni[depth] = false;
      ++depth;
      if (depth > max_depth) max_depth = depth;
      j = h->end;
      continue;
    }
    const ExprInstr& in = prog[j];
    switch (in.op) {
      case EX_CONST:
        body << "  " << U(depth) << " = " << hexbits(in.c) << ";\n";
        uni[depth] = true;
        ++depth;
        break;
      case EX_VAR:
        body << "  " << U(depth) << " = k[" << 1 + in.slot << "];\n";
        uni[depth] = true;
        ++depth;
        break;
      case EX_X:
        loop(S(depth) + "[e] = x[e];");
        uni[depth] = false;
        ++depth;
        break;
      case EX_ADD: case EX_SUB: case EX_MUL: case EX_POW: case EX_DIV: {
        --depth;
        const int l = depth - 1, r = depth;
        const char* fn = in.op == EX_ADD ? "__dadd_rn" : in.op == EX_SUB ? "__dsub_rn" : in.op == EX_MUL ? "__dmul_rn"
                       : in.op == EX_POW ? "ffb_pow" : "__ddiv_rn";
        if (uni[l] && uni[r]) {  // both uniform: a scalar (the compiler computes it once)
          body << "  " << U(l) << " = " << fn << "(" << U(l) << ", " << U(r) << ");\n";
        } else if (in.op == EX_DIV && uni[r]) {
          body << "  ffb_vdiv_uniform<E>(" << S(l) << ", " << U(r) << ");\n";
        } else if (in.op == EX_DIV) {
          widen(l);
          widen(r);
          body << "  ffb_vdiv<E>(" << S(l) << ", " << S(r) << ");\n";
        } else {
          const std::string lhs = elem(l), rhs = elem(r);
          loop(S(l) + "[e] = " + fn + "(" + lhs + ", " + rhs + ");");
          uni[l] = false;
        }
        break;
      }
      default: {  // unary
        const int d = depth - 1;
        if (uni[d]) {  // a uniform operand stays scalar: libdevice / IEEE, computed once
          const char* f = in.op == EX_NEG ? "-" : in.op == EX_EXP ? "exp" : in.op == EX_LOG ? "log"
                        : in.op == EX_SIN ? "sin" : in.op == EX_COS ? "cos" : in.op == EX_SQRT ? "__dsqrt_rn"
                        : in.op == EX_ABS ? "fabs" : in.op == EX_SINH ? "sinh" : in.op == EX_ASINH ? "asinh"
                        : nullptr;
          if (in.op == EX_SQUARE) {
            body << "  " << U(d) << " = __dmul_rn(" << U(d) << ", " << U(d) << ");\n";
          } else if (in.op == EX_CUBE) {
            body << "  " << U(d) << " = __dmul_rn(__dmul_rn(" << U(d) << ", " << U(d) << "), " << U(d) << ");\n";
          } else if (in.op == EX_FOURTH) {
            body << "  { const double t = __dmul_rn(" << U(d) << ", " << U(d) << "); " << U(d)
                 << " = __dmul_rn(t, t); }\n";
          } else {
            body << "  " << U(d) << " = " << f << "(" << U(d) << ");\n";
          }
          break;
        }
        const std::string a = S(d) + "[e]";
        switch (in.op) {
          case EX_NEG: loop(a + " = -" + a + ";"); break;
          case EX_SQUARE: loop(a + " = __dmul_rn(" + a + ", " + a + ");"); break;
          case EX_CUBE: loop(a + " = __dmul_rn(__dmul_rn(" + a + ", " + a + "), " + a + ");"); break;
          case EX_FOURTH: loop("{ const double t = __dmul_rn(" + a + ", " + a + "); " + a + " = __dmul_rn(t, t); }"); break;
          case EX_EXP: body << "  ffb_vexp<E>(" << S(d) << ", tb);\n"; break;
          case EX_LOG: body << "  ffb_vlog<E>(" << S(d) << ", tb);\n"; break;
          case EX_SQRT: body << "  ffb_vsqrt<E>(" << S(d) << ");\n"; break;
          case EX_ABS: loop(a + " = fabs(" + a + ");"); break;
          case EX_SIN: loop(a + " = sin(" + a + ");"); break;
          case EX_COS: loop(a + " = cos(" + a + ");"); break;
          case EX_SINH: loop(a + " = sinh(" + a + ");"); break;
          default: loop(a + " = asinh(" + a + ");"); break;
        }
        break;
      }
    }
    if (depth > max_depth) max_depth = depth;
  }
  o << "  {\n";
  for (int d = 0; d < max_depth; ++d) o << "  double s" << d << "[E];\n  double u" << d << ";\n";
  o << body.str();
  if (uni[0]) {
    o << "#pragma unroll\n  for (int e = 0; e < E; ++e) " << result << "[e] = u0;\n";
  } else {
    o << "#pragma unroll\n  for (int e = 0; e < E; ++e) " << result << "[e] = s0[e];\n";
  }
  o << "  }\n";
}

int program_end(const std::vector<ExprInstr>& prog, int off) {
  int j = off;
  while (prog[j].op != EX_END) ++j;
  return j;
}

// One formula function: `name`(x, k, v, tb) or, with hoisted ranges, name<E, T>(..., dsm).
void emit_formula(std::ostream& o, const std::vector<ExprInstr>& prog, int off,
                  const std::vector<const HoistSlot*>* hoisted, const std::string& name, bool with_dsm) {
  if (with_dsm) {
    o << "template <int E, int T>\n__device__ __forceinline__ void " << name
      << "(const double (&x)[E], const double* __restrict__ k, double (&v)[E], const MathTables* __restrict__ tb,\n"
         "    const double* __restrict__ dsm) {\n  (void)x; (void)k; (void)tb; (void)dsm;\n";
  } else {
    o << "template <int E>\n__device__ __forceinline__ void " << name
      << "(const double (&x)[E], const double* __restrict__ k, double (&v)[E], const MathTables* __restrict__ tb) {\n"
      << "  (void)x; (void)k; (void)tb;\n";
  }
  emit_block(o, prog, off, program_end(prog, off), hoisted, "v");
  o << "}\n";
}

// The forward-mode tangent of a formula (the analytic gradient of Expression leaves in the
// plan-specialised gradient pass): d value / d t for the variables whose slot bit is set in
// `seed` moving by t; values and tangents per event, libdevice math (accuracy, not bits:
// the pass's NLL slot comes from the leaf values of pass 1).
void emit_tangent(std::ostream& o, const std::vector<ExprInstr>& prog, int off, const std::string& name) {
  std::ostringstream b;
  int depth = 0, max_depth = 0;
  auto V = [](int d) { return "v" + std::to_string(d) + "[e]"; };
  auto T = [](int d) { return "t" + std::to_string(d) + "[e]"; };
  auto loop = [&](const std::string& stmt) {
    b << "#pragma unroll\n  for (int e = 0; e < E; ++e) { " << stmt << " }\n";
  };
  const int end = program_end(prog, off);
  for (int j = off; j < end; ++j) {
    const ExprInstr& in = prog[j];
    switch (in.op) {
      case EX_CONST:
        loop(V(depth) + " = " + hexbits(in.c) + "; " + T(depth) + " = 0.0;");
        ++depth;
        break;
      case EX_VAR:
        loop(V(depth) + " = k[" + std::to_string(1 + in.slot) + "]; " + T(depth) + " = ((seed >> " +
             std::to_string(in.slot) + ") & 1) ? 1.0 : 0.0;");
        ++depth;
        break;
      case EX_X:
        loop(V(depth) + " = x[e]; " + T(depth) + " = 0.0;");
        ++depth;
        break;
      case EX_ADD: case EX_SUB: case EX_MUL: case EX_DIV: case EX_POW: {
        --depth;
        const int l = depth - 1, r = depth;
        const std::string a = V(l), bb = V(r), ta = T(l), tb = T(r);
        if (in.op == EX_ADD) {
          loop(a + " = " + a + " + " + bb + "; " + ta + " = " + ta + " + " + tb + ";");
        } else if (in.op == EX_SUB) {
          loop(a + " = " + a + " - " + bb + "; " + ta + " = " + ta + " - " + tb + ";");
        } else if (in.op == EX_MUL) {
          loop(ta + " = " + ta + " * " + bb + " + " + a + " * " + tb + "; " + a + " = " + a + " * " + bb + ";");
        } else if (in.op == EX_DIV) {
          loop("const double q = " + a + " / " + bb + "; " + ta + " = (" + ta + " - q * " + tb + ") / " + bb + "; " +
               a + " = q;");
        } else {
          loop("const double r = ffb_pow(" + a + ", " + bb + "); " + ta + " = (" + ta + " != 0.0 ? " + bb +
               " * pow(" + a + ", " + bb + " - 1.0) * " + ta + " : 0.0) + (" + tb + " != 0.0 ? r * log(" + a +
               ") * " + tb + " : 0.0); " + a + " = r;");
        }
        break;
      }
      default: {
        const int d = depth - 1;
        const std::string a = V(d), t = T(d);
        std::string r, g;  // value, derivative of the op at a
        switch (in.op) {
          case EX_NEG: r = "-a"; g = "-1.0"; break;
          case EX_SQUARE: r = "a * a"; g = "2.0 * a"; break;
          case EX_CUBE: r = "a * a * a"; g = "3.0 * a * a"; break;
          case EX_FOURTH: r = "(a * a) * (a * a)"; g = "4.0 * a * a * a"; break;
          case EX_EXP: r = "exp(a)"; g = "r"; break;
          case EX_LOG: r = "log(a)"; g = "1.0 / a"; break;
          case EX_SIN: r = "sin(a)"; g = "cos(a)"; break;
          case EX_COS: r = "cos(a)"; g = "-sin(a)"; break;
          case EX_SQRT: r = "sqrt(a)"; g = "0.5 / r"; break;
          case EX_ABS: r = "fabs(a)"; g = "(a < 0.0 ? -1.0 : 1.0)"; break;
          case EX_SINH: r = "sinh(a)"; g = "cosh(a)"; break;
          default: r = "asinh(a)"; g = "1.0 / sqrt(a * a + 1.0)"; break;
        }
        loop("const double a = " + a + "; const double r = " + r + "; " + t + " = " + t + " != 0.0 ? (" + g +
             ") * " + t + " : 0.0; " + a + " = r;");
        break;
      }
    }
    if (depth > max_depth) max_depth = depth;
  }
  o << "template <int E>\n__device__ __forceinline__ void " << name
    << "(const double (&x)[E], const double* __restrict__ k, int seed, double (&dv)[E]) {\n"
    << "  (void)x; (void)k; (void)seed;\n";
  for (int d = 0; d < max_depth; ++d) o << "  double v" << d << "[E], t" << d << "[E];\n";
  o << b.str() << "#pragma unroll\n  for (int e = 0; e < E; ++e) dv[e] = t0[e];\n}\n";
}

}  // namespace

ExprHoist analyse_expr_hoist(const HostPlan& plan, const double* rows, int P) {
  ExprHoist out;
  if (!rows || P < 2) return out;
  const DevPlan& d = plan.dev;
  int next_col = d.ncols + d.ncached;
  auto bits = [](double v) {
    unsigned long long b;
    std::memcpy(&b, &v, sizeof b);
    return b;
  };
  for (int i = 0; i < d.nterms; ++i) {
    const DevTerm& t = d.t[i];
    if (t.kind != LK_EXPR) continue;
    int users = 0;
    for (int k = 0; k < d.nterms; ++k) users += (d.t[k].kind == LK_EXPR && d.t[k].order == t.order) ? 1 : 0;
    if (users != 1) continue;  // a program shared by several terms: not cached (per-term columns)
    const int off = t.order, end = program_end(plan.programs, off);
    const int n = end - off;
    std::vector<int> start(n), parent(n, -1), cost(n, 0);
    std::vector<char> inv(n, 0), hasx(n, 0);
    std::vector<int> st;
    auto uniform = [&](int slot) {
      const double* k0 = rows + t.coff + 1 + slot;
      for (int p = 1; p < P; ++p) {
        if (bits(k0[static_cast<std::size_t>(p) * d.stride]) != bits(*k0)) return false;
      }
      return true;
    };
    for (int j = 0; j < n; ++j) {
      const ExprInstr& in = plan.programs[off + j];
      switch (in.op) {
        case EX_CONST: start[j] = j; inv[j] = 1; st.push_back(j); break;
        case EX_VAR: start[j] = j; inv[j] = uniform(in.slot) ? 1 : 0; st.push_back(j); break;
        case EX_X: start[j] = j; inv[j] = 1; hasx[j] = 1; st.push_back(j); break;
        case EX_ADD: case EX_SUB: case EX_MUL: case EX_POW: case EX_DIV: {
          const int r = st.back(); st.pop_back();
          const int l = st.back(); st.pop_back();
          parent[l] = parent[r] = j;
          start[j] = start[l];
          inv[j] = inv[l] && inv[r];
          hasx[j] = hasx[l] || hasx[r];
          cost[j] = cost[l] + cost[r] + ((in.op == EX_POW || in.op == EX_DIV) ? 8 : 1);
          st.push_back(j);
          break;
        }
        default: {
          const int c = st.back(); st.pop_back();
          parent[c] = j;
          start[j] = start[c];
          inv[j] = inv[c];
          hasx[j] = hasx[c];
          const bool heavy = in.op == EX_EXP || in.op == EX_LOG || in.op == EX_SQRT || in.op == EX_SIN ||
                             in.op == EX_COS || in.op == EX_SINH || in.op == EX_ASINH;
          cost[j] = cost[c] + (heavy ? 8 : 1);
          st.push_back(j);
          break;
        }
      }
    }
    for (int j = 0; j < n; ++j) {
      const bool maximal = parent[j] < 0 || !inv[parent[j]];
      if (!inv[j] || !hasx[j] || !maximal || cost[j] < 3) continue;  // x alone / cheap: not worth a column
      if (next_col >= kMaxCols) break;
      out.slots.push_back(HoistSlot{i, off, off + start[j], off + j, next_col++, t.col, t.coff});
    }
  }
  return out;
}

std::string jit_expression_source(const HostPlan& plan, const ExprHoist* hoist) {
  // Each formula becomes code over the thread's E events at once (one array per stack
  // depth, every operation an unrolled loop), so the compiler interleaves the events.
  // exp / log / sqrt / division take branch-free fast forms (fastmath.cuh, <= 2 ulp; the
  // division's hoisted-reciprocal correction step is the IEEE quotient bar rare 1-ulp
  // cases) on the operands where those are exact enough; one warp vote per operation
  // sends the rare other operands (zero, negative, subnormal, inf, NaN) to the IEEE /
  // libdevice form, so special values come out as the reference computes them.
  std::ostringstream o;
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
       "__device__ __forceinline__ bool ffb_pos_normal(double a) {  // finite, > 0, not subnormal\n"
       "  return static_cast<unsigned>(__double2hiint(a)) - 0x00100000u < 0x7fe00000u;\n"
       "}\n"
       "template <int E>\n"
       "__device__ __forceinline__ void ffb_vexp(double (&a)[E], const MathTables* __restrict__ tb) {\n"
       "  bool rare = false;\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) {\n"
       "    const bool ok = a[e] == a[e];\n"
       "    rare |= !ok;\n"
       "    a[e] = ok ? fast_exp(a[e], tb) : a[e];\n"
       "  }\n"
       "  (void)rare;\n"
       "}\n"
       "template <int E>\n"
       "__device__ __forceinline__ void ffb_vlog(double (&a)[E], const MathTables* __restrict__ tb) {\n"
       "  bool ok[E], rare = false;\n"
       "  double r[E];\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) {\n"
       "    ok[e] = ffb_pos_normal(a[e]);\n"
       "    rare |= !ok[e];\n"
       "    r[e] = fast_log(ok[e] ? a[e] : 1.0, tb);\n"
       "  }\n"
       "  if (__any_sync(0xffffffffu, rare)) {\n"
       "#pragma unroll\n"
       "    for (int e = 0; e < E; ++e) r[e] = ok[e] ? r[e] : log(a[e]);\n"
       "  }\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) a[e] = r[e];\n"
       "}\n"
       "template <int E>\n"
       "__device__ __forceinline__ void ffb_vsqrt(double (&a)[E]) {\n"
       "  bool ok[E], rare = false;\n"
       "  double r[E];\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) {\n"
       "    ok[e] = ffb_pos_normal(a[e]);\n"
       "    rare |= !ok[e];\n"
       "    r[e] = fast_sqrt_unit(ok[e] ? a[e] : 1.0);\n"
       "  }\n"
       "  if (__any_sync(0xffffffffu, rare)) {\n"
       "#pragma unroll\n"
       "    for (int e = 0; e < E; ++e) r[e] = ok[e] ? r[e] : __dsqrt_rn(a[e]);\n"
       "  }\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) a[e] = r[e];\n"
       "}\n"
       // a / d with d the same for every event of the point: RN(1/d) once, one correction
       "template <int E>\n"
       "__device__ __forceinline__ void ffb_vdiv_uniform(double (&a)[E], double d) {\n"
       "  const double inv = __drcp_rn(d);\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) a[e] = div_by(a[e], d, inv);\n"
       "}\n"
       // a / b per event: fast reciprocal + correction where both are ordinary numbers
       "template <int E>\n"
       "__device__ __forceinline__ void ffb_vdiv(double (&a)[E], const double (&b)[E]) {\n"
       "  bool ok[E], rare = false;\n"
       "  double r[E];\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) {\n"
       "    const double m = fabs(b[e]);\n"
       "    ok[e] = m >= 0x1p-1000 && m <= 0x1p1000 && fabs(a[e]) <= 0x1p1000;\n"
       "    rare |= !ok[e];\n"
       "    const double bb = ok[e] ? b[e] : 1.0;\n"
       "    r[e] = div_by(a[e], bb, fast_rcp_signed(bb));\n"
       "  }\n"
       "  if (__any_sync(0xffffffffu, rare)) {\n"
       "#pragma unroll\n"
       "    for (int e = 0; e < E; ++e) r[e] = ok[e] ? r[e] : __ddiv_rn(a[e], b[e]);\n"
       "  }\n"
       "#pragma unroll\n"
       "  for (int e = 0; e < E; ++e) a[e] = r[e];\n"
       "}\n";
  // per program offset: the hoisted ranges (launch-constant subtrees, ExprHoist)
  std::map<int, std::vector<const HoistSlot*>> by_prog;
  if (hoist) {
    for (const HoistSlot& h : hoist->slots) by_prog[h.prog].push_back(&h);
  }
  std::vector<int> offsets;
  for (int i = 0; i < plan.dev.nterms; ++i) {
    if (plan.dev.t[i].kind != LK_EXPR) continue;
    const int off = plan.dev.t[i].order;
    bool seen = false;
    for (const int sv : offsets) seen = seen || sv == off;
    if (seen) continue;
    offsets.push_back(off);
    emit_formula(o, plan.programs, off, nullptr, "ffb_expr_" + std::to_string(off), false);
    emit_tangent(o, plan.programs, off, "ffb_expr_" + std::to_string(off) + "_t");
    auto it = by_prog.find(off);
    if (it != by_prog.end()) {
      emit_formula(o, plan.programs, off, &it->second, "ffb_expr_" + std::to_string(off) + "_h", true);
    }
  }
  o << "template <int E>\n"
       "__device__ __forceinline__ void ffb_expr_batch(int off, const double* __restrict__ k, const double (&x)[E],\n"
       "                                               double (&v)[E], const MathTables* __restrict__ tb) {\n"
       "  switch (off) {\n";
  for (const int off : offsets) o << "    case " << off << ": ffb_expr_" << off << "<E>(x, k, v, tb); break;\n";
  o << "    default: break;\n  }\n}\n";
  // the gradient pass's tangents (kernels_device.cuh leaf_grad, formula builds)
  o << "template <int E>\n"
       "__device__ __forceinline__ void ffb_expr_tangent(int off, const double* __restrict__ k, const double (&x)[E],\n"
       "                                                 int seed, double (&dv)[E]) {\n"
       "  switch (off) {\n";
  for (const int off : offsets) o << "    case " << off << ": ffb_expr_" << off << "_t<E>(x, k, seed, dv); break;\n";
  o << "    default: break;\n  }\n}\n";
  if (hoist && !hoist->slots.empty()) {
    // the launch-constant subtrees: computed once per staged tile (nll_kernel) into
    // shared-memory columns, read by the _h formulas for every point
    o << "#define FFB_EXPR_HOIST 1\n"
         "template <int E, int T>\n"
         "__device__ __forceinline__ void ffb_expr_batch_h(int off, const double* __restrict__ k, const double (&x)[E],\n"
         "                                                 double (&v)[E], const MathTables* __restrict__ tb,\n"
         "                                                 const double* __restrict__ dsm) {\n"
         "  (void)dsm;\n  switch (off) {\n";
    for (const int off : offsets) {
      if (by_prog.count(off)) {
        o << "    case " << off << ": ffb_expr_" << off << "_h<E, T>(x, k, v, tb, dsm); break;\n";
      } else {
        o << "    case " << off << ": ffb_expr_" << off << "<E>(x, k, v, tb); break;\n";
      }
    }
    o << "    default: break;\n  }\n}\n";
    o << "template <int E, int T>\n"
         "__device__ __forceinline__ void ffb_expr_hoist(const double* __restrict__ row, double* __restrict__ dsm,\n"
         "                                               const MathTables* __restrict__ tb) {\n"
         "  (void)tb;\n";
    for (const HoistSlot& h : hoist->slots) {
      o << "  {  // column " << h.col << ": program " << h.prog << " instructions [" << h.begin << ", " << h.end
        << "] of term " << h.term << "\n"
        << "    const double* __restrict__ k = row + " << h.coff << ";\n    double x[E];\n"
        << "#pragma unroll\n    for (int e = 0; e < E; ++e) x[e] = dsm[" << h.xcol << " * (T * E) + e * T];\n"
        << "    double r[E];\n";
      emit_block(o, plan.programs, h.begin, h.end + 1, nullptr, "r");
      o << "#pragma unroll\n    for (int e = 0; e < E; ++e) dsm[" << h.col << " * (T * E) + e * T] = r[e];\n  }\n";
    }
    o << "}\n";
  }
  o << "}  // namespace ffb\n";
  return o.str();
}

namespace {

// ---------------------------------------------------------------------------
// plan-specialised gradient pass (kernels_device.cuh nll_grad_spec_kernel)

// events per thread and pipeline stages of the plan-specialised gradient pass: single-column
// single sums keep 8 events per thread and three stages; multi-column / product plans hold
// the factor sums per event too, so 4 events and two stages (nll_grad_spec_kernel)
constexpr int kGradSpecMaxCols = 3;
int grad_spec_e(const DevPlan& d) { return d.simple && d.ncols == 1 ? 8 : 4; }
int grad_spec_smem(const DevPlan& d) {
  return (d.ncols == 1 ? kJitStages : 2) * d.ncols * kJitThreads * grad_spec_e(d) * static_cast<int>(sizeof(double));
}
std::string grad_spec_name(const DevPlan& d, int ks) {
  return "&ffb::nll_grad_spec_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(grad_spec_e(d)) + ", " +
         std::to_string(ks) + ">";
}

struct SpecModule {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  int occ = 1;
};
std::map<std::tuple<int, std::string, int>, SpecModule> g_spec;  // (device, source, kind set)

std::string grad_spec_source(const HostPlan& plan, const GradPlan& gp) {
  std::ostringstream o;
  const int nt = plan.dev.nterms;
  auto arr = [&](auto f) {
    std::ostringstream a;
    for (int i = 0; i < nt; ++i) a << (i ? ", " : "") << f(i);
    return a.str();
  };
  if (!plan.programs.empty()) o << jit_expression_source(plan);  // the formulas and their tangents
  int nseed = 0;
  for (int i = 0; i < nt; ++i) {
    if (plan.dev.t[i].kind == LK_EXPR) nseed = std::max(nseed, gp.dev.g[i].seeds + __builtin_popcount(gp.dev.g[i].pmask));
  }
  std::ostringstream seeds;
  for (int i = 0; i < std::max(nseed, 1); ++i) seeds << (i ? ", " : "") << (i < nseed ? gp.dev.seed[i] : 0);
  o << "// generated by jit.cpp: the plan's term list and slot layout for nll_grad_spec_kernel\n"
       "namespace ffb {\nstruct GradSpec {\n"
    << "  static constexpr int nterms = " << nt << ";\n"
    << "  static constexpr int seedoff[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].seeds; }) << "};\n"
    << "  static constexpr int seed[" << std::max(nseed, 1) << "] = {" << seeds.str() << "};\n"
    << "  static constexpr int kind[" << nt << "] = {" << arr([&](int i) { return plan.dev.t[i].kind; }) << "};\n"
    << "  static constexpr int order[" << nt << "] = {" << arr([&](int i) { return plan.dev.t[i].order; }) << "};\n"
    << "  static constexpr int pmask[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].pmask; }) << "};\n"
    << "  static constexpr int aslot[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].slot; }) << "};\n"
    << "  static constexpr int nslots = " << gp.dev.nslots << ";\n"
    << "  static constexpr int ncols = " << plan.dev.ncols << ";\n"
    << "  static constexpr bool simple = " << (plan.dev.simple ? "true" : "false") << ";\n"
    << "  static constexpr int nfactors = " << gp.dev.nfactors << ";\n"
    << "  static constexpr int col[" << nt << "] = {" << arr([&](int i) { return plan.dev.t[i].col; }) << "};\n"
    << "  static constexpr int flags[" << nt << "] = {" << arr([&](int i) { return plan.dev.t[i].flags; }) << "};\n"
    << "  static constexpr int factor[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].factor; }) << "};\n"
    << "  static constexpr int fbeg[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].fbeg; }) << "};\n"
    << "  static constexpr int fend[" << nt << "] = {" << arr([&](int i) { return gp.dev.g[i].fend; }) << "};\n"
    << "};\n}  // namespace ffb\n"
    << "#define FFB_GRAD_SPEC 1\n#include \"kernels_device.cuh\"\n";
  return o.str();
}

SpecModule* spec_module(const HostPlan& plan, const GradPlan& gp, int ks) {
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string src = grad_spec_source(plan, gp);
  const auto key = std::make_tuple(dev, src + opts_key(), ks);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_spec.find(key);
  if (it != g_spec.end()) return it->second.mod ? &it->second : nullptr;
  SpecModule m;
  DriverApi& drv = driver();
  const std::string name = grad_spec_name(plan.dev, ks);
  std::vector<char> cubin;
  std::vector<std::string> lowered;
  std::string log;
  if (drv.ok && compile(src, {name}, &cubin, &lowered, &log)) {
    cudaFree(nullptr);
    if (drv.module_load(&m.mod, cubin.data()) == CUDA_SUCCESS &&
        drv.get_function(&m.fn, m.mod, lowered[0].c_str()) == CUDA_SUCCESS) {
      const int smem = grad_spec_smem(plan.dev);
      drv.set_attribute(m.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
      drv.occupancy(&m.occ, m.fn, kJitThreads, smem);
      if (m.occ < 1) m.occ = 1;
    } else {
      m.mod = nullptr;
    }
  }
  if (!m.mod) g_status = "gradient pass: generic kernels (" + (drv.ok ? log.substr(0, 2000) : drv.why) + ")";
  auto& slot = g_spec[key];
  slot = m;
  return slot.mod ? &slot : nullptr;
}

}  // namespace

std::string grad_spec_text(const HostPlan& plan, const GradPlan& gp) { return grad_spec_source(plan, gp); }

bool grad_spec_compile_only(const HostPlan& plan, const GradPlan& gp, int ks, std::string* log) {
  std::vector<char> cubin;
  std::vector<std::string> low;
  return compile(grad_spec_source(plan, gp), {grad_spec_name(plan.dev, ks)}, &cubin, &low, log);
}

bool grad_spec_applies(const HostPlan& plan, const GradPlan& gp, const ColPtrs& cols, int P) {
  if (!jit_enabled() || !gp.ok || P != 1 || plan.dev.ncols > kGradSpecMaxCols) return false;
  if (std::getenv("FFB_NO_GRAD_SPEC") || std::getenv("FFB_NO_STREAM")) return false;
  for (int c = 0; c < plan.dev.ncols; ++c) {
    if (reinterpret_cast<uintptr_t>(cols.c[c]) & 15) return false;
  }
  return true;
}

bool grad_spec_prepare(const HostPlan& plan, const GradPlan& gp, int ks) {
  return spec_module(plan, gp, ks) != nullptr;
}

NllLaunchInfo launch_nll_grad_spec(const HostPlan& plan, const GradPlan& gp, const ColPtrs& cols, long long n,
                                   const double* d_consts, void* scratch, SumPair* d_out,
                                   unsigned long long* d_bad, cudaStream_t stream, int ks, cudaEvent_t ev_start,
                                   cudaEvent_t ev_stop) {
  NllLaunchInfo info;
  SpecModule* m = spec_module(plan, gp, ks);
  if (!m) usage_error("internal: launch_nll_grad_spec without a module");
  DriverApi& drv = driver();
  const int stile = kJitThreads * grad_spec_e(plan.dev);
  const long long ntl = (n + stile - 1) / stile;
  long long G = static_cast<long long>(device_sm_count()) * m->occ;
  if (G > ntl) G = ntl;
  DevPlan dp = plan.dev;
  ColPtrs cp = cols;
  long long nn = n;
  const double* kc = d_consts;
  int ntiles = static_cast<int>(ntl);
  SumPair* partial = static_cast<SumPair*>(scratch);
  unsigned long long* bad = d_bad;
  void* args[] = {&dp, &cp, &nn, &kc, &ntiles, &partial, &bad};
  cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), stream);
  if (ev_start) cudaEventRecord(ev_start, stream);
  const CUresult rc = drv.launch(m->fn, static_cast<unsigned>(G), 1, 1, kJitThreads, 1, 1, grad_spec_smem(plan.dev),
                                 reinterpret_cast<CUstream>(stream), args, nullptr);
  if (ev_stop) cudaEventRecord(ev_stop, stream);
  if (rc != CUDA_SUCCESS) numeric_error("cuLaunchKernel (plan-specialised gradient) failed: " + std::to_string(rc));
  launch_reduce(partial, static_cast<int>(G), gp.dev.nslots, d_out, stream);
  info.threads = kJitThreads;
  info.events_per_thread = grad_spec_e(plan.dev);
  info.tile = stile;
  info.ntiles = static_cast<int>(ntl);
  info.grid = static_cast<int>(G);
  info.launches = 2;
  info.jit = 1;
  return info;
}

bool jit_enabled() { return g_enabled.load(); }
void jit_enable(bool on) { g_enabled.store(on); }

std::string jit_status() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_status;
}

namespace {

// formula builds: the generated formulas (with the launch's cached subtrees), the plan's
// term list (PlanSpec) and the fused kernels
std::string full_source(const HostPlan& plan, const ExprHoist* hoist) {
  return "#define FFB_CONST_BANK 1\n" + jit_expression_source(plan, hoist) + plan_spec_struct(plan.dev) +
         "#include \"kernels_device.cuh\"\n";
}

int hoist_cols(const ExprHoist* hoist) { return hoist ? static_cast<int>(hoist->slots.size()) : 0; }

}  // namespace

bool jit_compile_only(const HostPlan& plan, std::string* log, const ExprHoist* hoist) {
  const bool h = hoist_cols(hoist) > 0;
  std::vector<std::string> names = {tile_name(plan, h)};
  if (has_stream(plan)) names.push_back(stream_name(plan));
  std::vector<char> cubin;
  std::vector<std::string> low;
  return compile(full_source(plan, hoist), names, &cubin, &low, log);
}

namespace {

Module* module_for(const HostPlan& plan, const ExprHoist* hoist) {
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string src = full_source(plan, hoist);
  const auto key = std::make_pair(dev, src + opts_key());
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_modules.find(key);
  if (it != g_modules.end()) return it->second.mod ? &it->second : nullptr;
  Module m;  // a failed compile is cached too (mod stays null): no retry per launch
  DriverApi& drv = driver();
  const int hc = hoist_cols(hoist);
  std::vector<std::string> names = {tile_name(plan, hc > 0)};
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
      m.smem_cols = plan.dev.ncols + hc;
      drv.occupancy(&m.tile_occ, m.tile, kJitThreads, m.smem_cols * kJitTile * sizeof(double));
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
  return module_for(plan, nullptr) != nullptr;
}

NllLaunchInfo launch_nll_jit(const HostPlan& plan, const ColPtrs& cols, long long n, const double* d_consts, int P,
                             void* scratch, SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream,
                             const double* h_rows, cudaEvent_t ev_start, cudaEvent_t ev_stop) {
  NllLaunchInfo info;
  if (P <= 0) return info;
  DriverApi& drv = driver();
  const int sms = device_sm_count();
  bool aligned = true;
  for (int c = 0; c < plan.dev.ncols; ++c) aligned = aligned && (reinterpret_cast<uintptr_t>(cols.c[c]) & 15) == 0;
  const bool streaming = has_stream(plan) && P <= kJitStreamMaxP && aligned && std::getenv("FFB_NO_STREAM") == nullptr;
  // launch-constant formula subtrees (tile kernel only): cached per staged tile
  ExprHoist hoist;
  if (!streaming && std::getenv("FFB_NO_CONST_CACHE") == nullptr) hoist = analyse_expr_hoist(plan, h_rows, P);
  const ExprHoist* hp = hoist.slots.empty() ? nullptr : &hoist;
  Module* m = module_for(plan, hp);
  if (!m && hp) {  // the cached build failed to compile: the plain formula build
    hp = nullptr;
    m = module_for(plan, nullptr);
  }
  if (!m) usage_error("internal: launch_nll_jit without a module");
  DevPlan dp = plan.dev;
  ColPtrs cp = cols;
  long long nn = n;
  const double* kc = d_consts;
  int PP = P;
  SumPair* partial = static_cast<SumPair*>(scratch);
  unsigned long long* bad = d_bad;
  cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long) * P, stream);
  const long long ntl = (n + kJitTile - 1) / kJitTile;
  CUresult rc;
  int rows;
  if (m->stream && streaming) {
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
    long long want = (nll_waves() * slots + ntiles - 1) / ntiles;
    if (want < 1) want = 1;
    if (want > P) want = P;
    int pchunk = static_cast<int>((P + want - 1) / want);
    const int nchunks = (P + pchunk - 1) / pchunk;
    void* args[] = {&dp, &cp, &nn, &kc, &PP, &pchunk, &ntiles, &partial, &bad};
    if (ev_start) cudaEventRecord(ev_start, stream);
    rc = drv.launch(m->tile, static_cast<unsigned>(static_cast<long long>(ntiles) * nchunks), 1, 1, kJitThreads, 1, 1,
                    m->smem_cols * kJitTile * sizeof(double), reinterpret_cast<CUstream>(stream), args, nullptr);
    if (ev_stop) cudaEventRecord(ev_stop, stream);
    rows = ntiles;
    info.nchunks = nchunks;
    info.grid = ntiles * nchunks;
    info.cached = hoist_cols(hp);
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

// ---------------------------------------------------------------------------
// plan-specialised likelihood (kernels_device.cuh eval_plan_spec): the launch's term
// list (after the launch-constant rewrite) as compile-time constants of the tile kernel

namespace {

struct PlanModule {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;      // tile kernel
  CUfunction stream = nullptr;  // few-point streaming kernel (single-column single-sum plans)
  int occ = 1, stream_occ = 1;
};

// the few-point streaming kernel: one column (any plan shape) or up to three (products
// over several observables; kernels_device.cuh nll_stream_kernel NC > 1)
constexpr int kSpecStreamMaxCols = 3;
bool spec_has_stream(const DevPlan& d) { return d.ncols <= kSpecStreamMaxCols && d.nderived == 0; }
int spec_stream_stages(const DevPlan& d) { return d.ncols == 1 ? kJitStages : 2; }

std::string plan_spec_stream_name(const DevPlan& d, int ks) {
  return "&ffb::nll_stream_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(kJitE) + ", 2, " +
         std::to_string(ks) + ", ffb::PlanSpec, " + std::to_string(d.ncols) + ">";
}
std::map<std::tuple<int, std::string, int>, PlanModule> g_plan_mods;  // (device, source, mode)

int spec_mode(const DevPlan& d, int ks) { return ks + (d.simple ? 0 : 3) + (d.nderived > 0 ? 6 : 0); }

// the plan-specialised tile kernel's events per thread and minimum CTAs per SM
// (FFB_SPEC_TILE="E,MINB" for A/B builds; nll_scratch_bytes sizes for E >= 4)
struct SpecTile {
  int e = kJitE, minb = 2;
};
const SpecTile& spec_tile() {
  static const SpecTile t = [] {
    SpecTile v;
    if (const char* s = std::getenv("FFB_SPEC_TILE")) {
      int e = 0, b = 0;
      if (std::sscanf(s, "%d,%d", &e, &b) == 2 && (e == 4 || e == 8) && b >= 1 && b <= 4) {
        v.e = e;
        v.minb = b;
      }
    }
    return v;
  }();
  return t;
}

std::string plan_spec_kernel_name(const DevPlan& d, int ks) {
  return "&ffb::nll_kernel<" + std::to_string(kJitThreads) + ", " + std::to_string(spec_tile().e) + ", " +
         (d.ncols == 1 ? "true" : "false") + ", " + std::to_string(spec_tile().minb) + ", " +
         std::to_string(spec_mode(d, ks)) + ", ffb::PlanSpec>";
}

PlanModule* plan_module(const DevPlan& d, int ks) {
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string src = plan_spec_source(d);
  const auto key = std::make_tuple(dev, src + opts_key(), spec_mode(d, ks));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_plan_mods.find(key);
  if (it != g_plan_mods.end()) return it->second.mod ? &it->second : nullptr;
  PlanModule m;  // failures are cached too: no recompile per launch
  DriverApi& drv = driver();
  std::vector<std::string> names = {plan_spec_kernel_name(d, ks)};
  if (spec_has_stream(d)) names.push_back(plan_spec_stream_name(d, ks));
  std::vector<char> cubin;
  std::vector<std::string> lowered;
  std::string log;
  if (drv.ok && compile(src, names, &cubin, &lowered, &log)) {
    cudaFree(nullptr);
    if (drv.module_load(&m.mod, cubin.data()) == CUDA_SUCCESS &&
        drv.get_function(&m.fn, m.mod, lowered[0].c_str()) == CUDA_SUCCESS &&
        (names.size() < 2 || drv.get_function(&m.stream, m.mod, lowered[1].c_str()) == CUDA_SUCCESS)) {
      const int st = kJitThreads * spec_tile().e;
      drv.set_attribute(m.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                        kMaxCols * st * static_cast<int>(sizeof(double)));
      drv.occupancy(&m.occ, m.fn, kJitThreads, (d.ncols + d.ncached) * st * sizeof(double));
      if (m.occ < 1) m.occ = 1;
      if (m.stream) {
        const int ss = spec_stream_stages(d) * d.ncols * kJitTile * static_cast<int>(sizeof(double));
        drv.set_attribute(m.stream, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, ss);
        drv.occupancy(&m.stream_occ, m.stream, kJitThreads, ss);
        if (m.stream_occ < 1) m.stream_occ = 1;
      }
    } else {
      m.mod = nullptr;
    }
  }
  if (!m.mod) g_status = "likelihood: generic kernels (" + (drv.ok ? log.substr(0, 2000) : drv.why) + ")";
  auto& slot = g_plan_mods[key];
  slot = m;
  return slot.mod ? &slot : nullptr;
}

}  // namespace

std::string plan_spec_struct(const DevPlan& d) {
  std::ostringstream o;
  o << "#include \"plan.hpp\"\nnamespace ffb {\nstruct PlanSpec {\n"
       "  static constexpr bool kOn = true;\n"
    << "  static constexpr int nterms = " << d.nterms << ";\n"
    << "  static constexpr bool simple = " << (d.simple ? "true" : "false") << ";\n"
    << "  static constexpr int stride = " << d.stride << ";\n"
    << "  static constexpr DevTerm t[" << d.nterms << "] = {";
  for (int i = 0; i < d.nterms; ++i) {
    const DevTerm& t = d.t[i];
    o << (i ? ", " : "") << "{" << t.kind << ", " << t.col << ", " << t.order << ", " << t.flags << ", " << t.coff
      << "}";
  }
  o << "};\n  static constexpr int nderived = " << d.nderived << ";\n  static constexpr DevDerive dv["
    << (d.nderived > 0 ? d.nderived : 1) << "] = {";
  for (int i = 0; i < d.nderived; ++i) {
    const DevDerive& v = d.dv[i];
    // (the source row stays launch data, DevPlan::dv: not part of the build)
    o << (i ? ", " : "") << "{" << v.col << ", " << v.coff << ", " << v.kind << ", " << v.order << ", " << v.dst
      << ", 0}";
  }
  if (d.nderived == 0) o << "{0, 0, 0, 0, 0, 0}";
  o << "};\n};\n}  // namespace ffb\n";
  return o.str();
}

std::string plan_spec_source(const DevPlan& d) {
  // FFB_CONST_BANK: the exp / log polynomial constants as constant-bank DFMA operands
  // instead of 64-bit immediates materialised per use (A/B, profiles/r01_ab1: +0.2-2.3 %
  // on C2-C4, -0.5 % on C1)
  return "// generated by jit.cpp: the launch's term list for nll_kernel<..., PlanSpec>\n"
         "#define FFB_CONST_BANK 1\n#define FFB_NLL_ITEM_LOOP 1\n" +
         plan_spec_struct(d) + "#include \"kernels_device.cuh\"\n";
}

namespace {
std::atomic<double> g_spec_min{[] {
  if (std::getenv("FFB_NO_PLAN_SPEC")) return -1.0;
  const char* v = std::getenv("FFB_PLAN_SPEC_MIN");
  return v ? std::atof(v) : 5e7;
}()};
}  // namespace

double plan_spec_min_work(double v) {
  const double was = g_spec_min.load();
  if (v >= 0.0 || v == -1.0) g_spec_min.store(v);
  return was;
}

bool plan_spec_applies(const HostPlan& plan, const DevPlan& launch, long long n, int P) {
  const double min_work = g_spec_min.load();
  if (min_work < 0.0 || !jit_enabled() || !plan.programs.empty() || launch.nterms < 1) return false;
  // few-point launches of multi-column or product plans: the static tile kernel
  if (P <= kJitStreamMaxP && !spec_has_stream(launch)) return false;
  return static_cast<double>(n) * P >= min_work;
}

bool plan_spec_prepare(const DevPlan& launch, int ks) { return plan_module(launch, ks) != nullptr; }

bool plan_spec_compile_only(const DevPlan& launch, int ks, std::string* log) {
  std::vector<char> cubin;
  std::vector<std::string> low;
  std::vector<std::string> names = {plan_spec_kernel_name(launch, ks)};
  if (spec_has_stream(launch)) names.push_back(plan_spec_stream_name(launch, ks));
  return compile(plan_spec_source(launch), names, &cubin, &low, log);
}

NllLaunchInfo launch_nll_spec(const DevPlan& launch, const ColPtrs& cols, long long n, const double* d_consts, int P,
                              void* scratch, SumPair* d_out, unsigned long long* d_bad, cudaStream_t stream, int ks,
                              int waves, cudaEvent_t ev_start, cudaEvent_t ev_stop) {
  NllLaunchInfo info;
  if (P <= 0) return info;
  PlanModule* m = plan_module(launch, ks);
  if (!m) usage_error("internal: launch_nll_spec without a module");
  DriverApi& drv = driver();
  DevPlan dp = launch;
  ColPtrs cp = cols;
  long long nn = n;
  const double* kc = d_consts;
  int PP = P;
  SumPair* partial = static_cast<SumPair*>(scratch);
  unsigned long long* bad = d_bad;
  cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long) * P, stream);
  long long ntl = (n + kJitTile - 1) / kJitTile;
  if (ntl < 1) ntl = 1;
  int ntiles = static_cast<int>(ntl);
  bool aligned = true;
  for (int c = 0; c < launch.ncols; ++c) aligned = aligned && (reinterpret_cast<uintptr_t>(cols.c[c]) & 15) == 0;
  if (m->stream && P <= kJitStreamMaxP && aligned && std::getenv("FFB_NO_STREAM") == nullptr) {
    // few points: the persistent streaming kernel (kernels_device.cuh nll_stream_kernel)
    long long G = static_cast<long long>(device_sm_count()) * m->stream_occ;
    if (G > ntl) G = ntl;
    void* sargs[] = {&dp, &cp, &nn, &kc, &PP, &ntiles, &partial, &bad};
    if (ev_start) cudaEventRecord(ev_start, stream);
    const CUresult rc = drv.launch(m->stream, static_cast<unsigned>(G), 1, 1, kJitThreads, 1, 1,
                                   spec_stream_stages(launch) * launch.ncols * kJitTile * sizeof(double),
                                   reinterpret_cast<CUstream>(stream), sargs, nullptr);
    if (ev_stop) cudaEventRecord(ev_stop, stream);
    if (rc != CUDA_SUCCESS) numeric_error("cuLaunchKernel (plan-specialised likelihood) failed: " + std::to_string(rc));
    launch_reduce(partial, static_cast<int>(G), P, d_out, stream);
    info.threads = kJitThreads;
    info.events_per_thread = kJitE;
    info.tile = kJitTile;
    info.ntiles = ntiles;
    info.nchunks = 0;
    info.grid = static_cast<int>(G);
    info.launches = 2;
    info.jit = 2;
    return info;
  }
  // the static builds' grid rule (kernels.cu nll_shape): >= `waves` waves of resident CTAs
  const int stile = kJitThreads * spec_tile().e;
  ntl = (n + stile - 1) / stile;
  if (ntl < 1) ntl = 1;
  ntiles = static_cast<int>(ntl);
  const long long slots = static_cast<long long>(device_sm_count()) * m->occ;
  long long want = (waves * slots + ntiles - 1) / ntiles;
  if (want < 1) want = 1;
  if (want > P) want = P;
  int pchunk = static_cast<int>((P + want - 1) / want);
  const int nchunks = (P + pchunk - 1) / pchunk;
  void* args[] = {&dp, &cp, &nn, &kc, &PP, &pchunk, &ntiles, &partial, &bad};
  if (ev_start) cudaEventRecord(ev_start, stream);
  const long long grid = nll_grid(static_cast<long long>(ntiles) * nchunks, slots);
  const CUresult rc =
      drv.launch(m->fn, static_cast<unsigned>(grid), 1, 1, kJitThreads, 1, 1,
                 (launch.ncols + launch.ncached) * stile * sizeof(double),
                 reinterpret_cast<CUstream>(stream), args, nullptr);
  if (ev_stop) cudaEventRecord(ev_stop, stream);
  if (rc != CUDA_SUCCESS) numeric_error("cuLaunchKernel (plan-specialised likelihood) failed: " + std::to_string(rc));
  launch_reduce(partial, ntiles, P, d_out, stream);
  info.threads = kJitThreads;
  info.events_per_thread = spec_tile().e;
  info.tile = stile;
  info.ntiles = ntiles;
  info.nchunks = nchunks;
  info.grid = static_cast<int>(grid);
  info.launches = 2;
  info.jit = 2;
  return info;
}

}  // namespace ffb
