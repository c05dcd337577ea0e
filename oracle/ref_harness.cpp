// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// ctypes-friendly C shim over the *unmodified* reference engine (`ffit`,
// /root/reference/proj/src/*.cpp compiled by oracle/Makefile into
// oracle/_ref/libffit_ref.so).  The reference's own C ABI (include/ffit.h)
// can only build datasets from CSV files or its sampler; parity tests need
// in-memory columns, so this shim wraps the C++ API it documents:
//   Model::from_string              (proj/include/ffit/model.hpp:52-56)
//   DataSet(names, columns)         (proj/include/ffit/dataset.hpp:25)
//   nll / probabilities             (proj/include/ffit/eval.hpp:41-44, src/eval.cpp:165-192)
//   normalization                   (proj/include/ffit/eval.hpp:26, src/eval.cpp:71-86)
//   sample                          (proj/include/ffit/sampling.hpp, src/sampling.cpp:172-197)
//   fit_to                          (proj/include/ffit/fit.hpp:47, src/fit.cpp:86-251)
//   expr::compile / Program::eval   (proj/include/ffit/expr.hpp:128-135)
// Exported symbols are prefixed `ref_`; every reference symbol stays hidden
// (-fvisibility=hidden) so this library can share a process with the
// product's `ffit_*` exports.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ffit/eval.hpp"
#include "ffit/expr.hpp"
#include "ffit/fit.hpp"
#include "ffit/model.hpp"
#include "ffit/sampling.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ffit::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

ffit::EvalMode to_mode(int m) {
  switch (m) {
    case 0: return ffit::EvalMode::Scalar;
    case 1: return ffit::EvalMode::BatchPrecise;
    case 2: return ffit::EvalMode::BatchFast;
  }
  throw ffit::Error(ffit::ErrorCode::Usage, "bad mode");
}

// Neumaier sum of -log(p) over the reference's own per-event values: the
// compensated NLL SURVEY.md §8(c2) grades the GPU against.
void neumaier_nll(const std::vector<double>& p, double* value, long long* first_invalid) {
  double s = 0.0, c = 0.0;
  long long bad = -1;
  for (std::size_t i = 0; i < p.size(); ++i) {
    if (!(p[i] > 0.0) || !std::isfinite(p[i])) {
      bad = static_cast<long long>(i);
      break;
    }
    const double v = -std::log(p[i]);
    const double t = s + v;
    if (std::fabs(s) >= std::fabs(v)) c += (s - t) + v;
    else c += (v - t) + s;
    s = t;
  }
  *first_invalid = bad;
  *value = bad >= 0 ? std::numeric_limits<double>::infinity() : s + c;
}

}  // namespace

struct ref_model {
  std::unique_ptr<ffit::Model> m;
  std::string text;
};
struct ref_dataset {
  ffit::DataSet d;
};

REF_API const char* ref_last_error(void) { return g_err.c_str(); }

REF_API int ref_model_parse(const char* text, ref_model** out) {
  return guarded([&] {
    auto r = std::make_unique<ref_model>();
    r->m = ffit::Model::from_string(text);
    r->text = text;
    *out = r.release();
  });
}

REF_API void ref_model_free(ref_model* m) { delete m; }

REF_API int ref_set_param(ref_model* m, const char* name, double v) {
  return guarded([&] { m->m->graph.set_value(m->m->graph.id_of(name), v); });
}

REF_API int ref_get_param(ref_model* m, const char* name, double* v, double* err) {
  return guarded([&] {
    const ffit::Node& n = m->m->graph.node(m->m->graph.id_of(name));
    *v = n.value;
    if (err) *err = n.error;
  });
}

REF_API int ref_dataset_create(const char* name, const double* col, long long n,
                               ref_dataset** out) {
  return guarded([&] {
    std::vector<double> v(col, col + n);
    *out = new ref_dataset{ffit::DataSet({name}, {std::move(v)})};
  });
}

REF_API void ref_dataset_free(ref_dataset* d) { delete d; }

REF_API int ref_nll(ref_model* m, ref_dataset* d, int mode, double* value,
                    unsigned long long* n_eval, long long* first_invalid) {
  return guarded([&] {
    const ffit::NllValue v = ffit::nll(*m->m, d->d, to_mode(mode));
    *value = v.value;
    if (n_eval) *n_eval = v.n_evaluations;
    if (first_invalid) *first_invalid = v.first_invalid;
  });
}

REF_API int ref_nll_compensated(ref_model* m, ref_dataset* d, int mode, double* value,
                                long long* first_invalid) {
  return guarded([&] {
    std::vector<double> p(d->d.n_rows());
    ffit::probabilities(*m->m, d->d, to_mode(mode), p);
    neumaier_nll(p, value, first_invalid);
  });
}

REF_API int ref_probabilities(ref_model* m, ref_dataset* d, int mode, double* out) {
  return guarded([&] {
    ffit::probabilities(*m->m, d->d, to_mode(mode), std::span<double>(out, d->d.n_rows()));
  });
}

REF_API int ref_normalization(ref_model* m, double* out) {
  return guarded([&] {
    *out = ffit::normalization(m->m->pdf, m->m->obs_lower(), m->m->obs_upper(), m->m->graph);
  });
}

REF_API int ref_eval_unnorm(ref_model* m, const double* xs, long long n, double* out) {
  return guarded([&] {
    for (long long i = 0; i < n; ++i) out[i] = m->m->pdf.eval_unnorm(xs[i], m->m->graph);
  });
}

REF_API int ref_sample(ref_model* m, long long n, unsigned long long seed, double* out,
                       double* efficiency) {
  return guarded([&] {
    ffit::SampleStats st;
    const ffit::DataSet ds = ffit::sample(*m->m, static_cast<std::size_t>(n), seed, &st);
    const auto col = ds.column(m->m->obs_name());
    std::copy(col.begin(), col.end(), out);
    if (efficiency) *efficiency = st.proposed == 0 ? -1.0 : st.efficiency();
  });
}

// Reference Rng stream (xoshiro256++ seeded by splitmix64), to pin restatements.
REF_API void ref_rng_uniform(unsigned long long seed, long long n, double* out) {
  ffit::Rng r(seed);
  for (long long i = 0; i < n; ++i) out[i] = r.uniform();
}

REF_API void ref_rng_gauss(unsigned long long seed, long long n, double* out) {
  ffit::Rng r(seed);
  for (long long i = 0; i < n; ++i) out[i] = r.gauss();
}

REF_API int ref_fit(ref_model* m, ref_dataset* d, int mode, double tol, long max_iter,
                    int* converged, double* nll_min, unsigned long long* calls,
                    int* unc_valid) {
  return guarded([&] {
    ffit::FitOptions o;
    o.mode = to_mode(mode);
    if (tol > 0) o.tolerance = tol;
    if (max_iter > 0) o.max_iterations = static_cast<int>(max_iter);
    const ffit::FitResult r = ffit::fit_to(*m->m, d->d, o);
    *converged = r.converged ? 1 : 0;
    *nll_min = r.nll_min;
    *calls = r.n_nll_calls;
    *unc_valid = r.uncertainties_valid ? 1 : 0;
  });
}

// CPU baseline leg (bench.py --impl reference): P parameter points split
// across `threads` host threads, each with its own Model over the shared
// immutable DataSet (allowed by SPEC.md:166,480).  points is P x nnames,
// row-major; values[p] receives the reference nll() for point p.
REF_API int ref_nll_points_threaded(const char* text, ref_dataset* d, int mode,
                                    const char* const* names, int nnames,
                                    const double* points, int P, int threads,
                                    double* values) {
  return guarded([&] {
    std::atomic<int> next{0};
    std::vector<std::string> errs(threads);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          auto model = ffit::Model::from_string(text);
          std::vector<ffit::NodeId> ids;
          for (int k = 0; k < nnames; ++k) ids.push_back(model->graph.id_of(names[k]));
          for (int p = next++; p < P; p = next++) {
            for (int k = 0; k < nnames; ++k) {
              model->graph.set_value(ids[k], points[static_cast<std::size_t>(p) * nnames + k]);
            }
            values[p] = ffit::nll(*model, d->d, to_mode(mode)).value;
          }
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (const auto& e : errs) {
      if (!e.empty()) throw ffit::Error(ffit::ErrorCode::Numeric, e);
    }
  });
}

// One formula over `nvars` variables: compile, then evaluate the scalar program at `npts`
// rows of values (row-major npts x nvars).  Errors carry the reference's messages.
REF_API int ref_expr_eval(const char* text, const char* const* vars, int nvars, const double* values,
                          int npts, double* out) {
  return guarded([&] {
    std::vector<std::string> names(vars, vars + nvars);
    const ffit::expr::Program prog = ffit::expr::compile(std::string(text), names);
    for (int i = 0; i < npts; ++i) {
      out[i] = prog.eval(std::span<const double>(values + static_cast<std::size_t>(i) * nvars,
                                                 static_cast<std::size_t>(nvars)));
    }
  });
}
