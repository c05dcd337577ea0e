// extern "C" boundary (include/ffit_b200.h).  Same status-code / ownership /
// thread-local-error contract as the reference (proj/src/capi.cpp:28-50).
#include "../../include/ffit_b200.h"
#include "shard.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <charconv>
#include <fstream>
#include <limits>
#include <memory>
#include <sstream>
#include <string>

#include "engine.hpp"
#include "fit.hpp"
#include "jit.hpp"
#include "sampler.hpp"
#include "soa_io.hpp"

#define FFB_API extern "C" __attribute__((visibility("default")))

struct ffit_model {
  std::unique_ptr<ffb::Model> m;
  std::unique_ptr<ffb::Engine> engine;
};

struct ffit_dataset {
  std::shared_ptr<ffb::DeviceDataset> d;
};

struct ffit_fit_result {
  ffb::FitResult r;
};

struct ffcu_shard_group {
  ffit_model* m = nullptr;  // the caller's model (parameters, write-back of fits)
  std::unique_ptr<ffb::ShardGroup> g;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FFIT_OK;
  } catch (const ffb::Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FFIT_ERR_NUMERIC;
  }
}

void require(const void* p, const char* what) {
  if (!p) ffb::usage_error(std::string(what) + " must not be null");
}

// Every reference mode runs the fused sm_100a kernel.  The reference defines Scalar as
// bitwise equal to BatchPrecise (proj/src/eval.cpp:96-117 vs 119-163, pinned by
// proj/tests/test_eval.cpp:113-157), so FFIT_MODE_SCALAR returns the GPU's Precise result
// bit for bit; the reference CLI's `bench` / `parity` (proj/tools/ffit_main.cpp:177,
// 188-189, 216-217) compare Scalar against the batch modes and find 0 deviation.
void require_gpu_mode(ffit_mode mode) {
  switch (mode) {
    case FFIT_MODE_SCALAR:
    case FFIT_MODE_BATCH_PRECISE:
    case FFIT_MODE_BATCH_FAST:
    case FFIT_MODE_GPU:
      return;
  }
  ffb::usage_error("unknown evaluation mode");
}

ffb::Engine& engine(ffit_model* m) {
  if (!m->engine) m->engine = std::make_unique<ffb::Engine>(*m->m);
  return *m->engine;
}

std::vector<double> point_or_current(const ffb::Model& m, const double* point) {
  if (point) return std::vector<double>(point, point + m.params.size());
  return m.theta();
}

std::unique_ptr<ffit_model> make_model(std::unique_ptr<ffb::Model> mm) {
  auto m = std::make_unique<ffit_model>();
  m->m = std::move(mm);
  m->engine = std::make_unique<ffb::Engine>(*m->m);  // compiles the plan: fail early
  return m;
}

// CSV cells exactly as the reference reads them (proj/src/dataset.cpp:11-45): split on
// ',', trailing ' ' / '\r' and leading ' ' trimmed (tabs are kept), each cell parsed by
// std::from_chars over the whole cell (locale-independent; no leading '+', no hex).
std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> out;
  std::size_t start = 0;
  while (true) {
    const std::size_t comma = line.find(',', start);
    out.push_back(line.substr(start, comma == std::string::npos ? std::string::npos : comma - start));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  for (auto& f : out) {
    while (!f.empty() && (f.back() == '\r' || f.back() == ' ')) f.pop_back();
    std::size_t i = 0;
    while (i < f.size() && f[i] == ' ') ++i;
    f.erase(0, i);
  }
  return out;
}

double parse_cell(const std::string& cell, std::size_t row, const std::string& col) {
  double v = 0.0;
  const char* first = cell.data();
  const char* last = first + cell.size();
  const auto [ptr, ec] = std::from_chars(first, last, v);
  if (ec != std::errc() || ptr != last) {
    ffb::data_error("unparsable numeric cell at row " + std::to_string(row) + ", column '" + col + "': '" + cell +
                    "'");
  }
  return v;
}

}  // namespace

FFB_API const char* ffit_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// models

FFB_API int ffit_model_load(const char* path, ffit_model** out) {
  return guarded([&] {
    require(path, "path");
    require(out, "out");
    std::ifstream in(path);
    if (!in) ffb::data_error(std::string("cannot open model file: ") + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    *out = make_model(ffb::Model::parse(buf.str(), path)).release();
  });
}

FFB_API int ffit_model_parse(const char* text, ffit_model** out) {
  return guarded([&] {
    require(text, "text");
    require(out, "out");
    *out = make_model(ffb::Model::parse(text)).release();
  });
}

FFB_API void ffit_model_free(ffit_model* m) { delete m; }

FFB_API const char* ffit_model_observable(const ffit_model* m) {
  return m->m->observables[0].name.c_str();
}

FFB_API int ffit_model_observable_range(const ffit_model* m, double* lo, double* hi) {
  return guarded([&] {
    require(m, "model");
    if (lo) *lo = m->m->observables[0].lo;
    if (hi) *hi = m->m->observables[0].hi;
  });
}

FFB_API int ffit_model_param_count(const ffit_model* m) {
  return static_cast<int>(m->m->params.size());
}

FFB_API const char* ffit_model_param_name(const ffit_model* m, int i) {
  if (i < 0 || i >= static_cast<int>(m->m->params.size())) return nullptr;
  return m->m->params[i].name.c_str();
}

FFB_API int ffit_model_param_is_constant(const ffit_model* m, const char* name, int* constant) {
  return guarded([&] {
    require(m, "model");
    require(constant, "constant");
    const int id = name ? m->m->param_index(name) : -1;
    if (id < 0) ffb::usage_error("unknown parameter: " + std::string(name ? name : "(null)"));
    *constant = m->m->params[id].constant ? 1 : 0;
  });
}

FFB_API int ffit_model_get_param(const ffit_model* m, const char* name, double* value,
                                 double* uncertainty) {
  return guarded([&] {
    require(m, "model");
    const int id = name ? m->m->param_index(name) : -1;
    if (id < 0) ffb::usage_error("unknown parameter: " + std::string(name ? name : "(null)"));
    if (value) *value = m->m->params[id].value;
    if (uncertainty) *uncertainty = m->m->params[id].error;
  });
}

FFB_API int ffit_model_set_param(ffit_model* m, const char* name, double value) {
  return guarded([&] {
    require(m, "model");
    const int id = name ? m->m->param_index(name) : -1;
    if (id < 0) ffb::usage_error("unknown parameter: " + std::string(name ? name : "(null)"));
    m->m->set_value(id, value);
  });
}

// ---------------------------------------------------------------------------
// datasets

// DataSet::from_csv (proj/src/dataset.cpp:61-121): header line, rows outside an
// observable's range dropped and counted; then one upload to HBM.
FFB_API int ffit_dataset_read_csv(const ffit_model* m, const char* path, ffit_dataset** out,
                                  long* dropped) {
  return guarded([&] {
    require(m, "model");
    require(path, "path");
    require(out, "out");
    std::ifstream in(path);
    if (!in) ffb::data_error(std::string("cannot open file: ") + path);
    std::string line;
    if (!std::getline(in, line)) ffb::data_error(std::string("empty file: ") + path);
    const std::vector<std::string> header = split_csv(line);
    const auto& obs = m->m->observables;
    std::vector<std::size_t> idx(obs.size());
    for (std::size_t s = 0; s < obs.size(); ++s) {
      bool found = false;
      for (std::size_t h = 0; h < header.size(); ++h) {
        if (header[h] == obs[s].name) {
          idx[s] = h;
          found = true;
          break;
        }
      }
      if (!found) ffb::data_error("missing column '" + obs[s].name + "' in " + path);
    }
    std::vector<std::vector<double>> cols(obs.size());
    std::vector<double> parsed(obs.size());
    long nd = 0;
    std::size_t row = 0;
    while (std::getline(in, line)) {
      ++row;
      if (line.empty() || line == "\r") continue;
      const std::vector<std::string> f = split_csv(line);
      if (f.size() < header.size()) {
        ffb::data_error("row " + std::to_string(row) + " has " + std::to_string(f.size()) +
                        " fields, header has " + std::to_string(header.size()));
      }
      bool in_range = true;
      for (std::size_t s = 0; s < obs.size(); ++s) {
        const double v = parse_cell(f[idx[s]], row, obs[s].name);
        parsed[s] = v;
        if (!(v >= obs[s].lo && v <= obs[s].hi)) in_range = false;
      }
      if (!in_range) {
        ++nd;
        continue;
      }
      for (std::size_t s = 0; s < obs.size(); ++s) cols[s].push_back(parsed[s]);
    }
    std::vector<std::string> names;
    std::vector<const double*> ptrs;
    for (std::size_t s = 0; s < obs.size(); ++s) {
      names.push_back(obs[s].name);
      ptrs.push_back(cols[s].data());
    }
    auto d = ffb::DeviceDataset::upload(names, ptrs, static_cast<long long>(cols[0].size()));
    if (dropped) *dropped = nd;
    *out = new ffit_dataset{std::move(d)};
  });
}

// DataSet::write_csv (proj/src/dataset.cpp:123-146): %.17g round-trip.
FFB_API int ffit_dataset_write_csv(const ffit_dataset* ds, const char* path) {
  return guarded([&] {
    require(ds, "dataset");
    require(path, "path");
    const auto& d = *ds->d;
    std::vector<std::vector<double>> cols(d.cols.size(), std::vector<double>(static_cast<std::size_t>(d.n)));
    for (std::size_t c = 0; c < cols.size(); ++c) d.download(static_cast<int>(c), cols[c].data());
    std::FILE* f = std::fopen(path, "w");
    if (!f) ffb::data_error(std::string("cannot write file: ") + path);
    for (std::size_t c = 0; c < d.names.size(); ++c) std::fprintf(f, c ? ",%s" : "%s", d.names[c].c_str());
    std::fputc('\n', f);
    for (long long i = 0; i < d.n; ++i) {
      for (std::size_t c = 0; c < cols.size(); ++c) std::fprintf(f, c ? ",%.17g" : "%.17g", cols[c][i]);
      std::fputc('\n', f);
    }
    if (std::fclose(f) != 0) ffb::data_error(std::string("write failed: ") + path);
  });
}

FFB_API long ffit_dataset_rows(const ffit_dataset* ds) { return static_cast<long>(ds->d->n); }

FFB_API void ffit_dataset_free(ffit_dataset* ds) { delete ds; }

FFB_API int ffit_sample(ffit_model* m, long n, unsigned long long seed, ffit_dataset** out,
                        double* efficiency) {
  return guarded([&] {
    require(m, "model");
    require(out, "out");
    if (n < 0) ffb::usage_error("sample size must be >= 0");
    ffb::SampleStats st;
    const auto cols = ffb::sample(*m->m, n, seed, &st);
    std::vector<std::string> names;
    std::vector<const double*> ptrs;
    for (std::size_t s = 0; s < cols.size(); ++s) {
      names.push_back(m->m->observables[s].name);
      ptrs.push_back(cols[s].data());
    }
    auto d = ffb::DeviceDataset::upload(names, ptrs, n);
    if (efficiency) {
      *efficiency = st.proposed == 0 ? -1.0
                                     : static_cast<double>(st.accepted) / static_cast<double>(st.proposed);
    }
    *out = new ffit_dataset{std::move(d)};
  });
}

FFB_API int ffcu_sample_host(ffit_model* m, long long n, unsigned long long seed, double* const* cols,
                             double* efficiency) {
  return guarded([&] {
    require(m, "model");
    require(cols, "cols");
    ffb::SampleStats st;
    const auto out = ffb::sample(*m->m, n, seed, &st);
    for (std::size_t s = 0; s < out.size(); ++s) {
      require(cols[s], "cols[i]");
      std::memcpy(cols[s], out[s].data(), static_cast<std::size_t>(n) * sizeof(double));
    }
    if (efficiency) {
      *efficiency = st.proposed == 0 ? -1.0
                                     : static_cast<double>(st.accepted) / static_cast<double>(st.proposed);
    }
  });
}

// ---------------------------------------------------------------------------
// evaluation

FFB_API int ffit_nll(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double* value,
                     unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require_gpu_mode(mode);
    const std::vector<double> th = m->m->theta();
    m->m->check_params(m->m->root, th.data());  // require_valid_params, proj/src/eval.cpp:120
    const ffb::NllResult r = engine(m).nll_points(*ds->d, th.data(), 1);
    if (value) *value = r.value[0];
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffit_probabilities(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double* out) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(out, "out");
    require_gpu_mode(mode);
    const std::vector<double> th = m->m->theta();
    engine(m).probabilities(*ds->d, th.data(), out, false);
  });
}

FFB_API int ffcu_probabilities_at(ffit_model* m, const ffit_dataset* ds, const double* point,
                                  double* out) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(out, "out");
    const std::vector<double> th = point_or_current(*m->m, point);
    engine(m).probabilities(*ds->d, th.data(), out, false);
  });
}

FFB_API int ffcu_nll_points(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                            double* values, long long* first_invalid,
                            unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(values, "values");
    if (P < 0) ffb::usage_error("P must be >= 0");
    if (P == 0) {
      if (n_evaluations) *n_evaluations = 0;
      return;
    }
    const ffb::NllResult r = engine(m).nll_points(*ds->d, points, P);
    for (int p = 0; p < P; ++p) {
      values[p] = r.value[p];
      if (first_invalid) first_invalid[p] = r.first_invalid[p];
    }
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_nll_points_partial(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                                    double* sc, long long* first_invalid,
                                    unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(sc, "sc");
    if (P < 0) ffb::usage_error("P must be >= 0");
    if (P == 0) return;
    const ffb::NllResult r = engine(m).nll_points(*ds->d, points, P);
    for (int p = 0; p < P; ++p) {
      sc[2 * p] = r.pairs[p].s;
      sc[2 * p + 1] = r.pairs[p].c;
      if (first_invalid) first_invalid[p] = r.first_invalid[p];
    }
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_nll_points_device(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                                   double* d_sc, unsigned long long* d_bad, void* stream,
                                   unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(d_sc, "d_sc");
    require(d_bad, "d_bad");
    const int k = engine(m).nll_points_device(*ds->d, points, P, reinterpret_cast<ffb::SumPair*>(d_sc),
                                              d_bad, static_cast<cudaStream_t>(stream));
    if (n_evaluations) *n_evaluations = static_cast<unsigned long long>(k);
  });
}

FFB_API int ffcu_nll_points_device_upload(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                                          double* d_sc, unsigned long long* d_bad, void* stream, void* upload_stream,
                                          unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(d_sc, "d_sc");
    require(d_bad, "d_bad");
    const int k = engine(m).nll_points_device(*ds->d, points, P, reinterpret_cast<ffb::SumPair*>(d_sc), d_bad,
                                              static_cast<cudaStream_t>(stream),
                                              static_cast<cudaStream_t>(upload_stream));
    if (n_evaluations) *n_evaluations = static_cast<unsigned long long>(k);
  });
}

FFB_API int ffcu_grad_slot_count(ffit_model* m, int* nslots) {
  return guarded([&] {
    require(m, "model");
    require(nslots, "nslots");
    const ffb::GradPlan& gp = engine(m).grad_plan();
    if (!gp.ok) ffb::usage_error("analytic gradient unavailable for this model: " + gp.why);
    *nslots = gp.dev.nslots;
  });
}

FFB_API int ffcu_nll_grad(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                          double* values, double* grads, long long* first_invalid,
                          unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(values, "values");
    require(grads, "grads");
    if (P < 0) ffb::usage_error("P must be >= 0");
    if (P == 0) {
      if (n_evaluations) *n_evaluations = 0;
      return;
    }
    const ffb::NllGradResult r = engine(m).nll_grad_points(*ds->d, points, P);
    const std::size_t npar = m->m->params.size();
    for (int p = 0; p < P; ++p) {
      values[p] = r.value[p];
      if (first_invalid) first_invalid[p] = r.first_invalid[p];
    }
    std::copy(r.grad.begin(), r.grad.begin() + static_cast<std::ptrdiff_t>(P * npar), grads);
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_nll_grad_partial(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                                  double* sc, long long* first_invalid, unsigned long long* n_evaluations) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(points, "points");
    require(sc, "sc");
    if (P < 0) ffb::usage_error("P must be >= 0");
    if (P == 0) return;
    const ffb::NllGradResult r = engine(m).nll_grad_points(*ds->d, points, P);
    for (std::size_t k = 0; k < r.slots.size(); ++k) {
      sc[2 * k] = r.slots[k].s;
      sc[2 * k + 1] = r.slots[k].c;
    }
    if (first_invalid) {
      for (int p = 0; p < P; ++p) first_invalid[p] = r.first_invalid[p];
    }
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_nll_grad_finish(ffit_model* m, const double* points, int P, const double* slot_sums,
                                 double n_events, double* values, double* grads) {
  return guarded([&] {
    require(m, "model");
    require(points, "points");
    require(slot_sums, "slot_sums");
    require(values, "values");
    require(grads, "grads");
    if (P < 0) ffb::usage_error("P must be >= 0");
    engine(m).grad_finish(points, P, slot_sums, n_events, values, grads);
  });
}

FFB_API int ffcu_combine_pairs_device(const double* d_in, int R, int P, double* d_out, void* stream) {
  return guarded([&] {
    require(d_in, "d_in");
    require(d_out, "d_out");
    ffb::count_launches(ffb::launch_combine_ranks(reinterpret_cast<const ffb::SumPair*>(d_in), R, P,
                                                  reinterpret_cast<ffb::SumPair*>(d_out),
                                                  static_cast<cudaStream_t>(stream)));
    ffb::cuda_check(cudaGetLastError(), "combine_ranks");
  });
}

FFB_API int ffcu_combine_shards_device(const double* d_in, int R, int rows, int P, const long long* d_offsets,
                                       double* d_out, unsigned long long* d_bad, void* stream) {
  return guarded([&] {
    require(d_in, "d_in");
    require(d_offsets, "d_offsets");
    require(d_out, "d_out");
    require(d_bad, "d_bad");
    if (R < 1 || rows < 0 || P < 0) ffb::usage_error("combine_shards: bad sizes");
    ffb::count_launches(ffb::launch_combine_shards(d_in, R, rows, P, d_offsets, reinterpret_cast<ffb::SumPair*>(d_out),
                                                   d_bad, static_cast<cudaStream_t>(stream)));
    ffb::cuda_check(cudaGetLastError(), "combine_shards");
  });
}

FFB_API int ffcu_extended_terms(const ffit_model* m, const double* points, int P, double n_events,
                                double* out) {
  return guarded([&] {
    require(m, "model");
    require(points, "points");
    require(out, "out");
    const std::size_t npar = m->m->params.size();
    for (int p = 0; p < P; ++p) out[p] = m->m->extended_term(points + p * npar, n_events);
  });
}

FFB_API int ffcu_eval_batch(ffit_model* m, const char* pdf, const ffit_dataset* ds, double* out) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(out, "out");
    const int id = pdf ? m->m->pdf_index(pdf) : m->m->root;
    if (id < 0) ffb::usage_error(std::string("unknown pdf: ") + pdf);
    const std::vector<double> th = m->m->theta();
    engine(m).eval_batch(id, *ds->d, th.data(), out, false);
  });
}

FFB_API int ffcu_eval_batch_device(ffit_model* m, const char* pdf, const ffit_dataset* ds,
                                   double* d_out, void* stream) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(d_out, "d_out");
    const int id = pdf ? m->m->pdf_index(pdf) : m->m->root;
    if (id < 0) ffb::usage_error(std::string("unknown pdf: ") + pdf);
    const std::vector<double> th = m->m->theta();
    engine(m).eval_batch(id, *ds->d, th.data(), d_out, true, static_cast<cudaStream_t>(stream));
  });
}

FFB_API int ffcu_normalization(const ffit_model* m, const char* pdf, const double* point, double* out) {
  return guarded([&] {
    require(m, "model");
    require(out, "out");
    const int id = pdf ? m->m->pdf_index(pdf) : m->m->root;
    if (id < 0) ffb::usage_error(std::string("unknown pdf: ") + pdf);
    const std::vector<double> th = point_or_current(*m->m, point);
    m->m->check_params(id, th.data());
    *out = m->m->normalization(id, th.data());
  });
}

FFB_API int ffcu_model_set_device_normalization(ffit_model* m, int on) {
  return guarded([&] {
    require(m, "model");
    m->engine->set_device_normalization(on != 0);
  });
}

FFB_API int ffcu_model_device_normalization(const ffit_model* m) {
  return m && m->engine && m->engine->device_normalization() ? 1 : 0;
}

FFB_API int ffcu_device_normalization(ffit_model* m, const char* pdf, const double* points, int P, double* out) {
  return guarded([&] {
    require(m, "model");
    require(out, "out");
    if (P < 0) ffb::usage_error("negative point count");
    const int id = pdf ? m->m->pdf_index(pdf) : m->m->root;
    if (id < 0) ffb::usage_error(std::string("unknown pdf: ") + pdf);
    if (P == 0) return;
    std::vector<double> own;
    if (!points) {
      if (P != 1) ffb::usage_error("points == NULL needs P == 1 (the model's current values)");
      own = m->m->theta();
      points = own.data();
    }
    std::vector<double> res(P);  // out stays untouched on failure
    m->engine->device_normalization_of(id, points, P, res.data());
    std::copy(res.begin(), res.end(), out);
  });
}

FFB_API unsigned long long ffcu_device_normalization_launches(const ffit_model* m) {
  return m && m->engine ? m->engine->device_norm_launches() : 0ull;
}

FFB_API int ffcu_plan_info(const ffit_model* m, int* nterms, int* ncols, int* stride) {
  return guarded([&] {
    require(m, "model");
    const ffb::DevPlan& p = m->engine->likelihood_plan().dev;
    if (nterms) *nterms = p.nterms;
    if (ncols) *ncols = p.ncols;
    if (stride) *stride = p.stride;
  });
}

FFB_API int ffcu_plan_term(const ffit_model* m, int i, int* kind, int* col, int* order, int* flags,
                           int* coff) {
  return guarded([&] {
    require(m, "model");
    const ffb::DevPlan& p = m->engine->likelihood_plan().dev;
    if (i < 0 || i >= p.nterms) ffb::usage_error("term index out of range");
    if (kind) *kind = p.t[i].kind;
    if (col) *col = p.t[i].col;
    if (order) *order = p.t[i].order;
    if (flags) *flags = p.t[i].flags;
    if (coff) *coff = p.t[i].coff;
  });
}

FFB_API int ffcu_point_constants(const ffit_model* m, const double* point, double* row) {
  return guarded([&] {
    require(m, "model");
    require(row, "row");
    const std::vector<double> th = point_or_current(*m->m, point);
    ffb::build_constants(m->engine->likelihood_plan(), *m->m, th.data(), row);
  });
}

FFB_API int ffcu_coef_derivatives(const ffit_model* m, const double* point, int param, double* out) {
  return guarded([&] {
    require(m, "model");
    require(out, "out");
    if (param < 0 || param >= static_cast<int>(m->m->params.size())) ffb::usage_error("parameter index out of range");
    const std::vector<double> th = point_or_current(*m->m, point);
    const ffb::HostPlan& plan = m->engine->likelihood_plan();
    m->m->check_params(plan.pdf, th.data());
    const std::vector<double> d = ffb::coef_derivatives(plan, *m->m, th.data(), param, 1.0);
    std::copy(d.begin(), d.end(), out);
  });
}

FFB_API int ffcu_expr_eval(const char* text, const char* const* vars, int nvars, const double* values, int npts,
                           double* out) {
  return guarded([&] {
    require(text, "text");
    if (nvars < 0 || npts < 0) ffb::usage_error("nvars and npts must be >= 0");
    if (nvars > 0) require(vars, "vars");
    if (npts > 0) {
      require(values, "values");
      require(out, "out");
    }
    std::vector<std::string> names;
    for (int i = 0; i < nvars; ++i) names.emplace_back(vars[i]);
    const ffb::ExprProgram prog = ffb::compile_expression(text, names);
    for (int i = 0; i < npts; ++i) out[i] = prog.eval(values + static_cast<std::size_t>(i) * nvars);
  });
}

FFB_API int ffcu_expression_jit(int enable) {
  const int was = ffb::jit_enabled() ? 1 : 0;
  if (enable >= 0) ffb::jit_enable(enable != 0);
  return was;
}

FFB_API const char* ffcu_expression_jit_status(void) {
  thread_local std::string s;
  s = ffb::jit_status();
  return s.c_str();
}

FFB_API int ffcu_expression_jit_source(const ffit_model* m, int compile, char* buf, int cap) {
  return guarded([&] {
    require(m, "model");
    const ffb::HostPlan& plan = m->engine->likelihood_plan();
    if (plan.programs.empty()) ffb::usage_error("the model has no Expression pdf");
    const std::string src = ffb::jit_expression_source(plan);
    std::string text = src;
    if (compile) {
      std::string log;
      if (!ffb::jit_compile_only(plan, &log)) {
        ffb::numeric_error("NVRTC compile of the formula-specialised kernels failed: " + log.substr(0, 4000));
      }
    }
    if (buf && cap > 0) {
      const std::size_t k = std::min<std::size_t>(text.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, text.data(), k);
      buf[k] = '\0';
    }
  });
}

FFB_API int ffcu_expression_jit_source_points(ffit_model* m, const double* points, int P, int compile, char* buf,
                                              int cap) {
  return guarded([&] {
    require(m, "model");
    require(points, "points");
    const ffb::HostPlan& plan = engine(m).likelihood_plan();
    if (plan.programs.empty()) ffb::usage_error("the model has no Expression pdf");
    const std::size_t npar = m->m->params.size();
    std::vector<double> rows(static_cast<std::size_t>(P > 0 ? P : 0) * plan.dev.stride);
    for (int p = 0; p < P; ++p) {
      ffb::build_constants(plan, *m->m, points + p * npar, rows.data() + static_cast<std::size_t>(p) * plan.dev.stride,
                           std::ldexp(1.0, ffb::kPScaleLog2));
    }
    const ffb::ExprHoist hoist = ffb::analyse_expr_hoist(plan, rows.data(), P);
    const std::string text = ffb::jit_expression_source(plan, &hoist);
    if (compile) {
      std::string log;
      if (!ffb::jit_compile_only(plan, &log, &hoist)) {
        ffb::numeric_error("NVRTC compile of the formula-specialised kernels failed: " + log.substr(0, 4000));
      }
    }
    if (buf && cap > 0) {
      const std::size_t k = std::min<std::size_t>(text.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, text.data(), k);
      buf[k] = '\0';
    }
  });
}

FFB_API int ffcu_last_launch_jit(const ffit_model* m) { return m && m->engine ? m->engine->last_launch().jit : 0; }

FFB_API double ffcu_plan_spec_min_work(double v) { return ffb::plan_spec_min_work(v); }

FFB_API int ffcu_plan_spec_source(ffit_model* m, const double* points, int P, int compile, char* buf, int cap) {
  return guarded([&] {
    require(m, "model");
    const ffb::HostPlan& plan = engine(m).likelihood_plan();
    if (!plan.programs.empty()) ffb::usage_error("models with Expression pdfs take the formula-specialised build");
    ffb::DevPlan lp = plan.dev;
    std::vector<double> rows;
    if (points && P > 0) {  // the launch-constant rewrite these points would get
      const std::size_t npar = m->m->params.size();
      rows.resize(static_cast<std::size_t>(P) * plan.dev.stride);
      for (int p = 0; p < P; ++p) {
        ffb::build_constants(plan, *m->m, points + p * npar, rows.data() + static_cast<std::size_t>(p) * plan.dev.stride,
                             std::ldexp(1.0, ffb::kPScaleLog2));
      }
      ffb::cache_launch_constants(lp, rows.data(), P);
    }
    const std::string text = ffb::plan_spec_source(lp);
    if (compile) {
      const int ks = rows.empty() ? 2 : ffb::plan_kind_set(lp, rows.data(), P);
      std::string log;
      if (!ffb::plan_spec_compile_only(lp, ks, &log)) {
        ffb::numeric_error("NVRTC compile of the plan-specialised likelihood failed: " + log.substr(0, 4000));
      }
    }
    if (buf && cap > 0) {
      const std::size_t k = std::min<std::size_t>(text.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, text.data(), k);
      buf[k] = '\0';
    }
  });
}

FFB_API int ffcu_grad_spec_source(ffit_model* m, int compile_ks, char* buf, int cap) {
  return guarded([&] {
    require(m, "model");
    const ffb::GradPlan& gp = engine(m).grad_plan();
    if (!gp.ok) ffb::usage_error("analytic gradient unavailable for this model: " + gp.why);
    const ffb::HostPlan& plan = m->engine->likelihood_plan();
    if (compile_ks >= 0) {
      std::string log;
      if (!ffb::grad_spec_compile_only(plan, gp, compile_ks, &log)) {
        ffb::numeric_error("NVRTC compile of the plan-specialised gradient pass failed: " + log.substr(0, 4000));
      }
    }
    const std::string text = ffb::grad_spec_text(plan, gp);
    if (buf && cap > 0) {
      const std::size_t k = std::min<std::size_t>(text.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, text.data(), k);
      buf[k] = '\0';
    }
  });
}

FFB_API int ffcu_last_grad_jit(ffit_model* m) { return m && engine(m).last_grad_jit() ? 1 : 0; }

FFB_API int ffcu_model_pdf_count(const ffit_model* m) { return static_cast<int>(m->m->pdfs.size()); }

FFB_API const char* ffcu_model_pdf_name(const ffit_model* m, int i) {
  if (i < 0 || i >= static_cast<int>(m->m->pdfs.size())) return nullptr;
  return m->m->pdfs[i].name.c_str();
}

FFB_API int ffcu_model_observable_count(const ffit_model* m) {
  return static_cast<int>(m->m->observables.size());
}

FFB_API const char* ffcu_model_observable_name(const ffit_model* m, int i) {
  if (i < 0 || i >= static_cast<int>(m->m->observables.size())) return nullptr;
  return m->m->observables[i].name.c_str();
}

// ---------------------------------------------------------------------------
// device datasets

FFB_API int ffcu_dataset_from_host(const char* const* names, const double* const* cols, int ncols,
                                   long long n, ffit_dataset** out) {
  return guarded([&] {
    require(names, "names");
    require(out, "out");
    if (ncols <= 0) ffb::usage_error("a dataset needs at least one column");
    if (n > 0) require(cols, "cols");
    std::vector<std::string> nm;
    std::vector<const double*> c;
    for (int i = 0; i < ncols; ++i) {
      require(names[i], "names[i]");
      nm.push_back(names[i]);
      c.push_back(n > 0 ? cols[i] : nullptr);
    }
    *out = new ffit_dataset{ffb::DeviceDataset::upload(nm, c, n)};
  });
}

FFB_API int ffcu_soa_write(const char* path, const char* const* names, const double* const* cols, int ncols,
                           long long n) {
  return guarded([&] {
    require(path, "path");
    require(names, "names");
    if (ncols <= 0) ffb::usage_error("a dataset needs at least one column");
    if (n > 0) require(cols, "cols");
    std::vector<std::string> nm;
    std::vector<const double*> c;
    for (int i = 0; i < ncols; ++i) {
      require(names[i], "names[i]");
      nm.push_back(names[i]);
      c.push_back(n > 0 ? cols[i] : nullptr);
    }
    ffb::soa_write(path, nm, c, n);
  });
}

FFB_API int ffcu_dataset_save_soa(const ffit_dataset* ds, const char* path) {
  return guarded([&] {
    require(ds, "dataset");
    require(path, "path");
    const ffb::DeviceDataset& d = *ds->d;
    std::vector<std::vector<double>> host(d.cols.size(), std::vector<double>(static_cast<std::size_t>(d.n)));
    std::vector<const double*> c;
    for (std::size_t i = 0; i < d.cols.size(); ++i) {
      if (d.n > 0) d.download(static_cast<int>(i), host[i].data());
      c.push_back(host[i].data());
    }
    ffb::soa_write(path, d.names, c, d.n);
  });
}

FFB_API int ffcu_dataset_load_soa(const char* path, ffit_dataset** out, double* seconds) {
  return guarded([&] {
    require(path, "path");
    require(out, "out");
    ffb::SoaLoadStats st;
    auto d = ffb::soa_load_device(path, &st);
    if (seconds) *seconds = st.seconds;
    *out = new ffit_dataset{std::move(d)};
  });
}

FFB_API int ffcu_soa_info(const char* path, int* ncols, long long* nrows) {
  return guarded([&] {
    require(path, "path");
    const ffb::SoaHeader h = ffb::soa_read_header(path);
    if (ncols) *ncols = static_cast<int>(h.names.size());
    if (nrows) *nrows = h.nrows;
  });
}

FFB_API int ffcu_soa_column_name(const char* path, int col, char* buf, int cap) {
  return guarded([&] {
    require(path, "path");
    require(buf, "buf");
    const ffb::SoaHeader h = ffb::soa_read_header(path);
    if (col < 0 || col >= static_cast<int>(h.names.size())) ffb::usage_error("column index out of range");
    const std::string& s = h.names[col];
    if (cap < static_cast<int>(s.size()) + 1) ffb::usage_error("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

FFB_API int ffcu_soa_read_host(const char* path, double* const* cols) {
  return guarded([&] {
    require(path, "path");
    require(cols, "cols");
    ffb::SoaHeader h;
    const auto data = ffb::soa_read_host(path, &h);
    for (std::size_t c = 0; c < data.size(); ++c) {
      if (h.nrows > 0) {
        require(cols[c], "cols[c]");
        std::memcpy(cols[c], data[c].data(), static_cast<std::size_t>(h.nrows) * sizeof(double));
      }
    }
  });
}

FFB_API int ffcu_dataset_from_device(const char* const* names, const double* const* dev_cols, int ncols,
                                     long long n, int device, ffit_dataset** out) {
  return guarded([&] {
    require(names, "names");
    require(dev_cols, "dev_cols");
    require(out, "out");
    if (ncols <= 0) ffb::usage_error("a dataset needs at least one column");
    std::vector<std::string> nm;
    std::vector<const double*> c;
    for (int i = 0; i < ncols; ++i) {
      require(names[i], "names[i]");
      nm.push_back(names[i]);
      c.push_back(dev_cols[i]);
    }
    *out = new ffit_dataset{ffb::DeviceDataset::view(nm, c, n, device)};
  });
}

FFB_API int ffcu_dataset_copy_from_host(ffit_dataset* ds, const double* const* cols) {
  return guarded([&] {
    require(ds, "dataset");
    require(cols, "cols");
    if (!ds->d->owns) ffb::usage_error("cannot refill a view");
    std::vector<const double*> c(cols, cols + ds->d->cols.size());
    ds->d->copy_from_host(c);
  });
}

FFB_API int ffcu_dataset_copy_from_host_async(ffit_dataset* ds, const double* const* cols, void* stream) {
  return guarded([&] {
    require(ds, "dataset");
    require(cols, "cols");
    if (!ds->d->owns) ffb::usage_error("cannot refill a view");
    std::vector<const double*> c(cols, cols + ds->d->cols.size());
    ds->d->copy_from_host_async(c, static_cast<cudaStream_t>(stream));
  });
}

FFB_API int ffcu_dataset_slice(const ffit_dataset* ds, long long begin, long long end, ffit_dataset** out) {
  return guarded([&] {
    require(ds, "dataset");
    require(out, "out");
    if (begin < 0 || end < begin || end > ds->d->n) ffb::usage_error("slice out of range");
    std::vector<const double*> c;
    for (double* p : ds->d->cols) c.push_back(p + begin);
    auto v = ffb::DeviceDataset::view(ds->d->names, c, end - begin, ds->d->device);
    v->parent = ds->d;
    *out = new ffit_dataset{std::move(v)};
  });
}

FFB_API int ffcu_dataset_ncols(const ffit_dataset* ds) { return static_cast<int>(ds->d->cols.size()); }

FFB_API const char* ffcu_dataset_column_name(const ffit_dataset* ds, int i) {
  if (i < 0 || i >= static_cast<int>(ds->d->names.size())) return nullptr;
  return ds->d->names[i].c_str();
}

FFB_API int ffcu_dataset_download(const ffit_dataset* ds, int col, double* host_out) {
  return guarded([&] {
    require(ds, "dataset");
    require(host_out, "host_out");
    ds->d->download(col, host_out);
  });
}

FFB_API int ffcu_dataset_device_column(const ffit_dataset* ds, int col, const double** dev_ptr) {
  return guarded([&] {
    require(ds, "dataset");
    require(dev_ptr, "dev_ptr");
    if (col < 0 || col >= static_cast<int>(ds->d->cols.size())) ffb::usage_error("column index out of range");
    *dev_ptr = ds->d->cols[col];
  });
}

// ---------------------------------------------------------------------------
// fitting

FFB_API int ffit_fit(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double tolerance,
                     long max_iterations, ffit_fit_result** out) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(out, "out");
    require_gpu_mode(mode);
    ffb::FitOptions o;
    if (tolerance > 0.0) o.tolerance = tolerance;
    if (max_iterations > 0) o.max_iterations = static_cast<int>(max_iterations);
    auto r = std::make_unique<ffit_fit_result>();
    r->r = ffb::fit_nelder_mead(*m->m, engine(m), *ds->d, o);
    *out = r.release();
  });
}

FFB_API int ffcu_fit_gradient(ffit_model* m, const ffit_dataset* ds, double tolerance,
                              long max_iterations, ffit_fit_result** out) {
  return ffcu_fit_gradient_opts(m, ds, tolerance, max_iterations, -1, out);
}

FFB_API int ffcu_fit_gradient_opts(ffit_model* m, const ffit_dataset* ds, double tolerance,
                                   long max_iterations, int analytic, ffit_fit_result** out) {
  return guarded([&] {
    require(m, "model");
    require(ds, "dataset");
    require(out, "out");
    ffb::FitOptions o;
    o.record_trace = true;
    if (analytic < 0) {
      // automatic: analytic gradients, except for models with Expression pdfs while their
      // formula-specialised likelihood builds are on: the gradient of a Simpson-normalised
      // formula needs host quadratures of its derivative every call, and 2d+1 points of
      // the specialised build are faster (tools/expr_grad_bench.py: 0.87 vs 1.6 ms per
      // gradient on the config-2 text with m0 free, fit 0.012 vs 0.16 s)
      o.analytic_gradient = engine(m).likelihood_plan().programs.empty() || !ffb::jit_enabled();
    } else {
      o.analytic_gradient = analytic != 0;
    }
    if (tolerance > 0.0) o.tolerance = tolerance;
    if (max_iterations > 0) o.max_iterations = static_cast<int>(max_iterations);
    auto r = std::make_unique<ffit_fit_result>();
    r->r = ffb::fit_gradient(*m->m, engine(m), *ds->d, o);
    *out = r.release();
  });
}

// ---------------------------------------------------------------------------
// event-sharded likelihood over several GPUs (shard.hpp)

static_assert(sizeof(ncclUniqueId) == FFCU_NCCL_ID_BYTES, "NCCL unique id size");

FFB_API int ffcu_nccl_unique_id(void* id) {
  return guarded([&] {
    require(id, "id");
    ncclUniqueId u;
    ffb::nccl_check(ffb::nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

FFB_API const char* ffcu_nccl_version(void) {
  static thread_local std::string v;
  try {
    v = ffb::nccl().version;
  } catch (const std::exception& e) {
    v.clear();
  }
  return v.c_str();
}

FFB_API int ffcu_shard_group_create_rank(ffit_model* m, const ffit_dataset* shard, long long n_total,
                                         long long offset, const void* nccl_id, int world, int rank,
                                         ffcu_shard_group** out) {
  return guarded([&] {
    require(m, "model");
    require(shard, "dataset");
    require(nccl_id, "nccl_id");
    require(out, "out");
    ncclUniqueId u;
    std::memcpy(&u, nccl_id, sizeof(u));
    auto g = std::make_unique<ffcu_shard_group>();
    g->m = m;
    g->g = ffb::ShardGroup::create_rank(*m->m, shard->d, n_total, offset, u, world, rank);
    *out = g.release();
  });
}

FFB_API int ffcu_shard_group_create_local(ffit_model* m, const char* const* names, const double* const* host_cols,
                                          int ncols, long long n_total, const int* devices, int ndev,
                                          ffcu_shard_group** out) {
  return guarded([&] {
    require(m, "model");
    require(names, "names");
    require(host_cols, "host_cols");
    require(devices, "devices");
    require(out, "out");
    if (ncols <= 0 || ndev <= 0 || n_total < 0) ffb::usage_error("shard group: bad sizes");
    std::vector<std::string> nm;
    std::vector<const double*> cols;
    for (int i = 0; i < ncols; ++i) {
      require(names[i], "column name");
      if (n_total > 0) require(host_cols[i], "column");
      nm.emplace_back(names[i]);
      cols.push_back(host_cols[i]);
    }
    auto g = std::make_unique<ffcu_shard_group>();
    g->m = m;
    g->g = ffb::ShardGroup::create_local(*m->m, nm, cols, n_total, std::vector<int>(devices, devices + ndev));
    *out = g.release();
  });
}

FFB_API void ffcu_shard_group_free(ffcu_shard_group* g) { delete g; }

FFB_API int ffcu_shard_group_info(const ffcu_shard_group* g, int* world, int* local_devices, long long* n_total,
                                  long long* local_rows, long long* local_offset) {
  return guarded([&] {
    require(g, "group");
    if (world) *world = g->g->world();
    if (local_devices) *local_devices = g->g->local_count();
    if (n_total) *n_total = g->g->n_total();
    if (local_rows) *local_rows = g->g->local_rows(0);
    if (local_offset) *local_offset = g->g->local_offset(0);
  });
}

FFB_API int ffcu_shard_group_nll_points(ffcu_shard_group* g, const double* points, int P, double* values,
                                        long long* first_invalid, unsigned long long* n_evaluations) {
  return guarded([&] {
    require(g, "group");
    require(points, "points");
    require(values, "values");
    if (P < 0) ffb::usage_error("negative point count");
    const ffb::NllResult r = g->g->nll_points(points, P);
    std::copy(r.value.begin(), r.value.end(), values);
    if (first_invalid) std::copy(r.first_invalid.begin(), r.first_invalid.end(), first_invalid);
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_shard_group_nll_points_device(ffcu_shard_group* g, const double* points, int P, double* d_sc,
                                               unsigned long long* d_bad, void* stream, void* upload_stream,
                                               unsigned long long* n_evaluations) {
  return guarded([&] {
    require(g, "group");
    require(points, "points");
    require(d_sc, "d_sc");
    require(d_bad, "d_bad");
    const int k = g->g->nll_points_device(points, P, reinterpret_cast<ffb::SumPair*>(d_sc), d_bad,
                                          static_cast<cudaStream_t>(stream),
                                          static_cast<cudaStream_t>(upload_stream));
    if (n_evaluations) *n_evaluations = static_cast<unsigned long long>(k);
  });
}

FFB_API int ffcu_shard_group_nll_grad(ffcu_shard_group* g, const double* points, int P, double* values,
                                      double* grads, long long* first_invalid, unsigned long long* n_evaluations) {
  return guarded([&] {
    require(g, "group");
    require(points, "points");
    require(values, "values");
    require(grads, "grads");
    if (P < 0) ffb::usage_error("negative point count");
    const ffb::NllGradResult r = g->g->nll_grad_points(points, P);
    std::copy(r.value.begin(), r.value.end(), values);
    std::copy(r.grad.begin(), r.grad.end(), grads);
    if (first_invalid) std::copy(r.first_invalid.begin(), r.first_invalid.end(), first_invalid);
    if (n_evaluations) *n_evaluations = r.launches;
  });
}

FFB_API int ffcu_shard_group_fit(ffcu_shard_group* g, double tolerance, long max_iterations, ffit_fit_result** out) {
  return guarded([&] {
    require(g, "group");
    require(out, "out");
    ffb::FitOptions o;
    if (tolerance > 0.0) o.tolerance = tolerance;
    if (max_iterations > 0) o.max_iterations = static_cast<int>(max_iterations);
    auto r = std::make_unique<ffit_fit_result>();
    r->r = ffb::fit_nelder_mead(*g->m->m, *g->g, o);
    *out = r.release();
  });
}

FFB_API int ffcu_shard_group_fit_gradient(ffcu_shard_group* g, double tolerance, long max_iterations, int analytic,
                                          ffit_fit_result** out) {
  return guarded([&] {
    require(g, "group");
    require(out, "out");
    ffb::FitOptions o;
    o.record_trace = true;
    o.analytic_gradient = analytic < 0 ? g->g->engine(0).likelihood_plan().programs.empty() || !ffb::jit_enabled()
                                       : analytic != 0;
    if (tolerance > 0.0) o.tolerance = tolerance;
    if (max_iterations > 0) o.max_iterations = static_cast<int>(max_iterations);
    auto r = std::make_unique<ffit_fit_result>();
    r->r = ffb::fit_gradient(*g->m->m, *g->g, o);
    *out = r.release();
  });
}

FFB_API int ffit_result_converged(const ffit_fit_result* r) { return r->r.converged ? 1 : 0; }
FFB_API int ffcu_result_analytic_gradient(const ffit_fit_result* r) { return r->r.analytic_gradient ? 1 : 0; }
FFB_API double ffit_result_nll(const ffit_fit_result* r) { return r->r.nll_min; }
FFB_API unsigned long long ffit_result_nll_calls(const ffit_fit_result* r) { return r->r.n_nll_calls; }
FFB_API double ffit_result_wall_seconds(const ffit_fit_result* r) { return r->r.wall_seconds; }
FFB_API int ffit_result_uncertainties_valid(const ffit_fit_result* r) {
  return r->r.uncertainties_valid ? 1 : 0;
}
FFB_API int ffit_result_param_count(const ffit_fit_result* r) {
  return static_cast<int>(r->r.parameters.size());
}
FFB_API const char* ffit_result_param_name(const ffit_fit_result* r, int i) {
  if (i < 0 || i >= static_cast<int>(r->r.parameters.size())) return nullptr;
  return r->r.parameters[i].name.c_str();
}
FFB_API double ffit_result_param_value(const ffit_fit_result* r, int i) { return r->r.parameters[i].value; }
FFB_API double ffit_result_param_uncertainty(const ffit_fit_result* r, int i) {
  return r->r.parameters[i].uncertainty;
}
FFB_API void ffit_result_free(ffit_fit_result* r) { delete r; }

FFB_API int ffcu_result_iterations(const ffit_fit_result* r) { return r->r.iterations; }
FFB_API double ffcu_result_edm(const ffit_fit_result* r) { return r->r.edm; }
FFB_API unsigned long long ffcu_result_launches(const ffit_fit_result* r) { return r->r.n_launches; }
FFB_API int ffcu_result_trace(const ffit_fit_result* r, double* out, int cap) {
  const int n = static_cast<int>(r->r.trace.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = r->r.trace[i];
  return n;
}

// ---------------------------------------------------------------------------
// instrumentation

FFB_API int ffcu_last_launch(const ffit_model* m, int* info6) {
  return guarded([&] {
    require(m, "model");
    require(info6, "info6");
    const ffb::NllLaunchInfo i = m->engine->last_launch();
    info6[0] = i.threads;
    info6[1] = i.events_per_thread;
    info6[2] = i.tile;
    info6[3] = i.ntiles;
    info6[4] = i.nchunks;
    info6[5] = i.grid;
  });
}

FFB_API int ffcu_last_launch_cached(const ffit_model* m) { return m ? m->engine->last_launch().cached : 0; }

FFB_API unsigned long long ffcu_kernel_launches(void) { return ffb::kernel_launches(); }

FFB_API int ffcu_kernel_timer(int enable) {
  return guarded([&] { ffb::kernel_timer_enable(enable != 0); });
}

FFB_API int ffcu_kernel_timer_read(double* total_ms, unsigned long long* count) {
  return guarded([&] {
    require(total_ms, "total_ms");
    *total_ms = ffb::kernel_timer_read(count);
  });
}

FFB_API int ffcu_math_probe(int which, const double* in, double* out, long long n) {
  return guarded([&] {
    require(in, "in");
    require(out, "out");
    if (which < 0 || which > 3) ffb::usage_error("which must be 0 (exp), 1 (log), 2 (sqrt), 3 (rsqrt seed)");
    if (n <= 0) return;
    double *d_in = nullptr, *d_out = nullptr;
    const std::size_t bytes = static_cast<std::size_t>(n) * sizeof(double);
    ffb::cuda_check(cudaMalloc(&d_in, bytes), "cudaMalloc");
    ffb::cuda_check(cudaMalloc(&d_out, bytes), "cudaMalloc");
    cudaMemcpy(d_in, in, bytes, cudaMemcpyHostToDevice);
    ffb::count_launches(ffb::launch_math_probe(which, d_in, d_out, n, nullptr));
    const cudaError_t e = cudaMemcpy(out, d_out, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    ffb::cuda_check(e, "math_probe");
  });
}

FFB_API int ffcu_fp64_issue_probe(int others_per_8, double* fma_per_s) {
  return guarded([&] {
    require(fma_per_s, "fma_per_s");
    if (others_per_8 != 0 && others_per_8 != 2 && others_per_8 != 4 && others_per_8 != 5 && others_per_8 != 6 &&
        others_per_8 != 8 && others_per_8 != 16) {
      ffb::usage_error("ffcu_fp64_issue_probe: others_per_8 must be 0, 2, 4, 5, 6, 8 or 16");
    }
    cudaStream_t s;
    ffb::cuda_check(cudaStreamCreate(&s), "cudaStreamCreate");
    *fma_per_s = ffb::fp64_issue_probe(others_per_8, s);
    ffb::cuda_check(cudaGetLastError(), "fp64_issue_probe");
    cudaStreamDestroy(s);
    ffb::count_launches(2);
  });
}

FFB_API int ffcu_fp64_peak(double* fma_per_s, float* ms) {
  return guarded([&] {
    require(fma_per_s, "fma_per_s");
    cudaStream_t s;
    ffb::cuda_check(cudaStreamCreate(&s), "cudaStreamCreate");
    *fma_per_s = ffb::fp64_peak(s, ms);
    ffb::cuda_check(cudaGetLastError(), "fp64_peak");
    cudaStreamDestroy(s);
    ffb::count_launches(2);
  });
}
