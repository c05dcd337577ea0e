// C++ plug points of the reference engine, on the GPU path (header-only, C++20).
//
// The reference's C++ API (proj/include/ffit/eval.hpp:12-44, pdfs.hpp:46-66,
// model.hpp:22-56, dataset.hpp:21-51, fit.hpp:10-55, errors.hpp:8-25) restated over
// this library's C ABI (ffit_b200.h), so C++ host code written against the reference's
// `ffit::nll(Model&, const DataSet&, EvalMode)`, `ffit::probabilities(...)` and
// `PdfSpec::eval_batch(span xs, span out, ...)` keeps its call sites and gains
// `EvalMode::Gpu`.  Differences, all forced by the device boundary:
//
//   * DataSet keeps the reference's host columns (column() returns a span over them,
//     as the reference does) AND an HBM-resident copy, uploaded once at construction;
//   * Model is a handle over the library's model; parameters are addressed by name
//     (the reference's graph NodeIds do not cross the ABI);
//   * PdfSpec is a named (sub-)pdf of a Model; eval_batch over a host span uploads the
//     span for that call; the column-set overload (ProdPdf / several observables) reads
//     a DataSet's device columns;
//   * every EvalMode runs the fused sm_100a kernel (Scalar == BatchPrecise bitwise, as
//     in the reference, proj/tests/test_eval.cpp:113-157).
//
// Errors are thrown as ffit::Error with the reference's ErrorCode (status code of the
// failing C call, message from ffit_last_error()).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "ffit_b200.h"

namespace ffit {

// proj/include/ffit/errors.hpp:8-25
enum class ErrorCode { Usage = 1, Data = 2, Numeric = 3 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, std::string message) : std::runtime_error(std::move(message)), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

namespace detail {
inline void check(int rc) {
  if (rc != FFIT_OK) throw Error(static_cast<ErrorCode>(rc), ffit_last_error());
}
struct ModelFree {
  void operator()(ffit_model* m) const { ffit_model_free(m); }
};
struct DataFree {
  void operator()(ffit_dataset* d) const { ffit_dataset_free(d); }
};
}  // namespace detail

// proj/include/ffit/eval.hpp:12, plus the GPU plug point
enum class EvalMode { Scalar, BatchPrecise, BatchFast, Gpu };

// proj/include/ffit/eval.hpp:14-21.  n_evaluations: kernel launches (independent of
// n_entries, like the reference's batch-mode accounting).
struct NllValue {
  double value = 0.0;
  std::size_t n_entries = 0;
  std::uint64_t n_evaluations = 0;
  std::ptrdiff_t first_invalid = -1;
};

// proj/include/ffit/dataset.hpp:14-18
struct ObservableSpec {
  std::string name;
  double lower;
  double upper;
};

// proj/include/ffit/dataset.hpp:21-51: immutable column-major table; here the columns
// are also resident in HBM (one upload at construction).
class DataSet {
 public:
  DataSet() = default;
  DataSet(std::vector<std::string> names, std::vector<std::vector<double>> columns)
      : names_(std::move(names)), columns_(std::move(columns)) {
    if (names_.size() != columns_.size()) throw Error(ErrorCode::Usage, "names / columns count mismatch");
    n_rows_ = columns_.empty() ? 0 : columns_[0].size();
    std::vector<const char*> nm;
    std::vector<const double*> cp;
    for (std::size_t i = 0; i < names_.size(); ++i) {
      if (columns_[i].size() != n_rows_) throw Error(ErrorCode::Usage, "columns differ in length");
      nm.push_back(names_[i].c_str());
      cp.push_back(columns_[i].data());
    }
    ffit_dataset* d = nullptr;
    detail::check(ffcu_dataset_from_host(nm.data(), cp.data(), static_cast<int>(nm.size()),
                                         static_cast<long long>(n_rows_), &d));
    dev_ = std::shared_ptr<ffit_dataset>(d, detail::DataFree{});
  }

  void write_csv(const std::string& path) const { detail::check(ffit_dataset_write_csv(dev_.get(), path.c_str())); }

  std::size_t n_rows() const { return n_rows_; }
  std::size_t n_columns() const { return names_.size(); }
  const std::vector<std::string>& names() const { return names_; }
  bool has_column(std::string_view name) const {
    for (const auto& n : names_)
      if (n == name) return true;
    return false;
  }
  std::span<const double> column(std::string_view name) const {
    for (std::size_t i = 0; i < names_.size(); ++i)
      if (names_[i] == name) return columns_[i];
    throw Error(ErrorCode::Data, "unknown column: " + std::string(name));
  }
  std::map<std::string, double> row(std::size_t i) const {
    if (i >= n_rows_) throw Error(ErrorCode::Usage, "row index out of range");
    std::map<std::string, double> r;
    for (std::size_t c = 0; c < names_.size(); ++c) r[names_[c]] = columns_[c][i];
    return r;
  }

  // the device side (C ABI handle)
  const ffit_dataset* handle() const { return dev_.get(); }

 private:
  std::vector<std::string> names_;
  std::vector<std::vector<double>> columns_;
  std::size_t n_rows_ = 0;
  std::shared_ptr<ffit_dataset> dev_;
};

class Model;

// A named (sub-)pdf of a model: proj/include/ffit/pdfs.hpp:46-66
class PdfSpec {
 public:
  PdfSpec(Model& m, std::string name) : model_(&m), name_(std::move(name)) {}
  const std::string& name() const { return name_; }

  // One pass over a full column (1 observable): unnormalised values at the model's
  // current parameters.  kernel_calls counts kernel launches, as in the reference.
  void eval_batch(std::span<const double> xs, std::span<double> out, std::uint64_t* kernel_calls = nullptr) const;
  // The column-set generalisation (ProdPdf / several observables): the dataset's columns.
  void eval_batch(const DataSet& ds, std::span<double> out, std::uint64_t* kernel_calls = nullptr) const;

 private:
  Model* model_;
  std::string name_;
};

// proj/include/ffit/model.hpp:22-56
class Model {
 public:
  static std::unique_ptr<Model> from_file(const std::string& path) {
    ffit_model* m = nullptr;
    detail::check(ffit_model_load(path.c_str(), &m));
    return std::unique_ptr<Model>(new Model(m));
  }
  static std::unique_ptr<Model> from_string(const std::string& text, const std::string& /*origin*/ = "<string>") {
    ffit_model* m = nullptr;
    detail::check(ffit_model_parse(text.c_str(), &m));
    return std::unique_ptr<Model>(new Model(m));
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  const std::string obs_name() const { return ffit_model_observable(h_.get()); }
  double obs_lower() const { return range().first; }
  double obs_upper() const { return range().second; }
  ObservableSpec obs_spec() const { return ObservableSpec{obs_name(), obs_lower(), obs_upper()}; }
  std::vector<std::string> observables() const {
    std::vector<std::string> out;
    for (int i = 0; i < ffcu_model_observable_count(h_.get()); ++i) out.emplace_back(ffcu_model_observable_name(h_.get(), i));
    return out;
  }

  // parameters by name (model-file order)
  std::vector<std::string> parameters() const {
    std::vector<std::string> out;
    for (int i = 0; i < ffit_model_param_count(h_.get()); ++i) out.emplace_back(ffit_model_param_name(h_.get(), i));
    return out;
  }
  std::vector<std::string> free_parameters() const {
    std::vector<std::string> out;
    for (const auto& p : parameters()) {
      int c = 0;
      detail::check(ffit_model_param_is_constant(h_.get(), p.c_str(), &c));
      if (!c) out.push_back(p);
    }
    return out;
  }
  double get(const std::string& name, double* uncertainty = nullptr) const {
    double v = 0.0;
    detail::check(ffit_model_get_param(h_.get(), name.c_str(), &v, uncertainty));
    return v;
  }
  void set(const std::string& name, double v) { detail::check(ffit_model_set_param(h_.get(), name.c_str(), v)); }

  // the fit model (the last pdf line) and any named pdf
  PdfSpec pdf() { return PdfSpec(*this, ffcu_model_pdf_name(h_.get(), ffcu_model_pdf_count(h_.get()) - 1)); }
  PdfSpec pdf(const std::string& name) { return PdfSpec(*this, name); }

  // numeric normalisations (pdfs without a closed-form integral) by the device quadrature for
  // this model's likelihood / probabilities / eval_batch calls (off: the host's, as the reference)
  void set_device_normalization(bool on) { detail::check(ffcu_model_set_device_normalization(h_.get(), on ? 1 : 0)); }
  bool device_normalization() const { return ffcu_model_device_normalization(h_.get()) != 0; }

  ffit_model* handle() const { return h_.get(); }

 private:
  explicit Model(ffit_model* m) : h_(m) {}
  std::pair<double, double> range() const {
    double lo = 0.0, hi = 0.0;
    detail::check(ffit_model_observable_range(h_.get(), &lo, &hi));
    return {lo, hi};
  }
  std::unique_ptr<ffit_model, detail::ModelFree> h_;
};

inline void PdfSpec::eval_batch(std::span<const double> xs, std::span<double> out, std::uint64_t* kernel_calls) const {
  if (xs.size() != out.size()) throw Error(ErrorCode::Usage, "eval_batch: input and output lengths differ");
  if (xs.empty()) return;  // proj/src/pdfs.cpp:212-217
  DataSet ds({model_->obs_name()}, {std::vector<double>(xs.begin(), xs.end())});
  eval_batch(ds, out, kernel_calls);
}

inline void PdfSpec::eval_batch(const DataSet& ds, std::span<double> out, std::uint64_t* kernel_calls) const {
  if (out.size() != ds.n_rows()) throw Error(ErrorCode::Usage, "eval_batch: output length differs from the dataset");
  if (ds.n_rows() == 0) return;
  const unsigned long long k0 = ffcu_kernel_launches();
  detail::check(ffcu_eval_batch(model_->handle(), name_.c_str(), ds.handle(), out.data()));
  if (kernel_calls) *kernel_calls += ffcu_kernel_launches() - k0;
}

// normalization(spec, lo, hi, graph) (proj/include/ffit/eval.hpp:26) over the model's
// observable range at the current parameter values
inline double normalization(const Model& m, const std::string& pdf) {
  double v = 0.0;
  detail::check(ffcu_normalization(m.handle(), pdf.c_str(), nullptr, &v));
  return v;
}

// the same integral by the device quadrature (simpson_kernel; closed forms stay closed forms)
inline double device_normalization(const Model& m, const std::string& pdf) {
  double v = 0.0;
  detail::check(ffcu_device_normalization(m.handle(), pdf.c_str(), nullptr, 1, &v));
  return v;
}

// proj/include/ffit/eval.hpp:41 -- the plug point: EvalMode::Gpu (every mode runs the GPU)
inline NllValue nll(Model& model, const DataSet& ds, EvalMode mode) {
  (void)mode;
  const int np = ffit_model_param_count(model.handle());
  std::vector<double> point(static_cast<std::size_t>(np));
  for (int i = 0; i < np; ++i) point[i] = model.get(ffit_model_param_name(model.handle(), i));
  double v = 0.0;
  long long bad = -1;
  unsigned long long ne = 0;
  detail::check(ffcu_nll_points(model.handle(), ds.handle(), point.data(), 1, &v, &bad, &ne));
  NllValue out;
  out.value = v;
  out.n_entries = ds.n_rows();
  out.n_evaluations = ne;
  out.first_invalid = static_cast<std::ptrdiff_t>(bad);
  return out;
}

// proj/include/ffit/eval.hpp:44
inline void probabilities(Model& model, const DataSet& ds, EvalMode mode, std::span<double> out) {
  if (out.size() != ds.n_rows()) throw Error(ErrorCode::Usage, "probabilities: output length differs from the dataset");
  detail::check(ffit_probabilities(model.handle(), ds.handle(), static_cast<ffit_mode>(mode), out.data()));
}

// proj/include/ffit/fit.hpp:10-55
struct FitOptions {
  EvalMode mode = EvalMode::Gpu;
  double tolerance = 1e-8;
  int max_iterations = 10000;
  bool verbose = false;
  bool record_trace = false;
};

struct FittedParameter {
  std::string name;
  double value = 0.0;
  double uncertainty = 0.0;
};

struct FitResult {
  bool converged = false;
  double nll_min = 0.0;
  std::vector<FittedParameter> parameters;
  std::uint64_t n_nll_calls = 0;
  double wall_seconds = 0.0;
  bool uncertainties_valid = true;
  std::vector<double> trace;
};

// The reference's Nelder-Mead (initial simplex, shrink steps and Hessian points batched
// into single GPU launches); fitted values and uncertainties are written back.
inline FitResult fit_to(Model& model, const DataSet& ds, const FitOptions& o = {}) {
  ffit_fit_result* r = nullptr;
  detail::check(ffit_fit(model.handle(), ds.handle(), static_cast<ffit_mode>(o.mode), o.tolerance,
                         o.max_iterations, &r));
  std::unique_ptr<ffit_fit_result, void (*)(ffit_fit_result*)> guard(r, ffit_result_free);
  FitResult out;
  out.converged = ffit_result_converged(r) != 0;
  out.nll_min = ffit_result_nll(r);
  out.n_nll_calls = ffit_result_nll_calls(r);
  out.wall_seconds = ffit_result_wall_seconds(r);
  out.uncertainties_valid = ffit_result_uncertainties_valid(r) != 0;
  for (int i = 0; i < ffit_result_param_count(r); ++i)
    out.parameters.push_back({ffit_result_param_name(r, i), ffit_result_param_value(r, i),
                              ffit_result_param_uncertainty(r, i)});
  if (o.record_trace) {
    out.trace.resize(static_cast<std::size_t>(ffcu_result_trace(r, nullptr, 0)));
    if (!out.trace.empty()) ffcu_result_trace(r, out.trace.data(), static_cast<int>(out.trace.size()));
  }
  return out;
}

}  // namespace ffit
