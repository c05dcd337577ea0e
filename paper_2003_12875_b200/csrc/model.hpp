// Host-side model: observables, parameters and the PDF node tree.
//
// Mirrors the reference's node API (proj/include/ffit/pdfs.hpp:17-72: PdfKind,
// PdfSpec, check_params, analytic_integral, max_hint) and its model-file grammar
// (proj/src/model.cpp:113-252, proj/docs/model-file.md), extended with the kinds
// the GPU path adds: ArgusBG, Chebychev, Polynomial, ProdPdf (several observables)
// and the extended AddPdf.  The per-event computation never runs here: this file
// holds what the reference computes once per parameter point (validation,
// normalisation integrals; proj/src/eval.cpp:71-86) plus the toy generator's needs.
#pragma once

#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "common.hpp"
#include "expr.hpp"

namespace ffb {

enum class Kind {
  Gaussian,     // (x, mu, sigma)                proj/src/pdfs.cpp:15-26
  Exponential,  // (x, c)                        proj/src/pdfs.cpp:28-33
  ChiSquare,    // (x, k)                        proj/src/pdfs.cpp:35-52
  JohnsonSU,    // (x, mu, lambda, gamma, delta) proj/src/pdfs.cpp:54-77
  WeightedSum,  // (c1, f1, ..., cn): n-1 fractions, proj/src/pdfs.cpp:103-113,234-257
  AddExtended,  // AddPdf(c1, y1, ..., cn, yn): n yields, extended likelihood
  ArgusBG,      // (x, m0, c, p)
  Chebychev,    // (x, a1, ..., an)
  Polynomial,   // (x, a1, ..., an)
  ProdPdf,      // (p1, ..., pk) over independent observables
  Expression,   // ("formula", v1, ..., vk)      proj/src/model.cpp:218-232, proj/src/expr.cpp
};

const char* kind_name(Kind k);
bool is_leaf(Kind k);

struct Observable {
  std::string name;
  double lo = 0.0, hi = 0.0;
};

struct Parameter {
  std::string name;
  double value = 0.0, lo = 0.0, hi = 0.0;
  double error = 0.0;
  bool constant = false;
};

struct Pdf {
  Kind kind = Kind::Gaussian;
  std::string name;
  int obs = -1;                // observable index (leaves, sums: the common observable)
  std::vector<int> params;     // leaf parameters, or sum coefficients (fractions / yields)
  std::vector<int> children;   // component / factor pdf indices
  // Expression: the compiled formula and, per formula variable, the parameter index
  // or -1 for the observable (params then lists the distinct parameters)
  std::shared_ptr<const ExprProgram> program;
  std::vector<int> expr_vars;
};

class Model {
 public:
  std::vector<Observable> observables;
  std::vector<Parameter> params;
  std::vector<Pdf> pdfs;
  int root = -1;

  static std::unique_ptr<Model> parse(const std::string& text,
                                      const std::string& origin = "<string>");

  int param_index(const std::string& name) const;  // -1 if absent
  int pdf_index(const std::string& name) const;    // -1 if absent
  std::vector<double> theta() const;               // current values, declaration order
  std::vector<int> free_parameters() const;        // non-constant, declaration order
  bool extended() const { return pdfs[root].kind == Kind::AddExtended; }

  // Graph::set_value semantics (proj/src/graph.cpp:113-127): range-checked.
  void set_value(int param, double v);

  // PdfSpec::check_params (proj/src/pdfs.cpp:127-176) + restated kinds; throws Numeric.
  void check_params(int pdf, const double* theta) const;

  // Coefficients of a sum node: WeightedSum f_1..f_{n-1}, f_n = 1 - sum
  // (proj/src/pdfs.cpp:103-113); extended AddPdf f_k = y_k / nu.
  std::vector<double> fractions(int pdf, const double* theta) const;

  // normalization() (proj/src/eval.cpp:71-86): analytic where a closed form
  // exists, adaptive Simpson otherwise; ProdPdf = product of factor norms.
  double normalization(int pdf, const double* theta) const;
  std::optional<double> analytic_integral(int pdf, double lo, double hi,
                                          const double* theta) const;
  double simpson_integral(int pdf, const double* theta) const;
  // The 1-D nodes under `pdf` whose normalization() takes the Simpson route at theta (no
  // closed form), children before parents: what the device quadrature computes
  // (Engine::device_norms).
  std::vector<int> simpson_nodes(int pdf, const double* theta) const;

  // Unnormalised density at one point of a 1-D subtree (PdfSpec::eval_unnorm,
  // proj/src/pdfs.cpp:178-210).  Used for Simpson normalisation and the toy
  // generator only; the likelihood itself is evaluated on the GPU.
  double eval_unnorm_1d(int pdf, const double* theta, double x) const;

  // PdfSpec::max_hint: 1024-point grid max * 1.1 (proj/src/pdfs.cpp:309-323).
  double max_hint(int pdf, const double* theta) const;

  // Parameter derivatives for the fused gradient pass (model_grad.cpp): of the sum
  // coefficients, of a normalisation, of a 1-D subtree's unnormalised density.
  bool depends_on(int pdf, int param) const;
  std::vector<double> fractions_grad(int pdf, const double* theta, int param) const;
  double normalization_grad(int pdf, const double* theta, int param) const;
  double eval_unnorm_1d_grad(int pdf, const double* theta, double x, int param) const;

  // Extended term nu - N log nu (0 for non-extended models).
  double extended_term(const double* theta, double n_events) const;

  // Observable range of a 1-D subtree.
  const Observable& obs_of(int pdf) const { return observables[pdfs[pdf].obs]; }
};

// While alive on this thread, normalization(id, .) returns values[id] wherever it is not NaN
// (one entry per pdf): normalisations computed elsewhere -- the device quadrature -- for the
// parameter point being built.  The degenerate-value check still applies.
class NormOverride {
 public:
  explicit NormOverride(const double* values);
  ~NormOverride();
  NormOverride(const NormOverride&) = delete;
  NormOverride& operator=(const NormOverride&) = delete;

 private:
  const double* prev_;
};

// Adaptive Simpson with 32 pre-panels (proj/src/eval.cpp:14-69).
double integrate_adaptive_simpson(const std::function<double(double)>& f, double lo, double hi,
                                  double abs_tol, double rel_tol, int max_depth);

}  // namespace ffb
