// C++ host code written against the reference's C++ plug points (ffit::nll / probabilities /
// PdfSpec::eval_batch / fit_to, proj/include/ffit/{eval,pdfs,fit}.hpp), compiled against
// include/ffit_b200.hpp with EvalMode::Gpu.  Exit status 0 when every check holds.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ffit_b200.hpp"

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      ++failures;                                                      \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);       \
    } else {                                                           \
      std::printf("ok   %s\n", #cond);                                 \
    }                                                                  \
  } while (0)

int main() {
  auto model = ffit::Model::from_string(
      "observable x -5 5\n"
      "parameter mu 0.3 -2 2\n"
      "parameter sigma 1.1 0.1 3\n"
      "pdf g Gaussian(x, mu, sigma)\n");
  CHECK(model->obs_name() == "x" && model->obs_lower() == -5.0 && model->obs_upper() == 5.0);
  CHECK(model->free_parameters().size() == 2);
  std::vector<double> xs;
  for (int i = 0; i < 50001; ++i) xs.push_back(-4.9 + 9.8 * i / 50000.0);
  const ffit::DataSet ds({"x"}, {xs});
  CHECK(ds.n_rows() == xs.size() && ds.column("x")[7] == xs[7]);

  const ffit::NllValue g = ffit::nll(*model, ds, ffit::EvalMode::Gpu);
  const ffit::NllValue s = ffit::nll(*model, ds, ffit::EvalMode::Scalar);
  CHECK(std::isfinite(g.value) && g.first_invalid == -1 && g.n_entries == xs.size());
  CHECK(g.value == s.value && g.n_evaluations > 0);

  // probabilities and the span-style eval_batch: p = unnorm / norm, sum -log p == nll
  std::vector<double> p(xs.size()), u(xs.size());
  ffit::probabilities(*model, ds, ffit::EvalMode::Gpu, p);
  std::uint64_t calls = 0;
  model->pdf("g").eval_batch(xs, u, &calls);
  CHECK(calls >= 1);
  const double norm = ffit::normalization(*model, "g");
  const double want = 1.1 * std::sqrt(2.0 * M_PI) * 0.5 *
                      (std::erf((5.0 - 0.3) / (1.1 * std::sqrt(2.0))) - std::erf((-5.0 - 0.3) / (1.1 * std::sqrt(2.0))));
  CHECK(std::fabs(norm - want) <= 1e-13 * want);
  double worst = 0.0, sum = 0.0;
  for (std::size_t i = 0; i < xs.size(); ++i) {
    worst = std::fmax(worst, std::fabs(u[i] / norm - p[i]) / p[i]);
    const double d = xs[i] - 0.3;
    const double ref = std::exp(d * d * (-1.0 / (2.0 * 1.1 * 1.1)));
    worst = std::fmax(worst, std::fabs(u[i] - ref) / ref);
    sum += -std::log(p[i]);
  }
  CHECK(worst <= 1e-13);
  CHECK(std::fabs(sum - g.value) <= 1e-11 * std::fabs(g.value));

  // errors as ffit::Error with the reference's codes
  bool threw = false;
  try {
    model->set("sigma", -1.0);
  } catch (const ffit::Error& e) {
    threw = e.code() == ffit::ErrorCode::Numeric;
  }
  CHECK(threw);
  threw = false;
  try {
    std::vector<double> shorter(3);
    model->pdf("g").eval_batch(xs, shorter);
  } catch (const ffit::Error& e) {
    threw = e.code() == ffit::ErrorCode::Usage;
  }
  CHECK(threw);

  // a pdf without a closed-form integral: the device quadrature against the host's, and the
  // likelihood with the model's switch on
  {
    auto q = ffit::Model::from_string("observable x 0.1 15\nparameter k 3.5 0.5 20\npdf q ChiSquare(x, k)\n");
    const double host_norm = ffit::normalization(*q, "q");
    const double dev_norm = ffit::device_normalization(*q, "q");
    CHECK(std::fabs(dev_norm - host_norm) <= 1e-13 * host_norm);
    std::vector<double> qx;
    for (int i = 0; i < 5001; ++i) qx.push_back(0.2 + 14.0 * i / 5000.0);
    const ffit::DataSet qd({"x"}, {qx});
    const double host_nll = ffit::nll(*q, qd, ffit::EvalMode::Gpu).value;
    CHECK(!q->device_normalization());
    q->set_device_normalization(true);
    CHECK(q->device_normalization());
    const double dev_nll = ffit::nll(*q, qd, ffit::EvalMode::Gpu).value;
    CHECK(std::fabs(dev_nll - host_nll) <= 1e-13 * std::fabs(host_nll));
  }

  model->set("mu", 0.0);
  ffit::FitOptions o;
  o.tolerance = 1e-10;
  const ffit::FitResult r = ffit::fit_to(*model, ds, o);
  CHECK(r.converged && r.parameters.size() == 2 && r.nll_min <= g.value);
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
