// Fit drivers over a LikelihoodSource (one device or an event-sharded group).
//
// Transcribed blocks (the contract of ffit_fit is "the reference's Nelder-Mead" to 1e-6,
// which needs its iterates operation for operation; the batching into launches is new):
//   bound_transform / _inverse     proj/src/fit.cpp:12-28
//   invert (Gauss-Jordan)          proj/src/fit.cpp:53-84
//   Nelder-Mead simplex + loop     proj/src/fit.cpp:108-190 (initial simplex and shrink
//                                  issued as single multi-point launches)
//   hessian_at (point sequence)    proj/src/fit.cpp:200-225 (all points in one launch)
//   finish_with (write-back)       proj/src/fit.cpp:226-251
// fit_gradient (Minuit-style BFGS on analytic or central-difference gradients) is not in
// the reference.
#include "fit.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <numeric>

namespace ffb {

double bound_transform(double u, double lower, double upper) {
  return lower + (upper - lower) * (std::sin(u) + 1.0) * 0.5;  // proj/src/fit.cpp:12-14
}

double bound_transform_inverse(double p, double lower, double upper) {
  if (!(p > lower && p < upper)) {
    numeric_error("bound_transform_inverse: value " + std::to_string(p) + " not strictly inside (" +
                  std::to_string(lower) + ", " + std::to_string(upper) + ")");
  }
  return std::asin(2.0 * (p - lower) / (upper - lower) - 1.0);
}

namespace {

constexpr double kHalfPi = 1.5707963267948966;

// The objective over u-space points, evaluated in batches: one call = one
// multi-point GPU launch (the reference's Objective, proj/src/fit.cpp:30-49,
// evaluates one point per nll() call).
struct BatchObjective {
  Model& m;
  LikelihoodSource& src;
  std::vector<int> free_ids;
  unsigned long long calls = 0, batches = 0, kernels = 0;

  std::vector<double> theta_of(const std::vector<double>& u) const {
    std::vector<double> th = m.theta();
    for (std::size_t i = 0; i < free_ids.size(); ++i) {
      const Parameter& p = m.params[free_ids[i]];
      const double v = bound_transform(u[i], p.lo, p.hi);
      if (!(p.lo <= v && v <= p.hi)) {  // Graph::set_value, proj/src/graph.cpp:121-124
        numeric_error("set_value: " + std::to_string(v) + " outside range of '" + p.name + "'");
      }
      th[free_ids[i]] = v;
    }
    return th;
  }

  std::vector<double> operator()(const std::vector<std::vector<double>>& us) {
    const std::size_t npar = m.params.size();
    std::vector<double> rows(us.size() * npar);
    for (std::size_t k = 0; k < us.size(); ++k) {
      const std::vector<double> th = theta_of(us[k]);
      std::copy(th.begin(), th.end(), rows.begin() + static_cast<std::ptrdiff_t>(k * npar));
    }
    const NllResult r = src.nll_points(rows.data(), static_cast<int>(us.size()));
    calls += us.size();
    batches += 1;
    kernels += r.launches;
    return r.value;
  }

  double one(const std::vector<double>& u) { return (*this)({u})[0]; }

  void apply(const std::vector<double>& u) {
    const std::vector<double> th = theta_of(u);
    for (const int id : free_ids) m.params[id].value = th[id];
  }
};

// Gauss-Jordan with partial pivoting (proj/src/fit.cpp:53-84).
bool invert(std::vector<std::vector<double>>& a) {
  const std::size_t n = a.size();
  std::vector<std::vector<double>> inv(n, std::vector<double>(n, 0.0));
  for (std::size_t i = 0; i < n; ++i) inv[i][i] = 1.0;
  for (std::size_t col = 0; col < n; ++col) {
    std::size_t pivot = col;
    for (std::size_t r = col + 1; r < n; ++r) {
      if (std::fabs(a[r][col]) > std::fabs(a[pivot][col])) pivot = r;
    }
    if (!(std::fabs(a[pivot][col]) > 0.0) || !std::isfinite(a[pivot][col])) return false;
    std::swap(a[col], a[pivot]);
    std::swap(inv[col], inv[pivot]);
    const double d = a[col][col];
    for (std::size_t c = 0; c < n; ++c) {
      a[col][c] /= d;
      inv[col][c] /= d;
    }
    for (std::size_t r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = a[r][col];
      if (f == 0.0) continue;
      for (std::size_t c = 0; c < n; ++c) {
        a[r][c] -= f * a[col][c];
        inv[r][c] -= f * inv[col][c];
      }
    }
  }
  a = std::move(inv);
  return true;
}

std::vector<double> start_u(const Model& m, const std::vector<int>& free_ids) {
  std::vector<double> u(free_ids.size());
  for (std::size_t i = 0; i < free_ids.size(); ++i) {
    const Parameter& p = m.params[free_ids[i]];
    u[i] = bound_transform_inverse(p.value, p.lo, p.hi);
  }
  return u;
}

// Hessian points exactly as proj/src/fit.cpp:200-225 builds them (same
// floating-point operation sequence), evaluated as one batch.
bool hessian_at(BatchObjective& f, const std::vector<double>& u_min, double h,
                std::vector<std::vector<double>>& hess, std::vector<double>* grad = nullptr,
                double* f_centre = nullptr) {
  const std::size_t dim = u_min.size();
  std::vector<std::vector<double>> pts;
  pts.push_back(u_min);
  for (std::size_t i = 0; i < dim; ++i) {
    std::vector<double> up = u_min;
    up[i] = u_min[i] + h;
    pts.push_back(up);
    up[i] = u_min[i] - h;
    pts.push_back(up);
    for (std::size_t j = i + 1; j < dim; ++j) {
      up = u_min;
      up[i] += h;
      up[j] += h;
      pts.push_back(up);  // fpp
      up[j] -= 2.0 * h;
      pts.push_back(up);  // fpm
      up[i] -= 2.0 * h;
      pts.push_back(up);  // fmm
      up[j] += 2.0 * h;
      pts.push_back(up);  // fmp
    }
  }
  const std::vector<double> v = f(pts);
  hess.assign(dim, std::vector<double>(dim, 0.0));
  const double f0 = v[0];
  if (f_centre) *f_centre = f0;
  if (grad) grad->assign(dim, 0.0);
  std::size_t k = 1;
  for (std::size_t i = 0; i < dim; ++i) {
    const double fp = v[k++], fm = v[k++];
    if (grad) (*grad)[i] = (fp - fm) / (2.0 * h);  // the stencil's central difference (not in the reference)
    hess[i][i] = (fp - 2.0 * f0 + fm) / (h * h);
    for (std::size_t j = i + 1; j < dim; ++j) {
      const double fpp = v[k++], fpm = v[k++], fmm = v[k++], fmp = v[k++];
      hess[i][j] = hess[j][i] = (fpp - fpm - fmp + fmm) / (4.0 * h * h);
    }
  }
  return invert(hess);
}

// Rounding resolution of an NLL value: a few ulps of |f|.
double resolution(double f) { return 4.0 * std::numeric_limits<double>::epsilon() * std::fabs(f); }

// One Newton step from a BFGS minimum on the inverted u-space Hessian of the uncertainty
// estimate and the gradient at the same point (not in the reference; fit_gradient only).
// BFGS stops once its estimated distance to the minimum (EDM) is below the NLL's own
// rounding -- on a 2e8-event NLL ~ 5e8 that leaves it up to ~1e-3 sigma from the minimum;
// the full Hessian's step lands within the gradient's noise, for one more NLL point.  The
// step is kept unless the NLL rises beyond its rounding.
void newton_polish(BatchObjective& f, std::vector<double>& u, double& f_u, const std::vector<double>& g,
                   const std::vector<std::vector<double>>& hinv, FitResult& r) {
  const std::size_t d = u.size();
  std::vector<double> un = u;
  double pred = 0.0;
  for (std::size_t i = 0; i < d; ++i) {
    double s = 0.0;
    for (std::size_t j = 0; j < d; ++j) s -= hinv[i][j] * g[j];
    un[i] += s;
    pred -= 0.5 * g[i] * s;
  }
  if (!(pred > 0.0) || !std::isfinite(pred)) return;
  const double fn = f.one(un);
  // kept unless the NLL rises by more than its own rounding: a step whose predicted gain is
  // below the rounding cannot be judged by the NLL value, only by the model
  if (std::isfinite(fn) && fn <= f_u + resolution(f_u)) {
    u = un;
    f_u = fn;
    r.edm = 0.0;  // the step was the model's own estimate of the remaining distance
  }
}

// Leaves the model at u_min and writes values and uncertainties from the inverted
// u-space Hessian.
void finish_with(Model& m, BatchObjective& f, const std::vector<double>& u_min, bool invertible,
                 const std::vector<std::vector<double>>& hess, FitResult& r) {
  f.apply(u_min);  // leave the model in the fitted state (proj/src/fit.cpp:228-229)
  r.uncertainties_valid = invertible;
  r.parameters.clear();
  for (std::size_t i = 0; i < f.free_ids.size(); ++i) {
    Parameter& p = m.params[f.free_ids[i]];
    FittedParameter fp;
    fp.name = p.name;
    fp.value = p.value;
    if (invertible && hess[i][i] > 0.0) {
      const double jac = 0.5 * (p.hi - p.lo) * std::fabs(std::cos(u_min[i]));
      fp.uncertainty = std::sqrt(hess[i][i]) * jac;
    } else {
      fp.uncertainty = 0.0;
      r.uncertainties_valid = false;
    }
    p.error = fp.uncertainty;
    r.parameters.push_back(fp);
  }
}

void finish(Model& m, BatchObjective& f, const std::vector<double>& u_min, double h, FitResult& r) {
  std::vector<std::vector<double>> hess;
  const bool invertible = hessian_at(f, u_min, h, hess);
  finish_with(m, f, u_min, invertible, hess, r);
}

void validate(const Model& m, const FitOptions& o, const std::vector<int>& free_ids) {
  if (!(o.tolerance > 0.0) || o.max_iterations <= 0) usage_error("invalid fit options");
  if (free_ids.empty()) usage_error("fit requires at least one non-constant parameter");
  const std::vector<double> th = m.theta();
  m.check_params(m.root, th.data());
}

}  // namespace

// Device buffers sized once for the largest launch a fit of d free parameters issues (the
// batched Hessian: 1 + 2d + 2d(d-1) points; analytic: 2d gradient points), before the
// fit's clock starts: a buffer growth mid-fit re-pins host memory and frees device memory
// (an implicit device synchronisation) at an unpredictable cost.
static void reserve_for_fit(Model& m, LikelihoodSource& src, bool analytic) {
  const int d = static_cast<int>(m.free_parameters().size());
  src.reserve(std::min(1 + 2 * d + 2 * d * std::max(d - 1, 0), 512), analytic ? 2 * d : 0);
}

FitResult fit_nelder_mead(Model& m, LikelihoodSource& src, const FitOptions& o) {
  reserve_for_fit(m, src, false);
  const auto t0 = std::chrono::steady_clock::now();
  BatchObjective f{m, src, m.free_parameters()};
  validate(m, o, f.free_ids);
  const std::size_t dim = f.free_ids.size();
  const std::vector<double> u0 = start_u(m, f.free_ids);

  // initial simplex (proj/src/fit.cpp:108-123): u0 and d offset vertices, one batch
  std::vector<std::vector<double>> simplex(dim + 1, u0);
  for (std::size_t i = 0; i < dim; ++i) {
    double step = 0.1 * (kHalfPi - u0[i]);
    if (step < 1e-3) step = -0.1 * (u0[i] + kHalfPi);
    simplex[i + 1][i] += step;
  }
  std::vector<double> fv = f(simplex);
  if (!std::isfinite(fv[0])) {
    numeric_error("NLL is not finite at the starting parameters (zero-probability entry)");
  }

  FitResult result;
  std::vector<std::size_t> order(dim + 1);
  std::vector<double> centroid(dim), xr(dim), xe(dim), xc(dim);
  bool converged = false;
  int iter = 0;
  for (; iter < o.max_iterations; ++iter) {  // proj/src/fit.cpp:130-190
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return fv[a] < fv[b]; });
    const std::size_t best = order.front();
    const std::size_t worst = order.back();
    const std::size_t second_worst = order[dim - 1];
    if (o.record_trace) result.trace.push_back(fv[best]);
    if (fv[worst] - fv[best] < o.tolerance) {
      converged = true;
      break;
    }
    for (std::size_t i = 0; i < dim; ++i) {
      double s = 0.0;
      for (std::size_t v = 0; v <= dim; ++v) {
        if (v != worst) s += simplex[v][i];
      }
      centroid[i] = s / static_cast<double>(dim);
    }
    for (std::size_t i = 0; i < dim; ++i) xr[i] = centroid[i] + (centroid[i] - simplex[worst][i]);
    const double fr = f.one(xr);
    if (fr < fv[best]) {
      for (std::size_t i = 0; i < dim; ++i) xe[i] = centroid[i] + 2.0 * (centroid[i] - simplex[worst][i]);
      const double fe = f.one(xe);
      if (fe < fr) {
        simplex[worst] = xe;
        fv[worst] = fe;
      } else {
        simplex[worst] = xr;
        fv[worst] = fr;
      }
    } else if (fr < fv[second_worst]) {
      simplex[worst] = xr;
      fv[worst] = fr;
    } else {
      const bool outside = fr < fv[worst];
      if (outside) {
        for (std::size_t i = 0; i < dim; ++i) xc[i] = centroid[i] + 0.5 * (xr[i] - centroid[i]);
      } else {
        for (std::size_t i = 0; i < dim; ++i) xc[i] = centroid[i] + 0.5 * (simplex[worst][i] - centroid[i]);
      }
      const double fc = f.one(xc);
      if (fc < std::min(fr, fv[worst])) {
        simplex[worst] = xc;
        fv[worst] = fc;
      } else {  // shrink: d independent points, one batch
        std::vector<std::size_t> idx;
        std::vector<std::vector<double>> pts;
        for (std::size_t v = 0; v <= dim; ++v) {
          if (v == best) continue;
          for (std::size_t i = 0; i < dim; ++i) {
            simplex[v][i] = simplex[best][i] + 0.5 * (simplex[v][i] - simplex[best][i]);
          }
          idx.push_back(v);
          pts.push_back(simplex[v]);
        }
        const std::vector<double> vals = f(pts);
        for (std::size_t k = 0; k < idx.size(); ++k) fv[idx[k]] = vals[k];
      }
    }
  }
  std::size_t best = 0;
  for (std::size_t v = 1; v <= dim; ++v) {
    if (fv[v] < fv[best]) best = v;
  }
  result.converged = converged;
  result.nll_min = fv[best];
  result.iterations = iter;
  finish(m, f, simplex[best], o.fd_step, result);
  result.n_nll_calls = f.calls;
  result.n_launches = f.batches;
  result.kernel_launches = f.kernels;
  result.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

namespace {

// Value and u-space gradient at a batch of u points.  Analytic: the fused NLL +
// gradient pass (one launch pair for all points), chain rule through the sine
// transform d theta / d u = (hi - lo) cos(u) / 2.  Otherwise central differences:
// 2d+1 NLL points per u point, one launch.
struct GradObjective {
  BatchObjective& f;
  bool analytic;
  double h;
  std::vector<double> curv;  // finite differences: diagonal curvature at the first point

  void operator()(const std::vector<std::vector<double>>& us, std::vector<double>& fv,
                  std::vector<std::vector<double>>& gu) {
    const std::size_t d = f.free_ids.size();
    fv.assign(us.size(), 0.0);
    gu.assign(us.size(), std::vector<double>(d, 0.0));
    if (analytic) {
      const std::size_t npar = f.m.params.size();
      std::vector<double> rows(us.size() * npar);
      for (std::size_t k = 0; k < us.size(); ++k) {
        const std::vector<double> th = f.theta_of(us[k]);
        std::copy(th.begin(), th.end(), rows.begin() + static_cast<std::ptrdiff_t>(k * npar));
      }
      const NllGradResult r = f.src.nll_grad_points(rows.data(), static_cast<int>(us.size()));
      f.calls += us.size();
      f.batches += 1;
      f.kernels += r.launches;
      for (std::size_t k = 0; k < us.size(); ++k) {
        fv[k] = r.value[k];
        for (std::size_t i = 0; i < d; ++i) {
          const Parameter& p = f.m.params[f.free_ids[i]];
          gu[k][i] = r.grad[k * npar + f.free_ids[i]] * 0.5 * (p.hi - p.lo) * std::cos(us[k][i]);
        }
      }
      return;
    }
    std::vector<std::vector<double>> pts;
    for (const auto& u : us) {
      pts.push_back(u);
      for (std::size_t i = 0; i < d; ++i) {
        std::vector<double> a = u, b = u;
        a[i] += h;
        b[i] -= h;
        pts.push_back(a);
        pts.push_back(b);
      }
    }
    const std::vector<double> v = f(pts);
    curv.assign(d, 0.0);
    for (std::size_t k = 0; k < us.size(); ++k) {
      const double* w = v.data() + k * (2 * d + 1);
      fv[k] = w[0];
      for (std::size_t i = 0; i < d; ++i) {
        gu[k][i] = (w[1 + 2 * i] - w[2 + 2 * i]) / (2.0 * h);
        if (k == 0) curv[i] = (w[1 + 2 * i] - 2.0 * w[0] + w[2 + 2 * i]) / (h * h);
      }
    }
  }
};

}  // namespace


FitResult fit_gradient(Model& m, LikelihoodSource& src, const FitOptions& o) {
  const bool analytic = o.analytic_gradient && src.grad_ok();
  reserve_for_fit(m, src, analytic);
  const auto t0 = std::chrono::steady_clock::now();
  BatchObjective f{m, src, m.free_parameters()};
  validate(m, o, f.free_ids);
  const std::size_t d = f.free_ids.size();
  const double h = o.fd_step;
  GradObjective fg{f, analytic, h, {}};
  std::vector<double> u = start_u(m, f.free_ids);
  std::vector<double> u_prev, g_prev, u_best = u;
  std::vector<std::vector<double>> H(d, std::vector<double>(d, 0.0));
  double f_prev = std::numeric_limits<double>::infinity(), f_best = f_prev;
  bool have_prev = false, converged = false;
  int backtracks = 0, iter = 0;
  FitResult result;
  result.analytic_gradient = analytic;
  const bool debug = std::getenv("FFB_FIT_DEBUG") != nullptr;
  std::vector<double> fv;
  std::vector<std::vector<double>> gv;
  for (; iter < o.max_iterations; ++iter) {
    std::vector<double> g;
    double f0;
    if (!have_prev) {
      // start: the centre plus, for the initial inverse-Hessian diagonal, the
      // gradient at u +- h e_i (analytic: one launch of 2d+1 points; finite
      // differences: the curvature comes from the centre's own 2d+1 NLL values)
      std::vector<std::vector<double>> us(1, u);
      if (analytic) {
        for (std::size_t i = 0; i < d; ++i) {
          std::vector<double> a = u, b = u;
          a[i] += h;
          b[i] -= h;
          us.push_back(a);
          us.push_back(b);
        }
      }
      fg(us, fv, gv);
      f0 = fv[0];
      if (!std::isfinite(f0)) numeric_error("NLL is not finite at the starting parameters (zero-probability entry)");
      g = gv[0];
      for (std::size_t i = 0; i < d; ++i) {
        const double curv = analytic ? (gv[1 + 2 * i][i] - gv[2 + 2 * i][i]) / (2.0 * h) : fg.curv[i];
        H[i][i] = curv > 0.0 ? 1.0 / curv : 1e-2;
      }
    } else {
      fg({u}, fv, gv);
      f0 = fv[0];
      g = gv[0];
      if (!std::isfinite(f0) || f0 > f_prev) {
        if (debug) std::fprintf(stderr, "[fit_gradient] iter %d f %.17g > %.17g: backtrack\n", iter, f0, f_prev);
        // a rise inside the NLL's own rounding after the model already predicted a
        // gain below it: the minimum is resolved as far as the NLL can resolve it
        if (f0 - f_prev <= resolution(f_prev) && result.edm <= 100.0 * resolution(f_prev)) {
          converged = true;
          break;
        }
        if (++backtracks > 40) break;
        for (std::size_t i = 0; i < d; ++i) u[i] = u_prev[i] + 0.5 * (u[i] - u_prev[i]);
        continue;
      }
      backtracks = 0;
      // BFGS update of the inverse Hessian
      std::vector<double> s(d), y(d);
      double sy = 0.0;
      for (std::size_t i = 0; i < d; ++i) {
        s[i] = u[i] - u_prev[i];
        y[i] = g[i] - g_prev[i];
        sy += s[i] * y[i];
      }
      if (sy > 0.0) {
        const double rho = 1.0 / sy;
        std::vector<double> Hy(d, 0.0);
        for (std::size_t i = 0; i < d; ++i) {
          for (std::size_t j = 0; j < d; ++j) Hy[i] += H[i][j] * y[j];
        }
        double yHy = 0.0;
        for (std::size_t i = 0; i < d; ++i) yHy += y[i] * Hy[i];
        for (std::size_t i = 0; i < d; ++i) {
          for (std::size_t j = 0; j < d; ++j) {
            H[i][j] += (1.0 + rho * yHy) * rho * s[i] * s[j] - rho * (Hy[i] * s[j] + s[i] * Hy[j]);
          }
        }
      }
    }
    if (o.record_trace) result.trace.push_back(f0);
    if (f0 < f_best) {
      f_best = f0;
      u_best = u;
    }
    double edm = 0.0;
    std::vector<double> step(d, 0.0);
    for (std::size_t i = 0; i < d; ++i) {
      for (std::size_t j = 0; j < d; ++j) step[i] -= H[i][j] * g[j];
      edm -= 0.5 * g[i] * step[i];
    }
    result.edm = edm;
    if (debug) std::fprintf(stderr, "[fit_gradient] iter %d f %.17g edm %.3g\n", iter, f0, edm);
    // EDM below the tolerance, or below what the NLL value itself resolves (a
    // 2e8-event NLL ~ 5e8 carries ~1e-7 of rounding: a tolerance of 1e-12 is then
    // unreachable, as Minuit's "EDM below machine accuracy")
    if ((edm < o.tolerance || edm < resolution(f0)) && have_prev) {
      converged = true;
      break;
    }
    u_prev = u;
    g_prev = g;
    f_prev = f0;
    have_prev = true;
    for (std::size_t i = 0; i < d; ++i) u[i] += step[i];
  }
  result.converged = converged;
  result.nll_min = f_best;
  result.iterations = iter;
  if (analytic) {
    // Hessian from central differences of the analytic gradient: the centre and 2d points in
    // one launch of the gradient pass (instead of 1 + 2d + 2d(d-1) NLL points), symmetrised
    std::vector<std::vector<double>> us(1, u_best);
    for (std::size_t i = 0; i < d; ++i) {
      std::vector<double> a = u_best, b = u_best;
      a[i] += h;
      b[i] -= h;
      us.push_back(a);
      us.push_back(b);
    }
    fg(us, fv, gv);
    std::vector<std::vector<double>> hess(d, std::vector<double>(d, 0.0));
    for (std::size_t i = 0; i < d; ++i) {
      for (std::size_t j = 0; j < d; ++j) {
        hess[i][j] = 0.5 * ((gv[1 + 2 * j][i] - gv[2 + 2 * j][i]) + (gv[1 + 2 * i][j] - gv[2 + 2 * i][j])) / (2.0 * h);
      }
    }
    const bool invertible = invert(hess);
    if (invertible) newton_polish(f, u_best, f_best, gv[0], hess, result);
    result.nll_min = f_best;
    finish_with(m, f, u_best, invertible, hess, result);
  } else {
    std::vector<std::vector<double>> hess;
    std::vector<double> g0;
    const bool invertible = hessian_at(f, u_best, h, hess, &g0);
    if (invertible) newton_polish(f, u_best, f_best, g0, hess, result);
    result.nll_min = f_best;
    finish_with(m, f, u_best, invertible, hess, result);
  }
  result.n_nll_calls = f.calls;
  result.n_launches = f.batches;
  result.kernel_launches = f.kernels;
  result.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

bool hessian_uncertainties(Model& m, LikelihoodSource& src, double h, FitResult& r) {
  BatchObjective f{m, src, m.free_parameters()};
  if (f.free_ids.empty()) usage_error("no free parameters");
  finish(m, f, start_u(m, f.free_ids), h, r);
  r.n_nll_calls += f.calls;
  r.n_launches += f.batches;
  return r.uncertainties_valid;
}

}  // namespace ffb
