// Parameter derivatives of the once-per-point host quantities (fractions,
// normalisation integrals) for the fused NLL + gradient pass: the device sums
// A_c = sum W leaf_c and the host applies d coef_c / d theta_j (plan_build.cpp
// coef_derivatives), which needs d N / d theta_j for every normalised subtree.
//
// Closed forms where the normalisation itself is one (Gaussian, Exponential,
// Chebychev, Polynomial, the analytic sums); otherwise the same adaptive Simpson
// the normalisation uses (proj/src/eval.cpp:14-69) applied to the derivative of the
// integrand, d/d theta int u(x) dx = int du/d theta dx -- the derivative of the exact
// normalisation, not a finite difference of the quadrature (whose 1e-10 tolerance
// would swamp a difference quotient).
#include <algorithm>
#include <cmath>

#include "model.hpp"

namespace ffb {

namespace {

double tval(const double* theta, const Pdf& p, int k) { return theta[p.params[k]]; }

}  // namespace

bool Model::depends_on(int id, int j) const {
  const Pdf& p = pdfs[id];
  for (const int k : p.params) {
    if (k == j) return true;
  }
  for (const int c : p.children) {
    if (depends_on(c, j)) return true;
  }
  return false;
}

std::vector<double> Model::fractions_grad(int id, const double* theta, int j) const {
  const Pdf& p = pdfs[id];
  std::vector<double> d;
  if (p.kind == Kind::WeightedSum) {  // f_i = theta[k_i], f_n = 1 - sum
    double sum = 0.0;
    for (const int k : p.params) {
      d.push_back(k == j ? 1.0 : 0.0);
      sum += d.back();
    }
    d.push_back(-sum);
  } else {  // f_k = y_k / nu
    double nu = 0.0, dnu = 0.0;
    for (const int k : p.params) {
      nu += theta[k];
      dnu += k == j ? 1.0 : 0.0;
    }
    for (const int k : p.params) d.push_back(((k == j ? 1.0 : 0.0) - theta[k] / nu * dnu) / nu);
  }
  return d;
}

double Model::eval_unnorm_1d_grad(int id, const double* theta, double x, int j) const {
  const Pdf& p = pdfs[id];
  if (!depends_on(id, j)) return 0.0;
  double r = 0.0;
  switch (p.kind) {
    case Kind::Gaussian: {
      const double mu = tval(theta, p, 0), sigma = tval(theta, p, 1);
      const double d = x - mu;
      const double u = std::exp(-d * d / (2.0 * sigma * sigma));
      if (p.params[0] == j) r += u * d / (sigma * sigma);
      if (p.params[1] == j) r += u * d * d / (sigma * sigma * sigma);
      return r;
    }
    case Kind::Exponential:
      return std::exp(tval(theta, p, 0) * x) * x;
    case Kind::ChiSquare:
      return x > 0.0 ? eval_unnorm_1d(id, theta, x) * 0.5 * std::log(x) : 0.0;
    case Kind::JohnsonSU: {
      const double mu = tval(theta, p, 0), lambda = tval(theta, p, 1), delta = tval(theta, p, 3);
      const double u = eval_unnorm_1d(id, theta, x);
      const double z = (x - mu) / lambda;
      const double q = 1.0 + z * z, sq = std::sqrt(q);
      const double as = std::asinh(z);
      const double t = tval(theta, p, 2) + delta * as;
      const double D = -z / q - t * delta / sq;  // d log u / dz
      if (p.params[0] == j) r += u * (-D / lambda);
      if (p.params[1] == j) r += u * (-(1.0 + z * D) / lambda);
      if (p.params[2] == j) r += u * (-t);
      if (p.params[3] == j) r += u * (1.0 / delta - t * as);
      return r;
    }
    case Kind::ArgusBG: {
      const double m0 = tval(theta, p, 0), c = tval(theta, p, 1), pw = tval(theta, p, 2);
      const double rr = x / m0;
      const double t = 1.0 - rr * rr;
      if (!(t > 0.0)) return 0.0;
      const double u = eval_unnorm_1d(id, theta, x);
      if (p.params[0] == j) r += u * (pw / t + c) * 2.0 * rr * rr / m0;
      if (p.params[1] == j) r += u * t;
      if (p.params[2] == j) r += u * std::log(t);
      return r;
    }
    case Kind::Chebychev: {
      const Observable& o = observables[p.obs];
      const double z = (2.0 * x - (o.lo + o.hi)) / (o.hi - o.lo);
      double tm1 = 1.0, tk = z;
      for (const int a : p.params) {
        if (a == j) r += tk;
        const double tn = 2.0 * z * tk - tm1;
        tm1 = tk;
        tk = tn;
      }
      return r;
    }
    case Kind::Polynomial: {
      double xk = x;
      for (const int a : p.params) {
        if (a == j) r += xk;
        xk *= x;
      }
      return r;
    }
    case Kind::WeightedSum:
    case Kind::AddExtended: {  // sum_i (f_i / N_i) u_i
      const std::vector<double> f = fractions(id, theta);
      const std::vector<double> df = fractions_grad(id, theta, j);
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const int c = p.children[i];
        const double n = normalization(c, theta);
        const double dn = normalization_grad(c, theta, j);
        const double dcoef = (df[i] * n - f[i] * dn) / (n * n);
        r += dcoef * eval_unnorm_1d(c, theta, x) + f[i] / n * eval_unnorm_1d_grad(c, theta, x, j);
      }
      return r;
    }
    case Kind::ProdPdf:
      if (p.children.size() == 1) return eval_unnorm_1d_grad(p.children[0], theta, x, j);
      usage_error("eval_unnorm_1d_grad: multi-observable ProdPdf");
    case Kind::Expression: {  // forward mode through the formula: every slot reading theta_j moves
      double vs[16], dvs[16];
      std::vector<double> vb, dvb;
      double* v = vs;
      double* dv = dvs;
      if (p.expr_vars.size() > 16) {
        vb.resize(p.expr_vars.size());
        dvb.resize(p.expr_vars.size());
        v = vb.data();
        dv = dvb.data();
      }
      for (std::size_t i = 0; i < p.expr_vars.size(); ++i) {
        v[i] = p.expr_vars[i] < 0 ? x : theta[p.expr_vars[i]];
        dv[i] = p.expr_vars[i] == j ? 1.0 : 0.0;
      }
      double d = 0.0;
      p.program->eval_dual(v, dv, &d);
      return d;
    }
  }
  return 0.0;
}

double Model::normalization_grad(int id, const double* theta, int j) const {
  if (!depends_on(id, j)) return 0.0;
  const Pdf& p = pdfs[id];
  if (p.kind == Kind::ProdPdf) {  // N = prod N_k
    double r = 0.0;
    for (std::size_t k = 0; k < p.children.size(); ++k) {
      double term = normalization_grad(p.children[k], theta, j);
      if (term == 0.0) continue;
      for (std::size_t l = 0; l < p.children.size(); ++l) {
        if (l != k) term *= normalization(p.children[l], theta);
      }
      r += term;
    }
    return r;
  }
  if (p.kind == Kind::WeightedSum || p.kind == Kind::AddExtended) {
    // a sum of normalised components integrates to sum_i f_i (int u_i) / N_i: every
    // ratio is 1 for the exact integrals, so d N = sum_i df_i (0: the fractions sum
    // to 1) whichever quadrature evaluates N itself
    const std::vector<double> df = fractions_grad(id, theta, j);
    double r = 0.0;
    for (const double v : df) r += v;
    return r;
  }
  const Observable& o = observables[p.obs];
  const double lo = o.lo, hi = o.hi;
  switch (p.kind) {
    case Kind::Gaussian: {  // N = int exp(-(x-mu)^2 / (2 sigma^2))
      const double mu = tval(theta, p, 0), sigma = tval(theta, p, 1);
      const double dl = lo - mu, dh = hi - mu;
      const double gl = std::exp(-dl * dl / (2.0 * sigma * sigma));
      const double gh = std::exp(-dh * dh / (2.0 * sigma * sigma));
      double r = 0.0;
      if (p.params[0] == j) r += gl - gh;
      if (p.params[1] == j) r += (normalization(id, theta) - dh * gh + dl * gl) / sigma;
      return r;
    }
    case Kind::Exponential: {  // N = (e^{c hi} - e^{c lo}) / c
      const double c = tval(theta, p, 0);
      const double xm = std::max(std::fabs(lo), std::fabs(hi));
      if (std::fabs(c) * xm < 0.5) {
        // small |c|: dN/dc = int x e^{cx} = sum_n c^n (hi^{n+2} - lo^{n+2}) / (n! (n+2)),
        // free of the closed form's cancellation
        // (the stop test bounds the remaining terms by |c|^n xm^{n+2} / n!, since
        // symmetric ranges make every other term exactly 0)
        double r = 0.0, cn = 1.0, hn = hi * hi, ln = lo * lo, bound = xm * xm;
        for (int n = 0; n < 80; ++n) {
          r += cn * (hn - ln) / (n + 2);
          if (n > 2 && std::fabs(cn) * bound <= 1e-17 * std::fabs(r)) break;
          cn *= c / (n + 1);
          hn *= hi;
          ln *= lo;
          bound *= xm;
        }
        return r;
      }
      const double eh = std::exp(c * hi), el = std::exp(c * lo);
      return ((hi * eh - lo * el) - (eh - el) / c) / c;
    }
    case Kind::Chebychev: {  // N = (hi-lo)/2 (2 + sum_{k even} a_k 2/(1-k^2))
      double r = 0.0;
      for (std::size_t k = 1; k <= p.params.size(); ++k) {
        if (p.params[k - 1] == j && k % 2 == 0) {
          r += 0.5 * (hi - lo) * (2.0 / (1.0 - static_cast<double>(k) * static_cast<double>(k)));
        }
      }
      return r;
    }
    case Kind::Polynomial: {  // N = (hi-lo) + sum a_k (hi^{k+1} - lo^{k+1}) / (k+1)
      double r = 0.0, hk = hi, lk = lo;
      for (std::size_t k = 1; k <= p.params.size(); ++k) {
        hk *= hi;
        lk *= lo;
        if (p.params[k - 1] == j) r += (hk - lk) / static_cast<double>(k + 1);
      }
      return r;
    }
    default:
      break;
  }
  // ArgusBG, ChiSquare, JohnsonSU and Simpson-normalised sums: quadrature of the
  // derivative integrand with the normalisation's own tolerances
  const auto f = [&](double x) { return eval_unnorm_1d_grad(id, theta, x, j); };
  // absolute tolerance from the integrand's own scale (a coarse int |f|), so that a
  // derivative integral near zero does not drive the recursion to full depth
  constexpr int kCoarse = 64;
  double mag = 0.0;
  for (int i = 0; i < kCoarse; ++i) mag += std::fabs(f(lo + (i + 0.5) * (hi - lo) / kCoarse));
  mag *= (hi - lo) / kCoarse;
  if (!(mag > 0.0)) return 0.0;
  return integrate_adaptive_simpson(f, lo, hi, 1e-13 * mag, 1e-12, 50);
}

}  // namespace ffb
