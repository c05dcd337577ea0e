/* TEST INFRASTRUCTURE ONLY.  CPU restatement ("oracle") of the reference engine's
 * batch likelihood path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker.  Never linked into or called by the product.
 *
 * Parity pins: the parts the reference implements (Gaussian, Exponential,
 * ChiSquare, JohnsonSU, WeightedSum, Rng/samplers, Simpson, nll/probabilities)
 * are checked against the reference itself, compiled from its own sources into
 * oracle/_ref/libffit_ref.so, and against golden vectors generated from it
 * (tests/golden/, tests/golden/make_golden.py).  The parts the reference lacks
 * (ArgusBG, Chebychev, Polynomial, ProdPdf, the extended term) are restated here
 * following the reference's conventions and cross-checked against the reference's
 * Expression + adaptive-Simpson route (Argus, Chebychev, Polynomial), against
 * sums of 1-D reference NLLs (ProdPdf), and against closed-form known answers
 * (extended term: parity unpinned by any reference test).
 *
 * Compiled with -ffp-contract=off (the reference's x86-64 baseline build has no
 * FMA, so nothing contracts there either) and no -ffast-math.
 */
#define _GNU_SOURCE
#include "ffit_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------------ */
/* Rng: xoshiro256++ seeded by splitmix64            proj/src/sampling.cpp:9-54 */

typedef struct {
  uint64_t s[4];
  double spare;
  int have_spare;
} orc_rng;

static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9E3779B97f4A7C15ull;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static void rng_init(orc_rng* r, uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&s);
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t rng_next(orc_rng* r) {
  uint64_t* st = r->s;
  const uint64_t result = rotl(st[0] + st[3], 23) + st[0];
  const uint64_t t = st[1] << 17;
  st[2] ^= st[0];
  st[3] ^= st[1];
  st[1] ^= st[2];
  st[0] ^= st[3];
  st[2] ^= t;
  st[3] = rotl(st[3], 45);
  return result;
}

static double rng_uniform(orc_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_uniform_in(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * rng_uniform(r);
}

static double rng_gauss(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - rng_uniform(r);
  const double u2 = rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double a = 2.0 * atan(1.0) * 4.0 * u2;
  r->spare = rr * sin(a);
  r->have_spare = 1;
  return rr * cos(a);
}

void orc_rng_uniform(unsigned long long seed, long long n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (long long i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}

void orc_rng_gauss(unsigned long long seed, long long n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (long long i = 0; i < n; ++i) out[i] = rng_gauss(&r);
}

static int contains_prod(const orc_node* nodes, int id);

/* ------------------------------------------------------------------------ */
/* kernels                                                                   */

static const double kSqrt2Pi = 2.5066282746310005024;

#define P(k) (theta[nd->par[k]])

/* WeightedSum fractions: f_1..f_{n-1} free, last = 1 - sum   proj/src/pdfs.cpp:103-113
 * Extended AddPdf (restated): f_k = y_k / nu, nu = sum y_k, all explicit. */
static int fractions(const orc_node* nd, const double* theta, double* f) {
  if (nd->kind == ORC_WSUM) {
    double sum = 0.0;
    for (int i = 0; i < nd->npar; ++i) {
      f[i] = P(i);
      sum += f[i];
    }
    f[nd->npar] = 1.0 - sum;
    return nd->npar + 1;
  }
  double nu = 0.0;
  for (int i = 0; i < nd->npar; ++i) nu += P(i);
  for (int i = 0; i < nd->npar; ++i) f[i] = P(i) / nu;
  return nd->npar;
}

static double leaf_unnorm(const orc_node* nd, const double* theta, double x) {
  switch (nd->kind) {
    case ORC_GAUSS: { /* proj/src/pdfs.cpp:15-26 */
      const double mu = P(0), sigma = P(1);
      const double neg_inv_2s2 = -1.0 / (2.0 * sigma * sigma);
      const double d = x - mu;
      return exp(d * d * neg_inv_2s2);
    }
    case ORC_EXPO: /* proj/src/pdfs.cpp:28-33 */
      return exp(P(0) * x);
    case ORC_CHISQ: { /* proj/src/pdfs.cpp:35-52 */
      const double k = P(0);
      const double half_k_m1 = 0.5 * k - 1.0;
      const double at_zero = k == 2.0 ? 1.0 : 0.0;
      const double xa = x > 0.0 ? x : 1.0;
      const double v = exp(half_k_m1 * log(xa) - 0.5 * xa);
      const double pos = x > 0.0 ? 1.0 : 0.0;
      const double zero = x == 0.0 ? 1.0 : 0.0;
      const double b = zero * at_zero;
      return pos * v + (1.0 - pos) * b; /* fastmath::select, fastmath.hpp:24-26 */
    }
    case ORC_JOHNSON: { /* proj/src/pdfs.cpp:54-77 */
      const double mu = P(0), lambda = P(1), gamma = P(2), delta = P(3);
      const double inv_lambda = 1.0 / lambda;
      const double coef = delta / (lambda * kSqrt2Pi);
      const double z = (x - mu) * inv_lambda;
      const double az = fabs(z);
      const double as = copysign(log(az + sqrt(z * z + 1.0)), z);
      const double t = gamma + delta * as;
      return coef / sqrt(1.0 + z * z) * exp(-0.5 * t * t);
    }
    case ORC_ARGUS: {
      /* RooArgusBG form (restated; BASELINE.json configs[1]):
       *   x * (1-(x/m0)^2)^p * exp(c * (1-(x/m0)^2)),  0 for x >= m0.
       * p == 0.5 is evaluated with sqrt, as the Expression cross-check
       * "x*sqrt(1-(x/m0)^2)*exp(c*(1-(x/m0)^2))" does. */
      const double m0 = P(0), c = P(1), p = P(2);
      const double r = x / m0;
      const double t = 1.0 - r * r;
      if (!(t > 0.0)) return 0.0;
      const double w = p == 0.5 ? sqrt(t) : pow(t, p);
      return x * w * exp(c * t);
    }
    case ORC_CHEB: {
      /* RooChebychev form (restated): 1 + sum_k a_k T_k(z), z the affine map of
       * [lo, hi] onto [-1, 1]; T_k by the three-term recurrence, summed in k order. */
      const double z = (2.0 * x - (nd->lo + nd->hi)) / (nd->hi - nd->lo);
      double acc = 1.0;
      double tm1 = 1.0, tk = z;
      for (int k = 0; k < nd->npar; ++k) {
        acc += P(k) * tk;
        const double tn = 2.0 * z * tk - tm1;
        tm1 = tk;
        tk = tn;
      }
      return acc;
    }
    case ORC_POLY: {
      /* RooPolynomial form (restated): 1 + sum_{k>=1} a_k x^k, powers built by
       * repeated multiplication, summed in k order. */
      double acc = 1.0, xk = x;
      for (int k = 0; k < nd->npar; ++k) {
        acc += P(k) * xk;
        xk *= x;
      }
      return acc;
    }
  }
  return NAN;
}

/* ------------------------------------------------------------------------ */
/* adaptive Simpson                                    proj/src/eval.cpp:14-69 */

typedef struct {
  const orc_node* nodes;
  int id;
  const double* theta;
  int err;
} simpson_ctx;

static double eval1d(simpson_ctx* c, double x) {
  /* 1-D integrand: every leaf of this (sub)tree reads the same observable */
  double row[64];
  for (int i = 0; i < 64; ++i) row[i] = x;
  return orc_unnorm(c->nodes, c->id, c->theta, row);
}

static double simpson_recurse(simpson_ctx* c, double a, double b, double fa, double fm,
                              double fb, double whole, double abs_tol, double rel_tol,
                              int depth) {
  const double m = 0.5 * (a + b);
  const double lm = 0.5 * (a + m);
  const double rm = 0.5 * (m + b);
  const double flm = eval1d(c, lm);
  const double frm = eval1d(c, rm);
  if (!isfinite(flm) || !isfinite(frm)) c->err = 1;
  const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
  const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
  const double delta = left + right - whole;
  const double tol = abs_tol > rel_tol * fabs(left + right) ? abs_tol : rel_tol * fabs(left + right);
  if (c->err || depth <= 0 || fabs(delta) <= 15.0 * tol) return left + right + delta / 15.0;
  return simpson_recurse(c, a, m, fa, flm, fm, left, 0.5 * abs_tol, rel_tol, depth - 1) +
         simpson_recurse(c, m, b, fm, frm, fb, right, 0.5 * abs_tol, rel_tol, depth - 1);
}

static int simpson(simpson_ctx* c, double lo, double hi, double abs_tol, double rel_tol,
                   int max_depth, double* out) {
  if (!(lo < hi)) return fail(1, "integration range must satisfy lo < hi");
  const int kPanels = 32;
  const double width = (hi - lo) / kPanels;
  double total = 0.0;
  for (int p = 0; p < kPanels; ++p) {
    const double a = lo + p * width;
    const double b = p == kPanels - 1 ? hi : a + width;
    const double m = 0.5 * (a + b);
    const double fa = eval1d(c, a), fm = eval1d(c, m), fb = eval1d(c, b);
    if (!isfinite(fa) || !isfinite(fm) || !isfinite(fb)) return fail(3, "non-finite integrand");
    const double whole = (b - a) / 6.0 * (fa + 4.0 * fm + fb);
    total += simpson_recurse(c, a, b, fa, fm, fb, whole, abs_tol / kPanels, rel_tol, max_depth);
    if (c->err) return fail(3, "non-finite integrand");
  }
  *out = total;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* closed-form integrals                              proj/src/pdfs.cpp:271-307 */

/* G(t) = int_0^t sqrt(s) exp(c s) ds  (Argus p = 0.5 after x dx = -(m0^2/2) dt).
 * c < 0, |c| t >= 1: G = k^-3/2 [ (sqrt(pi)/2) erf(sqrt(k t)) - sqrt(k t) e^{-k t} ], k = -c
 * otherwise:         G = t^{3/2} sum_n (c t)^n / (n! (n + 3/2))   (converges for all c t) */
static double argus_G(double c, double t) {
  if (t <= 0.0) return 0.0;
  if (c < 0.0 && -c * t >= 1.0) {
    const double k = -c;
    const double y = k * t;
    const double sy = sqrt(y);
    const double g = 0.88622692545275801365 * erf(sy) - sy * exp(-y);
    return g / (k * sqrt(k));
  }
  const double ct = c * t;
  double term = 1.0, sum = 0.0;
  for (int n = 0; n < 400; ++n) {
    const double add = term / (n + 1.5);
    sum += add;
    if (fabs(add) <= 1e-17 * fabs(sum)) break;
    term *= ct / (n + 1);
  }
  return t * sqrt(t) * sum;
}

/* returns 1 and *out when a closed form exists over [lo, hi] */
static int analytic(const orc_node* nodes, int id, const double* theta, double lo, double hi,
                    double* out) {
  const orc_node* nd = &nodes[id];
  switch (nd->kind) {
    case ORC_GAUSS: {
      const double mu = P(0), sigma = P(1);
      const double inv = 1.0 / (sigma * sqrt(2.0));
      *out = sigma * sqrt(atan(1.0) * 2.0) * (erf((hi - mu) * inv) - erf((lo - mu) * inv));
      return 1;
    }
    case ORC_EXPO: {
      const double c = P(0);
      if (fabs(c) < 1e-12) *out = hi - lo;
      else *out = (exp(c * hi) - exp(c * lo)) / c;
      return 1;
    }
    case ORC_ARGUS: {
      const double m0 = P(0), c = P(1), p = P(2);
      if (p != 0.5 || !(m0 > 0.0)) return 0;
      const double a = lo > 0.0 ? lo : 0.0;
      const double b = hi < m0 ? hi : m0;
      if (!(a < b)) {
        *out = 0.0;
        return 1;
      }
      /* t = 1 - (x/m0)^2 = (m0-x)(m0+x)/m0^2, written without the cancellation */
      const double ta = ((m0 - a) * (m0 + a)) / (m0 * m0);
      const double tb = ((m0 - b) * (m0 + b)) / (m0 * m0);
      *out = 0.5 * m0 * m0 * (argus_G(c, ta) - argus_G(c, tb));
      return 1;
    }
    case ORC_CHEB: {
      /* full-range only: (hi-lo)/2 * (2 + sum_{k even} a_k * 2/(1-k^2)) */
      if (lo != nd->lo || hi != nd->hi) return 0;
      double s = 2.0;
      for (int k = 1; k <= nd->npar; ++k) {
        if (k % 2 == 0) s += P(k - 1) * (2.0 / (1.0 - (double)k * (double)k));
      }
      *out = 0.5 * (hi - lo) * s;
      return 1;
    }
    case ORC_POLY: {
      double s = hi - lo;
      double hk = hi, lk = lo;
      for (int k = 1; k <= nd->npar; ++k) {
        hk *= hi;
        lk *= lo;
        s += P(k - 1) * (hk - lk) / (double)(k + 1);
      }
      *out = s;
      return 1;
    }
    case ORC_PROD: { /* restated ProdPdf: product of the factor normalisations */
      double r = 1.0;
      for (int i = 0; i < nd->nchild; ++i) {
        double ni;
        if (orc_normalization(nodes, nd->child[i], theta, &ni)) return 0;
        r *= ni;
      }
      *out = r;
      return 1;
    }
    case ORC_WSUM:
    case ORC_ADDEXT: { /* proj/src/pdfs.cpp:288-300: sum f_i * part_i / norm_i */
      double f[ORC_MAXC + 1];
      fractions(nd, theta, f);
      double acc = 0.0;
      for (int i = 0; i < nd->nchild; ++i) {
        double part, norm;
        const orc_node* ch = &nodes[nd->child[i]];
        if (!analytic(nodes, nd->child[i], theta, lo, hi, &part)) return 0;
        analytic(nodes, nd->child[i], theta, ch->lo, ch->hi, &norm);
        acc += f[i] * part / norm;
      }
      *out = acc;
      return 1;
    }
    default:
      return 0;
  }
}

int orc_simpson_norm(const orc_node* nodes, int id, const double* theta, double* out) {
  const orc_node* nd = &nodes[id];
  simpson_ctx c = {nodes, id, theta, 0};
  return simpson(&c, nd->lo, nd->hi, 1e-10 * (nd->hi - nd->lo), 1e-10, 60, out);
}

/* proj/src/eval.cpp:71-86; ProdPdf (restated): product of factor norms */
int orc_normalization(const orc_node* nodes, int id, const double* theta, double* out) {
  const orc_node* nd = &nodes[id];
  double r;
  int multi = 0; /* a sum over products on several observables */
  if (nd->kind == ORC_WSUM || nd->kind == ORC_ADDEXT) {
    for (int i = 0; i < nd->nchild; ++i) multi |= contains_prod(nodes, nd->child[i]);
  }
  if (nd->kind == ORC_PROD) {
    r = 1.0;
    for (int i = 0; i < nd->nchild; ++i) {
      double ni;
      const int rc = orc_normalization(nodes, nd->child[i], theta, &ni);
      if (rc) return rc;
      r *= ni;
    }
  } else if (multi) { /* sum_i f_i N_i / N_i */
    double f[ORC_MAXC + 1];
    fractions(nd, theta, f);
    r = 0.0;
    for (int i = 0; i < nd->nchild; ++i) {
      double ni;
      const int rc = orc_normalization(nodes, nd->child[i], theta, &ni);
      if (rc) return rc;
      r += f[i] * ni / ni;
    }
  } else if (!analytic(nodes, id, theta, nd->lo, nd->hi, &r)) {
    const int rc = orc_simpson_norm(nodes, id, theta, &r);
    if (rc) return rc;
  }
  if (!(r > 0.0) || !isfinite(r)) return fail(3, "degenerate PDF: normalization integral <= 0");
  *out = r;
  return 0;
}

/* proj/src/pdfs.cpp:127-176, extended with the restated kinds */
int orc_check_params(const orc_node* nodes, int id, const double* theta) {
  const orc_node* nd = &nodes[id];
  switch (nd->kind) {
    case ORC_GAUSS:
      if (!(P(1) > 0.0)) return fail(3, "invalid parameters: sigma must be > 0");
      return 0;
    case ORC_CHISQ:
      if (!(P(0) > 0.0)) return fail(3, "invalid parameters: k must be > 0");
      return 0;
    case ORC_JOHNSON:
      if (!(P(1) > 0.0)) return fail(3, "invalid parameters: lambda must be > 0");
      if (!(P(3) > 0.0)) return fail(3, "invalid parameters: delta must be > 0");
      return 0;
    case ORC_ARGUS:
      if (!(P(0) > 0.0)) return fail(3, "invalid parameters: m0 must be > 0");
      if (!(P(2) >= 0.0)) return fail(3, "invalid parameters: p must be >= 0");
      return 0;
    case ORC_WSUM: {
      double sum = 0.0;
      for (int i = 0; i < nd->npar; ++i) {
        const double f = P(i);
        sum += f;
        if (!(f >= 0.0 && f <= 1.0)) return fail(3, "invalid parameters: fraction must be in [0, 1]");
      }
      if (sum > 1.0) return fail(3, "invalid parameters: fractions sum to more than 1");
      break;
    }
    case ORC_ADDEXT: {
      double nu = 0.0;
      for (int i = 0; i < nd->npar; ++i) {
        if (!(P(i) >= 0.0)) return fail(3, "invalid parameters: yield must be >= 0");
        nu += P(i);
      }
      if (!(nu > 0.0)) return fail(3, "invalid parameters: total yield must be > 0");
      break;
    }
    default:
      break;
  }
  for (int i = 0; i < nd->nchild; ++i) {
    const int rc = orc_check_params(nodes, nd->child[i], theta);
    if (rc) return rc;
  }
  return 0;
}

/* scalar path: PdfSpec::eval_unnorm                  proj/src/pdfs.cpp:178-210 */
double orc_unnorm(const orc_node* nodes, int id, const double* theta, const double* row) {
  const orc_node* nd = &nodes[id];
  switch (nd->kind) {
    case ORC_WSUM:
    case ORC_ADDEXT: {
      double f[ORC_MAXC + 1];
      fractions(nd, theta, f);
      double acc = 0.0;
      for (int i = 0; i < nd->nchild; ++i) {
        double norm;
        if (orc_normalization(nodes, nd->child[i], theta, &norm)) return NAN;
        const double coef = f[i] / norm;
        acc += coef * orc_unnorm(nodes, nd->child[i], theta, row);
      }
      return acc;
    }
    case ORC_PROD: {
      double acc = orc_unnorm(nodes, nd->child[0], theta, row);
      for (int i = 1; i < nd->nchild; ++i) acc *= orc_unnorm(nodes, nd->child[i], theta, row);
      return acc;
    }
    default:
      return leaf_unnorm(nd, theta, row[nd->col]);
  }
}

/* batch path: PdfSpec::eval_batch                    proj/src/pdfs.cpp:212-269 */
int orc_eval_batch(const orc_node* nodes, int id, const double* theta,
                   const double* const* cols, long long n, double* out) {
  const orc_node* nd = &nodes[id];
  if (n == 0) return 0;
  int rc = orc_check_params(nodes, id, theta);
  if (rc) return rc;
  switch (nd->kind) {
    case ORC_WSUM:
    case ORC_ADDEXT: {
      double f[ORC_MAXC + 1];
      fractions(nd, theta, f);
      for (long long i = 0; i < n; ++i) out[i] = 0.0;
      double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
      for (int c = 0; c < nd->nchild; ++c) {
        double norm;
        rc = orc_normalization(nodes, nd->child[c], theta, &norm);
        if (!rc) rc = orc_eval_batch(nodes, nd->child[c], theta, cols, n, tmp);
        if (rc) {
          free(tmp);
          return rc;
        }
        const double coef = f[c] / norm;
        for (long long i = 0; i < n; ++i) out[i] += coef * tmp[i];
      }
      free(tmp);
      return 0;
    }
    case ORC_PROD: {
      rc = orc_eval_batch(nodes, nd->child[0], theta, cols, n, out);
      if (rc) return rc;
      double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
      for (int c = 1; c < nd->nchild; ++c) {
        rc = orc_eval_batch(nodes, nd->child[c], theta, cols, n, tmp);
        if (rc) {
          free(tmp);
          return rc;
        }
        for (long long i = 0; i < n; ++i) out[i] *= tmp[i];
      }
      free(tmp);
      return 0;
    }
    default: {
      const double* xs = cols[nd->col];
      for (long long i = 0; i < n; ++i) out[i] = leaf_unnorm(nd, theta, xs[i]);
      return 0;
    }
  }
}

/* probabilities (batch modes)                         proj/src/eval.cpp:174-192 */
int orc_probabilities(const orc_node* nodes, int root, const double* theta,
                      const double* const* cols, long long n, double* out) {
  int rc = orc_check_params(nodes, root, theta);
  if (rc) return rc;
  if (n == 0) return 0;
  double norm;
  rc = orc_normalization(nodes, root, theta, &norm);
  if (rc) return rc;
  rc = orc_eval_batch(nodes, root, theta, cols, n, out);
  if (rc) return rc;
  for (long long i = 0; i < n; ++i) out[i] = out[i] / norm;
  return 0;
}

/* Extended term (restated, RooFit convention): nu - N log nu, nu = sum of yields.
 * NLL_ext = -sum_i log(sum_k y_k p_k(x_i) / nu) + nu - N log nu. */
double orc_extended_term(const orc_node* nodes, int root, const double* theta, long long n) {
  const orc_node* nd = &nodes[root];
  if (nd->kind != ORC_ADDEXT) return 0.0;
  double nu = 0.0;
  for (int i = 0; i < nd->npar; ++i) nu += P(i);
  return nu - (double)n * log(nu);
}

/* nll_batch (Precise)                                 proj/src/eval.cpp:119-163
 * *naive = the reference's left-to-right sum; *compensated = Neumaier sum of the
 * same per-event -log(p) (the value parity is graded against). */
int orc_nll(const orc_node* nodes, int root, const double* theta, const double* const* cols,
            long long n, double* naive, double* compensated, long long* first_invalid) {
  int rc = orc_check_params(nodes, root, theta);
  if (rc) return rc;
  *first_invalid = -1;
  if (n == 0) {
    *naive = *compensated = orc_extended_term(nodes, root, theta, 0);
    return 0;
  }
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  rc = orc_probabilities(nodes, root, theta, cols, n, p);
  if (rc) {
    free(p);
    return rc;
  }
  for (long long i = 0; i < n; ++i) {
    if (!(p[i] > 0.0) || !isfinite(p[i])) {
      *first_invalid = i;
      *naive = *compensated = INFINITY;
      free(p);
      return 0;
    }
  }
  double v = 0.0, s = 0.0, c = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double l = -log(p[i]);
    v += l;
    const double t = s + l;
    if (fabs(s) >= fabs(l)) c += (s - t) + l;
    else c += (l - t) + s;
    s = t;
  }
  free(p);
  const double ext = orc_extended_term(nodes, root, theta, n);
  *naive = v + ext;
  *compensated = (s + c) + ext;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* threaded multi-point NLL: the CPU baseline "port" leg                     */

typedef struct {
  const orc_node* nodes;
  int root;
  const double* thetas;
  int ntheta, P;
  const double* const* cols;
  long long n;
  double* values;
  int next;
  pthread_mutex_t mu;
  int rc;
} points_job;

static void* points_worker(void* arg) {
  points_job* j = (points_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int p = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (p >= j->P) break;
    double naive, comp;
    long long bad;
    const int rc = orc_nll(j->nodes, j->root, j->thetas + (size_t)p * j->ntheta, j->cols, j->n,
                           &naive, &comp, &bad);
    if (rc) j->rc = rc;
    j->values[p] = comp;
  }
  return NULL;
}

int orc_nll_points(const orc_node* nodes, int root, const double* thetas, int ntheta, int P,
                   const double* const* cols, long long n, int threads, double* values) {
  points_job j = {nodes, root, thetas, ntheta, P, cols, n, values, 0,
                  PTHREAD_MUTEX_INITIALIZER, 0};
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, points_worker, &j);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  return j.rc;
}

/* ------------------------------------------------------------------------ */
/* seeded generator                                    proj/src/sampling.cpp:56-197
 * Reference semantics for the kinds it has (direct samplers for Gaussian,
 * Exponential, JohnsonSU and WeightedSum-of-direct; accept/reject on the whole
 * PDF against max_hint otherwise).  Restated kinds (ArgusBG, Chebychev,
 * Polynomial) carry their own accept/reject sampler against their own max_hint
 * and count as "direct" inside a mixture (pick-then-draw);
 * ProdPdf samples factor k from its own stream Rng(seed + 10 k).  */

typedef struct {
  const orc_node* nodes;
  const double* theta;
  orc_rng rng;
  double bound[64]; /* per-node A/R envelope (max_hint), 0 = unset */
  unsigned long long proposed, accepted;
  int err;
} sampler;

static int has_direct(const orc_node* nodes, int id) {
  const orc_node* nd = &nodes[id];
  switch (nd->kind) {
    case ORC_GAUSS: case ORC_EXPO: case ORC_JOHNSON:
    case ORC_ARGUS: case ORC_CHEB: case ORC_POLY:
      return 1;
    case ORC_WSUM: case ORC_ADDEXT:
      for (int i = 0; i < nd->nchild; ++i)
        if (!has_direct(nodes, nd->child[i])) return 0;
      return 1;
    default:
      return 0;
  }
}

/* PdfSpec::max_hint: 1024-point grid max * 1.1       proj/src/pdfs.cpp:309-323 */
static double max_hint(const orc_node* nodes, int id, const double* theta) {
  const orc_node* nd = &nodes[id];
  const double lo = nd->lo, hi = nd->hi;
  const int kGrid = 1024;
  double best = 0.0;
  const double step = (hi - lo) / (kGrid - 1);
  double row[64];
  for (int i = 0; i < kGrid; ++i) {
    const double x = i == kGrid - 1 ? hi : lo + i * step;
    for (int k = 0; k < 64; ++k) row[k] = x;
    const double v = orc_unnorm(nodes, id, theta, row);
    if (v > best) best = v;
  }
  return best * 1.1;
}

/* one accepted draw of accept_reject                  proj/src/sampling.cpp:56-88 */
static double ar_draw(sampler* s, int id) {
  const orc_node* nd = &s->nodes[id];
  const double bound = s->bound[id];
  double row[64];
  for (;;) {
    const double x = rng_uniform_in(&s->rng, nd->lo, nd->hi);
    for (int k = 0; k < 64; ++k) row[k] = x;
    const double p = orc_unnorm(s->nodes, id, s->theta, row);
    ++s->proposed;
    if (p > bound) {
      s->err = fail(3, "accept/reject: pdf exceeds envelope bound");
      return NAN;
    }
    if (rng_uniform(&s->rng) * bound < p) {
      ++s->accepted;
      return x;
    }
    if (s->proposed >= 1000000ull && (double)s->accepted / (double)s->proposed < 1e-6) {
      s->err = fail(3, "accept/reject: acceptance rate below 1e-6");
      return NAN;
    }
  }
}

/* draw_direct                                          proj/src/sampling.cpp:96-168 */
static double draw(sampler* s, int id) {
  const orc_node* nd = &s->nodes[id];
  const double* theta = s->theta;
  switch (nd->kind) {
    case ORC_GAUSS: {
      for (;;) {
        const double x = P(0) + P(1) * rng_gauss(&s->rng);
        if (x >= nd->lo && x <= nd->hi) return x;
      }
    }
    case ORC_EXPO: {
      const double c = P(0);
      const double u = rng_uniform(&s->rng);
      if (fabs(c) < 1e-12) return nd->lo + u * (nd->hi - nd->lo);
      return nd->lo + log1p(u * expm1(c * (nd->hi - nd->lo))) / c;
    }
    case ORC_JOHNSON: {
      for (;;) {
        const double z = rng_gauss(&s->rng);
        const double x = P(0) + P(1) * sinh((z - P(2)) / P(3));
        if (x >= nd->lo && x <= nd->hi) return x;
      }
    }
    case ORC_WSUM:
    case ORC_ADDEXT: {
      double f[ORC_MAXC + 1];
      fractions(nd, theta, f);
      double cum[ORC_MAXC + 1];
      double sum = 0.0;
      const int ncum = nd->nchild - 1;
      for (int i = 0; i < ncum; ++i) {
        sum += f[i];
        cum[i] = sum;
      }
      const double u = rng_uniform(&s->rng);
      int pick = nd->nchild - 1;
      for (int i = 0; i < ncum; ++i) {
        if (u < cum[i]) {
          pick = i;
          break;
        }
      }
      return draw(s, nd->child[pick]);
    }
    default: /* restated leaves: their own accept/reject */
      return ar_draw(s, id);
  }
}

static void prepare_bounds(sampler* s, int id) {
  const orc_node* nd = &s->nodes[id];
  if (nd->kind == ORC_ARGUS || nd->kind == ORC_CHEB || nd->kind == ORC_POLY) {
    s->bound[id] = max_hint(s->nodes, id, s->theta);
  }
  for (int i = 0; i < nd->nchild; ++i) prepare_bounds(s, nd->child[i]);
}

static int contains_prod(const orc_node* nodes, int id) {
  if (nodes[id].kind == ORC_PROD) return 1;
  for (int i = 0; i < nodes[id].nchild; ++i)
    if (contains_prod(nodes, nodes[id].child[i])) return 1;
  return 0;
}

static int sample_1d(const orc_node* nodes, int id, const double* theta, long long n,
                     unsigned long long seed, double* out, unsigned long long* proposed,
                     unsigned long long* accepted) {
  if (contains_prod(nodes, id)) return fail(1, "sampling needs a one-dimensional pdf per factor");
  sampler* s = (sampler*)calloc(1, sizeof(sampler));
  s->nodes = nodes;
  s->theta = theta;
  rng_init(&s->rng, seed);
  int rc = 0;
  if (has_direct(nodes, id)) {
    prepare_bounds(s, id);
    for (long long i = 0; i < n && !s->err; ++i) out[i] = draw(s, id);
  } else {
    s->bound[id] = max_hint(nodes, id, theta);
    if (s->bound[id] == 0.0) rc = fail(3, "cannot sample: pdf is zero over the whole range");
    for (long long i = 0; i < n && !s->err && !rc; ++i) out[i] = ar_draw(s, id);
  }
  if (s->err) rc = s->err;
  *proposed += s->proposed;
  *accepted += s->accepted;
  free(s);
  return rc;
}

int orc_sample(const orc_node* nodes, int root, const double* theta, long long n,
               unsigned long long seed, double* const* cols, double* efficiency) {
  int rc = orc_check_params(nodes, root, theta);
  if (rc) return rc;
  unsigned long long proposed = 0, accepted = 0;
  const orc_node* nd = &nodes[root];
  if (nd->kind == ORC_PROD) {
    for (int k = 0; k < nd->nchild; ++k) {
      const int c = nd->child[k];
      rc = sample_1d(nodes, c, theta, n, seed + 10ull * (unsigned long long)k,
                     cols[nodes[c].col], &proposed, &accepted);
      if (rc) return rc;
    }
  } else {
    rc = sample_1d(nodes, root, theta, n, seed, cols[nd->col], &proposed, &accepted);
    if (rc) return rc;
  }
  if (efficiency) *efficiency = proposed == 0 ? -1.0 : (double)accepted / (double)proposed;
  return 0;
}
