#include "plan_build.hpp"

#include <algorithm>
#include <cmath>

namespace ffb {

namespace {

constexpr double kSqrt2Pi = 2.5066282746310005024;

// One traversal serves both compile (structure) and build (constants): the
// flattening depends only on the tree, so every point yields the same terms.
struct Emitter {
  const Model& m;
  const double* theta;  // may be null when only the structure is wanted
  std::vector<DevTerm> terms;
  std::vector<double> consts;
  std::vector<int> col_obs;
  std::vector<int> term_pdf;
  std::vector<ExprInstr> programs;

  int slot(int obs) {
    for (std::size_t i = 0; i < col_obs.size(); ++i) {
      if (col_obs[i] == obs) return static_cast<int>(i);
    }
    col_obs.push_back(obs);
    return static_cast<int>(col_obs.size()) - 1;
  }

  double norm(int pdf) const { return theta ? m.normalization(pdf, theta) : 1.0; }
  std::vector<double> fracs(int pdf) const {
    if (theta) return m.fractions(pdf, theta);
    return std::vector<double>(m.pdfs[pdf].children.size(), 1.0);
  }
  double par(const Pdf& p, int k) const { return theta ? theta[p.params[k]] : 0.0; }

  // scale * unnorm(leaf)
  void leaf(int id, double scale) {
    const Pdf& p = m.pdfs[id];
    DevTerm t{};
    t.col = slot(p.obs);
    t.coff = static_cast<int>(consts.size());
    consts.push_back(scale);
    switch (p.kind) {
      case Kind::Gaussian: {  // GaussianKernel, proj/src/pdfs.cpp:15-26
        t.kind = LK_GAUSS;
        const double sigma = par(p, 1);
        consts.push_back(par(p, 0));
        consts.push_back(theta ? -1.0 / (2.0 * sigma * sigma) : 0.0);
        break;
      }
      case Kind::Exponential:  // ExponentialKernel, proj/src/pdfs.cpp:28-33
        t.kind = LK_EXPO;
        consts.push_back(par(p, 0));
        break;
      case Kind::ChiSquare: {  // ChiSquareKernel, proj/src/pdfs.cpp:35-52
        t.kind = LK_CHISQ;
        const double k = par(p, 0);
        consts.push_back(0.5 * k - 1.0);
        consts.push_back(k == 2.0 ? 1.0 : 0.0);
        break;
      }
      case Kind::JohnsonSU: {  // JohnsonKernel, proj/src/pdfs.cpp:54-77
        t.kind = LK_JOHNSON;
        const double lambda = theta ? par(p, 1) : 1.0, delta = par(p, 3);
        consts.push_back(par(p, 0));
        consts.push_back(1.0 / lambda);
        consts.push_back(par(p, 2));
        consts.push_back(delta);
        consts.push_back(delta / (lambda * kSqrt2Pi));
        break;
      }
      case Kind::ArgusBG:
        t.kind = LK_ARGUS;
        consts.push_back(par(p, 0));
        consts.push_back(par(p, 1));
        consts.push_back(par(p, 2));
        consts.push_back(theta ? 1.0 / par(p, 0) : 0.0);  // hoisted reciprocal of m0
        consts.push_back(0.0);  // launch-constant cache flag (kernels.cu cache_launch_constants)
        break;
      case Kind::Chebychev: {
        t.kind = LK_CHEB;
        t.order = static_cast<int>(p.params.size());
        const Observable& o = m.observables[p.obs];
        consts.push_back(o.lo + o.hi);
        consts.push_back(1.0 / (o.hi - o.lo));
        for (int k = 0; k < t.order; ++k) consts.push_back(par(p, k));
        break;
      }
      case Kind::Polynomial:
        t.kind = LK_POLY;
        t.order = static_cast<int>(p.params.size());
        for (int k = 0; k < t.order; ++k) consts.push_back(par(p, k));
        break;
      case Kind::Expression: {  // device program: variables -> the event value or the row
        t.kind = LK_EXPR;
        if (p.program->max_depth > kExprMaxDepth) {
          usage_error("Expression '" + p.name + "' needs a stack of " + std::to_string(p.program->max_depth) +
                      "; the device interpreter holds " + std::to_string(kExprMaxDepth));
        }
        t.order = static_cast<int>(programs.size());
        for (ExprInstr in : p.program->code) {
          if (in.op == EX_VAR) {
            if (p.expr_vars[in.slot] < 0) in.op = EX_X;
          }
          programs.push_back(in);
        }
        programs.push_back(ExprInstr{EX_END, 0, 0.0});
        for (const int v : p.expr_vars) consts.push_back(v < 0 || !theta ? 0.0 : theta[v]);
        break;
      }
      default:
        usage_error("internal: not a leaf");
    }
    terms.push_back(t);
    term_pdf.push_back(id);
  }

  // scale * unnorm(pdf) for a one-dimensional pdf, as a flat sum of leaves.
  // WeightedSum: unnorm = sum_i (f_i / N_i) unnorm_i (proj/src/pdfs.cpp:234-257).
  void sum(int id, double scale) {
    const Pdf& p = m.pdfs[id];
    if (is_leaf(p.kind)) {
      leaf(id, scale);
    } else if (p.kind == Kind::ProdPdf && p.children.size() == 1) {
      sum(p.children[0], scale);
    } else if ((p.kind == Kind::WeightedSum || p.kind == Kind::AddExtended) && p.obs >= 0) {
      const std::vector<double> f = fracs(id);
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const double coef = theta ? f[i] / norm(p.children[i]) : 1.0;
        sum(p.children[i], scale * coef);
      }
    } else {
      usage_error("pdf '" + p.name + "' (" + kind_name(p.kind) +
                  ") nests a product inside a one-dimensional sum; the GPU plan supports "
                  "sum-of-products-of-sums trees");
    }
  }

  void end(int flags) { terms.back().flags |= flags; }

  void factors(int id, std::vector<int>& out) {
    const Pdf& p = m.pdfs[id];
    if (p.kind == Kind::ProdPdf) {
      for (const int c : p.children) factors(c, out);
    } else {
      out.push_back(id);
    }
  }

  // scale * unnorm(ProdPdf) = scale * prod_k unnorm_k (restated ProdPdf).
  void product(int id, double scale) {
    std::vector<int> fs;
    factors(id, fs);
    for (std::size_t k = 0; k < fs.size(); ++k) {
      sum(fs[k], k == 0 ? scale : 1.0);
      end(TF_END_SUM);
    }
  }

  void root(int id, double scale) {
    const Pdf& p = m.pdfs[id];
    if (p.kind == Kind::ProdPdf) {
      product(id, scale);
      end(TF_END_PROD);
    } else if (p.obs >= 0) {
      sum(id, scale);
      end(TF_END_SUM | TF_END_PROD);
    } else {  // sum over products on several observables
      const std::vector<double> f = fracs(id);
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const int c = p.children[i];
        const double coef = theta ? f[i] / norm(c) : 1.0;
        if (m.pdfs[c].kind == Kind::ProdPdf) {
          product(c, scale * coef);
        } else {
          sum(c, scale * coef);
          end(TF_END_SUM);
        }
        end(TF_END_PROD);
      }
    }
  }
};

}  // namespace

HostPlan compile_plan(const Model& m, int pdf, bool normalized) {
  Emitter e{m, nullptr, {}, {}, {}, {}, {}};
  e.root(pdf, 1.0);
  if (e.terms.size() > static_cast<std::size_t>(kMaxTerms)) {
    usage_error("model has " + std::to_string(e.terms.size()) + " leaf terms; the GPU plan holds " +
                std::to_string(kMaxTerms));
  }
  if (e.col_obs.size() > static_cast<std::size_t>(kMaxCols)) {
    usage_error("model reads more than " + std::to_string(kMaxCols) + " observables");
  }
  HostPlan hp;
  hp.pdf = pdf;
  hp.normalized = normalized;
  hp.col_obs = e.col_obs;
  hp.term_pdf = e.term_pdf;
  hp.programs = e.programs;
  hp.dev.prog = nullptr;  // the engine points this at its device copy
  hp.dev.nterms = static_cast<int>(e.terms.size());
  hp.dev.ncols = static_cast<int>(e.col_obs.size());
  hp.dev.stride = static_cast<int>(e.consts.size());
  int ends = 0;
  bool first_factor = true;
  for (std::size_t i = 0; i < e.terms.size(); ++i) {
    hp.dev.t[i] = e.terms[i];
    const int f = e.terms[i].flags;
    if (f) ++ends;
    const int prev = i == 0 ? (TF_END_SUM | TF_END_PROD) : e.terms[i - 1].flags;
    if (prev & TF_END_SUM) hp.dev.t[i].flags |= TF_BEGIN_SUM;  // first term of a sum
    if (f & TF_END_SUM) {
      if (first_factor) hp.dev.t[i].flags |= TF_BEGIN_PROD;  // closes a product's first factor
      first_factor = false;
    }
    if (f & TF_END_PROD) first_factor = true;
  }
  hp.dev.simple = ends == 1 ? 1 : 0;
  return hp;
}

void build_constants(const HostPlan& plan, const Model& m, const double* theta, double* row,
                     double extra_scale) {
  for (std::size_t i = 0; i < m.params.size(); ++i) {
    // the device exp assumes finite arguments (fastmath.cuh); the reference's
    // set_value range check excludes NaN / inf the same way (proj/src/graph.cpp:121)
    if (!std::isfinite(theta[i])) {
      numeric_error("non-finite value for parameter '" + m.params[i].name + "'");
    }
  }
  m.check_params(plan.pdf, theta);
  const double scale =
      (plan.normalized ? 1.0 / m.normalization(plan.pdf, theta) : 1.0) * extra_scale;
  Emitter e{m, theta, {}, {}, {}, {}, {}};
  e.root(plan.pdf, scale);
  if (static_cast<int>(e.consts.size()) != plan.dev.stride) usage_error("internal: plan drift");
  for (int i = 0; i < plan.dev.stride; ++i) row[i] = e.consts[i];
}

namespace {

// (value, d/d theta_j) pairs: the coefficient traversal differentiated forward
struct Dual {
  double v, d;
};
Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
Dual operator/(Dual a, Dual b) { return {a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)}; }

// Mirrors Emitter's traversal (same terms in the same order) carrying Duals.
struct CoefGradEmitter {
  const Model& m;
  const double* theta;
  int j;
  std::vector<double> dcoef;

  Dual norm(int pdf) const { return {m.normalization(pdf, theta), m.normalization_grad(pdf, theta, j)}; }
  std::vector<Dual> fracs(int pdf) const {
    const std::vector<double> f = m.fractions(pdf, theta), df = m.fractions_grad(pdf, theta, j);
    std::vector<Dual> r(f.size());
    for (std::size_t i = 0; i < f.size(); ++i) r[i] = {f[i], df[i]};
    return r;
  }
  void sum(int id, Dual scale) {
    const Pdf& p = m.pdfs[id];
    if (is_leaf(p.kind)) {
      dcoef.push_back(scale.d);
    } else if (p.kind == Kind::ProdPdf && p.children.size() == 1) {
      sum(p.children[0], scale);
    } else {
      const std::vector<Dual> f = fracs(id);
      for (std::size_t i = 0; i < p.children.size(); ++i) sum(p.children[i], scale * (f[i] / norm(p.children[i])));
    }
  }
  void factors(int id, std::vector<int>& out) const {
    const Pdf& p = m.pdfs[id];
    if (p.kind == Kind::ProdPdf) {
      for (const int c : p.children) factors(c, out);
    } else {
      out.push_back(id);
    }
  }
  void product(int id, Dual scale) {
    std::vector<int> fs;
    factors(id, fs);
    for (std::size_t k = 0; k < fs.size(); ++k) sum(fs[k], k == 0 ? scale : Dual{1.0, 0.0});
  }
  void root(int id, Dual scale) {
    const Pdf& p = m.pdfs[id];
    if (p.kind == Kind::ProdPdf) {
      product(id, scale);
    } else if (p.obs >= 0) {
      sum(id, scale);
    } else {
      const std::vector<Dual> f = fracs(id);
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const int c = p.children[i];
        const Dual coef = scale * (f[i] / norm(c));
        if (m.pdfs[c].kind == Kind::ProdPdf) {
          product(c, coef);
        } else {
          sum(c, coef);
        }
      }
    }
  }
};

}  // namespace

std::vector<double> coef_derivatives(const HostPlan& plan, const Model& m, const double* theta, int j,
                                     double extra_scale) {
  CoefGradEmitter e{m, theta, j, {}};
  const Dual n = plan.normalized ? Dual{m.normalization(plan.pdf, theta), m.normalization_grad(plan.pdf, theta, j)}
                                 : Dual{1.0, 0.0};
  e.root(plan.pdf, Dual{extra_scale, 0.0} / n);
  if (static_cast<int>(e.dcoef.size()) != plan.dev.nterms) usage_error("internal: gradient plan drift");
  return e.dcoef;
}

GradPlan compile_grad_plan(const HostPlan& plan, const Model& m) {
  GradPlan gp;
  const DevPlan& d = plan.dev;
  int slot = 1, nseed = 0;
  gp.slot_param.assign(1, -1);
  int factor = 0, fbeg = 0;
  for (int i = 0; i < d.nterms; ++i) {
    DevGradTerm& g = gp.dev.g[i];
    g.slot = slot++;
    gp.slot_param.push_back(-1);
    gp.a_slot.push_back(g.slot);
    const Pdf& leaf = m.pdfs[plan.term_pdf[i]];
    for (std::size_t k = 0; k < leaf.params.size(); ++k) {
      if (m.params[leaf.params[k]].constant) continue;
      g.pmask |= 1 << k;
      gp.slot_param.push_back(leaf.params[k]);
      ++slot;
    }
    if (d.t[i].kind == LK_EXPR) {  // one seed (variable-slot mask) per differentiated parameter
      g.seeds = nseed;
      for (std::size_t k = 0; k < leaf.params.size(); ++k) {
        if (m.params[leaf.params[k]].constant) continue;
        int mask = 0;
        for (std::size_t s = 0; s < leaf.expr_vars.size(); ++s) {
          if (leaf.expr_vars[s] == leaf.params[k]) mask |= 1 << s;
        }
        if (nseed < kMaxGradSlots) gp.dev.seed[nseed] = mask;
        ++nseed;
      }
    }
    g.factor = factor;
    g.fbeg = fbeg;
    if (d.t[i].flags & TF_END_SUM) ++factor;
    if (d.t[i].flags & TF_END_PROD) {
      // close the product: every term since fbeg's first term gets fend
      for (int j = i; j >= 0 && gp.dev.g[j].fbeg == fbeg && gp.dev.g[j].fend == 0; --j) {
        gp.dev.g[j].fend = factor;
      }
      fbeg = factor;
    }
  }
  gp.dev.nslots = slot;
  gp.dev.nfactors = factor;
  int max_vars = 0;
  for (int i = 0; i < d.nterms; ++i) {
    if (d.t[i].kind == LK_EXPR) {
      max_vars = std::max(max_vars, static_cast<int>(m.pdfs[plan.term_pdf[i]].expr_vars.size()));
    }
  }
  if (nseed > kMaxGradSlots || max_vars > 30) {
    gp.why = "Expression gradients: more than " + std::to_string(kMaxGradSlots) +
             " differentiated formula parameters or 30 formula variables";
  } else if (slot > kMaxGradSlots) {
    gp.why = "gradient layout needs " + std::to_string(slot) + " accumulators; the device pass holds " +
             std::to_string(kMaxGradSlots);
  } else if (factor > kMaxFactors) {
    gp.why = "more than " + std::to_string(kMaxFactors) + " factors";
  } else if (!plan.normalized) {
    gp.why = "not a likelihood plan";
  } else {
    gp.ok = true;
  }
  return gp;
}

}  // namespace ffb
