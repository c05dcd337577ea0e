// Host-side model: parser, validation, normalisation integrals.
// See model.hpp for the reference interfaces each piece mirrors.
//
// Transcribed blocks (the model-file grammar and its error strings are the interface; the
// parser is outside the hot path):
//   to_double, tokenize, parse_call     proj/src/model.cpp:34-110
//   Model::parse directive loop         proj/src/model.cpp:112-252 (extended with the GPU
//                                       path's kinds: ArgusBG, Chebychev, Polynomial, ProdPdf,
//                                       extended AddPdf, several observables -- new code)
//   check_params messages / codes       proj/src/pdfs.cpp:127-176
#include "model.hpp"

#include <charconv>
#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <sstream>

namespace ffb {

namespace {

constexpr double kSqrt2Pi = 2.5066282746310005024;

const double* P(const double* theta, const Pdf& p, int k) { return &theta[p.params[k]]; }

[[noreturn]] void parse_fail(const std::string& origin, std::size_t line, const std::string& what) {
  throw Error(ErrorCode::Data, origin + ":" + std::to_string(line) + ": " + what);
}

double to_double(const std::string& tok, const std::string& origin, std::size_t line) {
  double v = 0.0;
  const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc() || ptr != tok.data() + tok.size()) {
    parse_fail(origin, line, "expected a number, got '" + tok + "'");
  }
  return v;
}

std::vector<std::string> tokenize(const std::string& line) {
  std::vector<std::string> out;
  std::istringstream is(line);
  std::string tok;
  while (is >> tok) out.push_back(tok);
  return out;
}

struct Call {
  std::string kind;
  std::vector<std::string> args;
};

// "Kind(a, b, ...)"; a quoted first argument is kept whole (Expression syntax,
// proj/src/model.cpp:68-109) only so that it can be rejected with a clear message.
Call parse_call(const std::string& text, const std::string& origin, std::size_t line) {
  const std::size_t open = text.find('(');
  if (open == std::string::npos || text.empty() || text.back() != ')') {
    parse_fail(origin, line, "expected <Kind>(<args>) in pdf definition");
  }
  Call c;
  c.kind = text.substr(0, open);
  const std::string inner = text.substr(open + 1, text.size() - open - 2);
  std::size_t pos = 0;
  while (pos < inner.size()) {
    while (pos < inner.size() && (inner[pos] == ' ' || inner[pos] == '\t')) ++pos;
    if (pos >= inner.size()) break;
    std::string arg;
    if (inner[pos] == '"') {
      const std::size_t close = inner.find('"', pos + 1);
      if (close == std::string::npos) parse_fail(origin, line, "unterminated string");
      arg = inner.substr(pos + 1, close - pos - 1);
      pos = close + 1;
    } else {
      std::size_t end = inner.find(',', pos);
      if (end == std::string::npos) end = inner.size();
      arg = inner.substr(pos, end - pos);
      while (!arg.empty() && (arg.back() == ' ' || arg.back() == '\t')) arg.pop_back();
      pos = end;
    }
    c.args.push_back(arg);
    while (pos < inner.size() && (inner[pos] == ' ' || inner[pos] == '\t')) ++pos;
    if (pos < inner.size()) {
      if (inner[pos] != ',') parse_fail(origin, line, "expected ',' between arguments");
      ++pos;
    }
  }
  return c;
}

// G(t) = int_0^t sqrt(s) e^{c s} ds  (ArgusBG p = 1/2 after x dx = -(m0^2/2) dt)
double argus_G(double c, double t) {
  if (t <= 0.0) return 0.0;
  if (c < 0.0 && -c * t >= 1.0) {
    const double k = -c;
    const double y = k * t;
    const double sy = std::sqrt(y);
    const double g = 0.88622692545275801365 * std::erf(sy) - sy * std::exp(-y);
    return g / (k * std::sqrt(k));
  }
  const double ct = c * t;
  double term = 1.0, sum = 0.0;
  for (int n = 0; n < 400; ++n) {
    const double add = term / (n + 1.5);
    sum += add;
    if (std::fabs(add) <= 1e-17 * std::fabs(sum)) break;
    term *= ct / (n + 1);
  }
  return t * std::sqrt(t) * sum;
}

}  // namespace

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Gaussian: return "Gaussian";
    case Kind::Exponential: return "Exponential";
    case Kind::ChiSquare: return "ChiSquare";
    case Kind::JohnsonSU: return "JohnsonSU";
    case Kind::WeightedSum: return "WeightedSum";
    case Kind::AddExtended: return "AddPdf(extended)";
    case Kind::ArgusBG: return "ArgusBG";
    case Kind::Chebychev: return "Chebychev";
    case Kind::Polynomial: return "Polynomial";
    case Kind::ProdPdf: return "ProdPdf";
    case Kind::Expression: return "Expression";
  }
  return "?";
}

bool is_leaf(Kind k) {
  return k != Kind::WeightedSum && k != Kind::AddExtended && k != Kind::ProdPdf;
}

int Model::param_index(const std::string& name) const {
  for (std::size_t i = 0; i < params.size(); ++i) {
    if (params[i].name == name) return static_cast<int>(i);
  }
  return -1;
}

int Model::pdf_index(const std::string& name) const {
  for (std::size_t i = 0; i < pdfs.size(); ++i) {
    if (pdfs[i].name == name) return static_cast<int>(i);
  }
  return -1;
}

std::vector<double> Model::theta() const {
  std::vector<double> t(params.size());
  for (std::size_t i = 0; i < params.size(); ++i) t[i] = params[i].value;
  return t;
}

std::vector<int> Model::free_parameters() const {
  std::vector<int> out;
  for (std::size_t i = 0; i < params.size(); ++i) {
    if (!params[i].constant) out.push_back(static_cast<int>(i));
  }
  return out;
}

void Model::set_value(int id, double v) {
  if (id < 0 || id >= static_cast<int>(params.size())) usage_error("invalid parameter index");
  Parameter& p = params[id];
  if (p.constant) usage_error("set_value: parameter '" + p.name + "' is constant");
  if (!(p.lo <= v && v <= p.hi)) {
    numeric_error("set_value: " + std::to_string(v) + " outside range of '" + p.name + "'");
  }
  p.value = v;
}

// ---------------------------------------------------------------------------
// parser: proj/src/model.cpp:113-252 grammar + GPU-path extensions

std::unique_ptr<Model> Model::parse(const std::string& text, const std::string& origin) {
  auto m = std::make_unique<Model>();
  std::map<std::string, int> names;  // every declared name (observables, params, pdfs)
  std::istringstream in(text);
  std::string line;
  std::size_t line_no = 0;

  auto obs_id = [&](const std::string& n) -> int {
    for (std::size_t i = 0; i < m->observables.size(); ++i) {
      if (m->observables[i].name == n) return static_cast<int>(i);
    }
    return -1;
  };
  auto param_id = [&](const std::string& n) -> int {
    const int id = m->param_index(n);
    if (id < 0) {
      if (names.count(n)) parse_fail(origin, line_no, "'" + n + "' is not a parameter");
      parse_fail(origin, line_no, "undeclared name: " + n);
    }
    return id;
  };
  auto pdf_id = [&](const std::string& n) -> int {
    const int id = m->pdf_index(n);
    if (id < 0) parse_fail(origin, line_no, "undeclared pdf: " + n);
    return id;
  };
  auto declare = [&](const std::string& n) {
    if (names.count(n)) usage_error("duplicate node name: " + n);
    names[n] = 1;
  };

  while (std::getline(in, line)) {
    ++line_no;
    const std::size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    const std::vector<std::string> toks = tokenize(line);
    if (toks.empty()) continue;

    if (toks[0] == "observable") {
      if (toks.size() != 4) parse_fail(origin, line_no, "observable <name> <lo> <hi>");
      Observable o{toks[1], to_double(toks[2], origin, line_no), to_double(toks[3], origin, line_no)};
      if (!(o.lo < o.hi)) usage_error("observable '" + o.name + "': lower must be < upper");
      declare(o.name);
      m->observables.push_back(o);
    } else if (toks[0] == "parameter") {
      if (toks.size() != 5 && !(toks.size() == 6 && toks[5] == "const")) {
        parse_fail(origin, line_no, "parameter <name> <value> <lo> <hi> [const]");
      }
      Parameter p;
      p.name = toks[1];
      p.value = to_double(toks[2], origin, line_no);
      p.lo = to_double(toks[3], origin, line_no);
      p.hi = to_double(toks[4], origin, line_no);
      p.constant = toks.size() == 6;
      if (!(p.lo <= p.value && p.value <= p.hi)) {
        usage_error("parameter '" + p.name + "': value outside range");
      }
      if (!(p.lo < p.hi) && !p.constant) usage_error("parameter '" + p.name + "': empty range");
      declare(p.name);
      m->params.push_back(p);
    } else if (toks[0] == "pdf") {
      if (toks.size() < 3) parse_fail(origin, line_no, "pdf <name> <Kind>(<args>)");
      if (m->observables.empty()) {
        parse_fail(origin, line_no, "observable must be declared before pdfs");
      }
      std::string rest = toks[2];
      for (std::size_t i = 3; i < toks.size(); ++i) rest += " " + toks[i];
      const Call call = parse_call(rest, origin, line_no);
      Pdf pdf;
      pdf.name = toks[1];

      auto expect_args = [&](std::size_t lo, std::size_t hi) {
        if (call.args.size() < lo || call.args.size() > hi) {
          parse_fail(origin, line_no, call.kind + " expects " + std::to_string(lo) +
                                          (hi != lo ? "+" : "") + " argument(s), got " +
                                          std::to_string(call.args.size()));
        }
      };
      auto leaf = [&](Kind k, std::size_t nparams_lo, std::size_t nparams_hi) {
        expect_args(1 + nparams_lo, 1 + nparams_hi);
        pdf.kind = k;
        pdf.obs = call.args.empty() ? -1 : obs_id(call.args[0]);
        if (pdf.obs < 0) {
          parse_fail(origin, line_no, call.kind + ": first argument must be an observable");
        }
        for (std::size_t i = 1; i < call.args.size(); ++i) pdf.params.push_back(param_id(call.args[i]));
      };

      if (call.kind == "Gaussian") {
        leaf(Kind::Gaussian, 2, 2);
      } else if (call.kind == "Exponential") {
        leaf(Kind::Exponential, 1, 1);
      } else if (call.kind == "ChiSquare") {
        leaf(Kind::ChiSquare, 1, 1);
      } else if (call.kind == "JohnsonSU") {
        leaf(Kind::JohnsonSU, 4, 4);
      } else if (call.kind == "ArgusBG") {
        leaf(Kind::ArgusBG, 3, 3);
      } else if (call.kind == "Chebychev") {
        leaf(Kind::Chebychev, 0, 12);
      } else if (call.kind == "Polynomial") {
        leaf(Kind::Polynomial, 0, 12);
      } else if (call.kind == "WeightedSum" || call.kind == "AddPdf") {
        // WeightedSum(c1, f1, ..., cn): n-1 fractions (proj/src/model.cpp:190-209);
        // AddPdf(c1, y1, ..., cn, yn): n yields -> extended likelihood.
        const std::size_t na = call.args.size();
        const bool extended = call.kind == "AddPdf" && na % 2 == 0;
        if (na < 2 || (!extended && (na < 3 || na % 2 == 0))) {
          parse_fail(origin, line_no, call.kind + "(c1, f1, c2, f2, ..., cn)" +
                                          (call.kind == "AddPdf" ? " or AddPdf(c1, y1, ..., cn, yn)" : ""));
        }
        pdf.kind = extended ? Kind::AddExtended : Kind::WeightedSum;
        for (std::size_t i = 0; i < na; ++i) {
          if (i % 2 == 0) pdf.children.push_back(pdf_id(call.args[i]));
          else pdf.params.push_back(param_id(call.args[i]));
        }
        if (pdf.children.size() > 16) parse_fail(origin, line_no, "at most 16 components");
        int obs = m->pdfs[pdf.children[0]].obs;
        for (const int c : pdf.children) {
          if (m->pdfs[c].kind == Kind::AddExtended) {
            parse_fail(origin, line_no, "an extended AddPdf can only be the model itself");
          }
          if (m->pdfs[c].obs != obs) obs = -1;  // multi-observable sum (of products)
        }
        pdf.obs = obs;
      } else if (call.kind == "ProdPdf") {
        if (call.args.empty()) parse_fail(origin, line_no, "ProdPdf(p1, p2, ...)");
        pdf.kind = Kind::ProdPdf;
        std::vector<int> seen;
        std::function<void(int)> collect = [&](int id) {
          const Pdf& c = m->pdfs[id];
          if (c.kind == Kind::ProdPdf) {
            for (const int cc : c.children) collect(cc);
            return;
          }
          if (c.kind == Kind::AddExtended) {
            parse_fail(origin, line_no, "an extended AddPdf can only be the model itself");
          }
          if (c.obs < 0) parse_fail(origin, line_no, "ProdPdf factors must be one-dimensional");
          for (const int s : seen) {
            if (s == c.obs) {
              parse_fail(origin, line_no,
                         "ProdPdf factors must depend on distinct observables ('" +
                             m->observables[c.obs].name + "' repeats)");
            }
          }
          seen.push_back(c.obs);
        };
        for (const std::string& a : call.args) {
          const int id = pdf_id(a);
          pdf.children.push_back(id);
          collect(id);
        }
        pdf.obs = pdf.children.size() == 1 ? m->pdfs[pdf.children[0]].obs : -1;
      } else if (call.kind == "Expression") {
        // Expression("<formula>", v1, ..., vk) (proj/src/model.cpp:218-232): the variables
        // are the observable and parameters the formula may use, in program-slot order
        if (call.args.empty()) parse_fail(origin, line_no, "Expression(\"<formula>\", <var>, ...)");
        pdf.kind = Kind::Expression;
        std::vector<std::string> vars(call.args.begin() + 1, call.args.end());
        for (const std::string& v : vars) {
          const int o = obs_id(v);
          if (o >= 0) {
            if (pdf.obs >= 0 && pdf.obs != o) {
              parse_fail(origin, line_no, "an Expression pdf depends on one observable");
            }
            pdf.obs = o;
            pdf.expr_vars.push_back(-1);
            continue;
          }
          if (!names.count(v)) parse_fail(origin, line_no, "undeclared name: " + v);
          const int k = param_id(v);
          pdf.expr_vars.push_back(k);
          if (std::find(pdf.params.begin(), pdf.params.end(), k) == pdf.params.end()) pdf.params.push_back(k);
        }
        if (pdf.obs < 0) {
          if (m->observables.size() != 1) {
            parse_fail(origin, line_no, "an Expression pdf must name its observable");
          }
          pdf.obs = 0;  // the reference's single model observable
        }
        try {
          pdf.program = std::make_shared<const ExprProgram>(compile_expression(call.args[0], vars));
        } catch (const Error& e) {
          parse_fail(origin, line_no, e.what());
        }
      } else {
        parse_fail(origin, line_no, "unknown pdf kind: " + call.kind);
      }
      declare(pdf.name);
      m->pdfs.push_back(pdf);
      m->root = static_cast<int>(m->pdfs.size()) - 1;
    } else {
      parse_fail(origin, line_no, "unknown directive: " + toks[0]);
    }
  }
  if (m->observables.empty()) throw Error(ErrorCode::Data, origin + ": no observable declared");
  if (m->root < 0) throw Error(ErrorCode::Data, origin + ": no pdf declared");
  return m;
}

// ---------------------------------------------------------------------------

void Model::check_params(int id, const double* theta) const {
  const Pdf& p = pdfs[id];
  auto issue = [&](int param, const char* what) {
    numeric_error("invalid parameters for '" + p.name + "': " + params[param].name + ": " + what);
  };
  switch (p.kind) {
    case Kind::Gaussian:
      if (!(theta[p.params[1]] > 0.0)) issue(p.params[1], "sigma must be > 0");
      break;
    case Kind::ChiSquare:
      if (!(theta[p.params[0]] > 0.0)) issue(p.params[0], "k must be > 0");
      break;
    case Kind::JohnsonSU:
      if (!(theta[p.params[1]] > 0.0)) issue(p.params[1], "lambda must be > 0");
      if (!(theta[p.params[3]] > 0.0)) issue(p.params[3], "delta must be > 0");
      break;
    case Kind::ArgusBG:
      if (!(theta[p.params[0]] > 0.0)) issue(p.params[0], "m0 must be > 0");
      if (!(theta[p.params[2]] >= 0.0)) issue(p.params[2], "p must be >= 0");
      break;
    case Kind::WeightedSum: {
      double sum = 0.0;
      for (const int f : p.params) {
        sum += theta[f];
        if (!(theta[f] >= 0.0 && theta[f] <= 1.0)) issue(f, "fraction must be in [0, 1]");
      }
      if (sum > 1.0) numeric_error("invalid parameters for '" + p.name + "': " + p.name +
                                   ": fractions sum to more than 1");
      break;
    }
    case Kind::AddExtended: {
      double nu = 0.0;
      for (const int y : p.params) {
        if (!(theta[y] >= 0.0)) issue(y, "yield must be >= 0");
        nu += theta[y];
      }
      if (!(nu > 0.0)) numeric_error("invalid parameters for '" + p.name + "': total yield must be > 0");
      break;
    }
    default:
      break;
  }
  for (const int c : p.children) check_params(c, theta);
}

std::vector<double> Model::fractions(int id, const double* theta) const {
  const Pdf& p = pdfs[id];
  std::vector<double> f;
  if (p.kind == Kind::WeightedSum) {
    double sum = 0.0;
    for (const int k : p.params) {
      f.push_back(theta[k]);
      sum += f.back();
    }
    f.push_back(1.0 - sum);
  } else {
    double nu = 0.0;
    for (const int k : p.params) nu += theta[k];
    for (const int k : p.params) f.push_back(theta[k] / nu);
  }
  return f;
}

double Model::extended_term(const double* theta, double n) const {
  if (!extended()) return 0.0;
  double nu = 0.0;
  for (const int k : pdfs[root].params) nu += theta[k];
  return nu - n * std::log(nu);
}

std::optional<double> Model::analytic_integral(int id, double lo, double hi,
                                               const double* theta) const {
  if (!(lo < hi)) usage_error("analytic_integral: invalid range");
  const Pdf& p = pdfs[id];
  switch (p.kind) {
    case Kind::Gaussian: {  // proj/src/pdfs.cpp:276-282
      const double mu = *P(theta, p, 0), sigma = *P(theta, p, 1);
      const double inv = 1.0 / (sigma * std::sqrt(2.0));
      return sigma * std::sqrt(std::atan(1.0) * 2.0) *
             (std::erf((hi - mu) * inv) - std::erf((lo - mu) * inv));
    }
    case Kind::Exponential: {  // proj/src/pdfs.cpp:283-287
      const double c = *P(theta, p, 0);
      if (std::fabs(c) < 1e-12) return hi - lo;
      return (std::exp(c * hi) - std::exp(c * lo)) / c;
    }
    case Kind::ArgusBG: {  // closed form for p = 1/2 (restated; pinned by tests/golden/argus_mp.json)
      const double m0 = *P(theta, p, 0), c = *P(theta, p, 1), pw = *P(theta, p, 2);
      if (pw != 0.5 || !(m0 > 0.0)) return std::nullopt;
      const double a = lo > 0.0 ? lo : 0.0;
      const double b = hi < m0 ? hi : m0;
      if (!(a < b)) return 0.0;
      // t = 1 - (x/m0)^2 = (m0-x)(m0+x)/m0^2, written without the cancellation
      const double ta = ((m0 - a) * (m0 + a)) / (m0 * m0);
      const double tb = ((m0 - b) * (m0 + b)) / (m0 * m0);
      return 0.5 * m0 * m0 * (argus_G(c, ta) - argus_G(c, tb));
    }
    case Kind::Chebychev: {  // full range: (hi-lo)/2 (2 + sum_{k even} a_k 2/(1-k^2))
      const Observable& o = observables[p.obs];
      if (lo != o.lo || hi != o.hi) return std::nullopt;
      double s = 2.0;
      for (std::size_t k = 1; k <= p.params.size(); ++k) {
        if (k % 2 == 0) {
          s += theta[p.params[k - 1]] * (2.0 / (1.0 - static_cast<double>(k) * static_cast<double>(k)));
        }
      }
      return 0.5 * (hi - lo) * s;
    }
    case Kind::Polynomial: {
      double s = hi - lo;
      double hk = hi, lk = lo;
      for (std::size_t k = 1; k <= p.params.size(); ++k) {
        hk *= hi;
        lk *= lo;
        s += theta[p.params[k - 1]] * (hk - lk) / static_cast<double>(k + 1);
      }
      return s;
    }
    case Kind::WeightedSum:
    case Kind::AddExtended: {  // proj/src/pdfs.cpp:288-300
      const std::vector<double> f = fractions(id, theta);
      double acc = 0.0;
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const int c = p.children[i];
        std::optional<double> part, norm;
        if (pdfs[c].kind == Kind::ProdPdf) {
          part = norm = normalization(c, theta);
        } else {
          const Observable& o = obs_of(c);
          part = analytic_integral(c, lo, hi, theta);
          if (!part) return std::nullopt;
          norm = analytic_integral(c, o.lo, o.hi, theta);
        }
        acc += f[i] * *part / *norm;
      }
      return acc;
    }
    case Kind::ProdPdf:
      return normalization(id, theta);
    case Kind::ChiSquare:
    case Kind::JohnsonSU:
    case Kind::Expression:
      return std::nullopt;
  }
  return std::nullopt;
}

double Model::eval_unnorm_1d(int id, const double* theta, double x) const {
  const Pdf& p = pdfs[id];
  switch (p.kind) {
    case Kind::Gaussian: {
      const double mu = *P(theta, p, 0), sigma = *P(theta, p, 1);
      const double k = -1.0 / (2.0 * sigma * sigma);
      const double d = x - mu;
      return std::exp(d * d * k);
    }
    case Kind::Exponential:
      return std::exp(*P(theta, p, 0) * x);
    case Kind::ChiSquare: {
      const double k = *P(theta, p, 0);
      const double half_k_m1 = 0.5 * k - 1.0;
      const double at_zero = k == 2.0 ? 1.0 : 0.0;
      const double xa = x > 0.0 ? x : 1.0;
      const double v = std::exp(half_k_m1 * std::log(xa) - 0.5 * xa);
      const double pos = x > 0.0 ? 1.0 : 0.0;
      const double zero = x == 0.0 ? 1.0 : 0.0;
      return pos * v + (1.0 - pos) * (zero * at_zero);
    }
    case Kind::JohnsonSU: {
      const double mu = *P(theta, p, 0), lambda = *P(theta, p, 1), gamma = *P(theta, p, 2),
                   delta = *P(theta, p, 3);
      const double inv_lambda = 1.0 / lambda;
      const double coef = delta / (lambda * kSqrt2Pi);
      const double z = (x - mu) * inv_lambda;
      const double as = std::copysign(std::log(std::fabs(z) + std::sqrt(z * z + 1.0)), z);
      const double t = gamma + delta * as;
      return coef / std::sqrt(1.0 + z * z) * std::exp(-0.5 * t * t);
    }
    case Kind::ArgusBG: {
      const double m0 = *P(theta, p, 0), c = *P(theta, p, 1), pw = *P(theta, p, 2);
      const double r = x / m0;
      const double t = 1.0 - r * r;
      if (!(t > 0.0)) return 0.0;
      const double w = pw == 0.5 ? std::sqrt(t) : std::pow(t, pw);
      return x * w * std::exp(c * t);
    }
    case Kind::Chebychev: {
      const Observable& o = observables[p.obs];
      const double z = (2.0 * x - (o.lo + o.hi)) / (o.hi - o.lo);
      double acc = 1.0, tm1 = 1.0, tk = z;
      for (const int a : p.params) {
        acc += theta[a] * tk;
        const double tn = 2.0 * z * tk - tm1;
        tm1 = tk;
        tk = tn;
      }
      return acc;
    }
    case Kind::Polynomial: {
      double acc = 1.0, xk = x;
      for (const int a : p.params) {
        acc += theta[a] * xk;
        xk *= x;
      }
      return acc;
    }
    case Kind::WeightedSum:
    case Kind::AddExtended: {
      if (p.obs < 0) usage_error("eval_unnorm_1d: multi-observable sum");
      const std::vector<double> f = fractions(id, theta);
      double acc = 0.0;
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        const double coef = f[i] / normalization(p.children[i], theta);
        acc += coef * eval_unnorm_1d(p.children[i], theta, x);
      }
      return acc;
    }
    case Kind::ProdPdf:
      if (p.children.size() == 1) return eval_unnorm_1d(p.children[0], theta, x);
      usage_error("eval_unnorm_1d: multi-observable ProdPdf");
    case Kind::Expression: {  // PdfSpec::eval_unnorm, proj/src/pdfs.cpp:200-207
      double small[16];
      std::vector<double> big;
      double* v = small;
      if (p.expr_vars.size() > 16) {
        big.resize(p.expr_vars.size());
        v = big.data();
      }
      for (std::size_t i = 0; i < p.expr_vars.size(); ++i) v[i] = p.expr_vars[i] < 0 ? x : theta[p.expr_vars[i]];
      return p.program->eval(v);
    }
  }
  return 0.0;
}

double Model::simpson_integral(int id, const double* theta) const {
  const Pdf& p = pdfs[id];
  if (p.obs < 0) usage_error("numeric normalisation needs a one-dimensional pdf");
  const Observable& o = observables[p.obs];
  // Same integrand values as PdfSpec::eval_unnorm (the sum coefficients are
  // deterministic per point, so they are computed once instead of per sample).
  std::function<double(double)> f;
  if (p.kind == Kind::WeightedSum || p.kind == Kind::AddExtended) {
    const std::vector<double> fr = fractions(id, theta);
    std::vector<double> coef(p.children.size());
    for (std::size_t i = 0; i < p.children.size(); ++i) {
      coef[i] = fr[i] / normalization(p.children[i], theta);
    }
    f = [this, &p, coef, theta](double x) {
      double acc = 0.0;
      for (std::size_t i = 0; i < p.children.size(); ++i) {
        acc += coef[i] * eval_unnorm_1d(p.children[i], theta, x);
      }
      return acc;
    };
  } else {
    f = [this, id, theta](double x) { return eval_unnorm_1d(id, theta, x); };
  }
  return integrate_adaptive_simpson(f, o.lo, o.hi, 1e-10 * (o.hi - o.lo), 1e-10, 60);
}

namespace {
thread_local const double* tl_norm_override = nullptr;
}

NormOverride::NormOverride(const double* values) : prev_(tl_norm_override) { tl_norm_override = values; }
NormOverride::~NormOverride() { tl_norm_override = prev_; }

std::vector<int> Model::simpson_nodes(int id, const double* theta) const {
  std::vector<int> out;
  std::function<void(int)> walk = [&](int n) {
    const Pdf& p = pdfs[n];
    for (const int c : p.children) walk(c);
    if (p.kind == Kind::ProdPdf || p.obs < 0) return;
    const Observable& o = observables[p.obs];
    if (!analytic_integral(n, o.lo, o.hi, theta) && std::find(out.begin(), out.end(), n) == out.end()) {
      out.push_back(n);
    }
  };
  walk(id);
  return out;
}

double Model::normalization(int id, const double* theta) const {
  const Pdf& p = pdfs[id];
  double r;
  if (tl_norm_override && !std::isnan(tl_norm_override[id])) {
    r = tl_norm_override[id];
  } else if (p.kind == Kind::ProdPdf) {
    r = 1.0;
    for (const int c : p.children) r *= normalization(c, theta);
  } else if (p.obs < 0) {
    // sum over products on different observables: sum f_i N_i / N_i
    const std::vector<double> f = fractions(id, theta);
    r = 0.0;
    for (std::size_t i = 0; i < p.children.size(); ++i) {
      const double n = normalization(p.children[i], theta);
      r += f[i] * n / n;
    }
  } else {
    const Observable& o = observables[p.obs];
    const auto a = analytic_integral(id, o.lo, o.hi, theta);
    r = a ? *a : simpson_integral(id, theta);
  }
  if (!(r > 0.0) || !std::isfinite(r)) {
    numeric_error("degenerate PDF '" + p.name + "': normalization integral is " + std::to_string(r));
  }
  return r;
}

double Model::max_hint(int id, const double* theta) const {
  const Observable& o = obs_of(id);
  constexpr int kGrid = 1024;
  double best = 0.0;
  const double step = (o.hi - o.lo) / (kGrid - 1);
  for (int i = 0; i < kGrid; ++i) {
    const double x = i == kGrid - 1 ? o.hi : o.lo + i * step;
    const double v = eval_unnorm_1d(id, theta, x);
    if (v > best) best = v;
  }
  return best * 1.1;
}

namespace {

double simpson_recurse(const std::function<double(double)>& f, double a, double b, double fa,
                       double fm, double fb, double whole, double abs_tol, double rel_tol,
                       int depth) {
  const double m = 0.5 * (a + b);
  const double lm = 0.5 * (a + m);
  const double rm = 0.5 * (m + b);
  const double flm = f(lm);
  const double frm = f(rm);
  if (!std::isfinite(flm)) numeric_error("non-finite integrand at x=" + std::to_string(lm));
  if (!std::isfinite(frm)) numeric_error("non-finite integrand at x=" + std::to_string(rm));
  const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
  const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
  const double delta = left + right - whole;
  if (depth <= 0 || std::fabs(delta) <= 15.0 * std::max(abs_tol, rel_tol * std::fabs(left + right))) {
    return left + right + delta / 15.0;
  }
  return simpson_recurse(f, a, m, fa, flm, fm, left, 0.5 * abs_tol, rel_tol, depth - 1) +
         simpson_recurse(f, m, b, fm, frm, fb, right, 0.5 * abs_tol, rel_tol, depth - 1);
}

}  // namespace

double integrate_adaptive_simpson(const std::function<double(double)>& f, double lo, double hi,
                                  double abs_tol, double rel_tol, int max_depth) {
  if (!(lo < hi)) usage_error("integration range must satisfy lo < hi");
  constexpr int kPanels = 32;
  const double width = (hi - lo) / kPanels;
  double total = 0.0;
  for (int p = 0; p < kPanels; ++p) {
    const double a = lo + p * width;
    const double b = p == kPanels - 1 ? hi : a + width;
    const double m = 0.5 * (a + b);
    const double fa = f(a), fm = f(m), fb = f(b);
    for (const double v : {fa, fm, fb}) {
      if (!std::isfinite(v)) numeric_error("non-finite integrand");
    }
    const double whole = (b - a) / 6.0 * (fa + 4.0 * fm + fb);
    total += simpson_recurse(f, a, b, fa, fm, fb, whole, abs_tol / kPanels, rel_tol, max_depth);
  }
  return total;
}

}  // namespace ffb
