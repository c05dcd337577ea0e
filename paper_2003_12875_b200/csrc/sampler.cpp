// Seeded toy generator (host).  Not on the hot path: it produces the seeded SoA
// inputs every config and test uses.  It reproduces the reference sampler
// bit-for-bit for the kinds the reference has (proj/src/sampling.cpp:9-197:
// xoshiro256++ / splitmix64 Rng, Box-Muller with cached spare, range-rejected
// Gaussian, inverse-CDF Exponential, JohnsonSU, WeightedSum pick-by-fraction,
// accept/reject against max_hint otherwise).  The restated kinds (ArgusBG,
// Chebychev, Polynomial) carry their own accept/reject against their own
// max_hint and count as direct samplers inside a mixture (pick-then-draw); a
// ProdPdf samples factor k from its own stream Rng(seed + 10 k).
#include "sampler.hpp"

#include <cmath>

namespace ffb {

Rng::Rng(std::uint64_t seed) {
  std::uint64_t x = seed;
  for (auto& w : s_) {
    x += 0x9E3779B97f4A7C15ull;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    w = z ^ (z >> 31);
  }
}

std::uint64_t Rng::next() {
  auto rotl = [](std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); };
  const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}

double Rng::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

double Rng::gauss() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * std::atan(1.0) * 4.0 * u2;
  spare_ = r * std::sin(a);
  have_spare_ = true;
  return r * std::cos(a);
}

namespace {

struct Sampler {
  const Model& m;
  const double* theta;
  Rng rng;
  std::vector<double> bound;
  SampleStats stats;

  bool direct(int id) const {
    const Pdf& p = m.pdfs[id];
    switch (p.kind) {
      case Kind::Gaussian: case Kind::Exponential: case Kind::JohnsonSU:
      case Kind::ArgusBG: case Kind::Chebychev: case Kind::Polynomial:
        return true;
      case Kind::WeightedSum: case Kind::AddExtended:
        for (const int c : p.children) {
          if (!direct(c)) return false;
        }
        return p.obs >= 0;
      default:
        return false;
    }
  }

  void prepare(int id) {
    const Pdf& p = m.pdfs[id];
    if (p.kind == Kind::ArgusBG || p.kind == Kind::Chebychev || p.kind == Kind::Polynomial) {
      bound[id] = m.max_hint(id, theta);
    }
    for (const int c : p.children) prepare(c);
  }

  // one accepted draw of accept_reject (proj/src/sampling.cpp:56-88)
  double ar(int id) {
    const Observable& o = m.obs_of(id);
    const double b = bound[id];
    for (;;) {
      const double x = o.lo + (o.hi - o.lo) * rng.uniform();
      const double p = m.eval_unnorm_1d(id, theta, x);
      ++stats.proposed;
      if (p > b) {
        numeric_error("accept/reject: pdf(" + std::to_string(x) + ") = " + std::to_string(p) +
                      " exceeds envelope bound " + std::to_string(b));
      }
      if (rng.uniform() * b < p) {
        ++stats.accepted;
        return x;
      }
      if (stats.proposed >= 1000000ull &&
          static_cast<double>(stats.accepted) / static_cast<double>(stats.proposed) < 1e-6) {
        numeric_error("accept/reject: acceptance rate below 1e-6, pathological envelope");
      }
    }
  }

  // draw_direct (proj/src/sampling.cpp:96-168)
  double draw(int id) {
    const Pdf& p = m.pdfs[id];
    const Observable& o = m.obs_of(id);
    switch (p.kind) {
      case Kind::Gaussian: {
        const double mu = theta[p.params[0]], sigma = theta[p.params[1]];
        for (;;) {
          const double x = mu + sigma * rng.gauss();
          if (x >= o.lo && x <= o.hi) return x;
        }
      }
      case Kind::Exponential: {
        const double c = theta[p.params[0]];
        const double u = rng.uniform();
        if (std::fabs(c) < 1e-12) return o.lo + u * (o.hi - o.lo);
        return o.lo + std::log1p(u * std::expm1(c * (o.hi - o.lo))) / c;
      }
      case Kind::JohnsonSU: {
        const double mu = theta[p.params[0]], lambda = theta[p.params[1]],
                     gamma = theta[p.params[2]], delta = theta[p.params[3]];
        for (;;) {
          const double z = rng.gauss();
          const double x = mu + lambda * std::sinh((z - gamma) / delta);
          if (x >= o.lo && x <= o.hi) return x;
        }
      }
      case Kind::WeightedSum:
      case Kind::AddExtended: {
        const std::vector<double> f = m.fractions(id, theta);
        double sum = 0.0;
        std::vector<double> cum;
        for (std::size_t i = 0; i + 1 < p.children.size(); ++i) {
          sum += f[i];
          cum.push_back(sum);
        }
        const double u = rng.uniform();
        std::size_t pick = p.children.size() - 1;
        for (std::size_t i = 0; i < cum.size(); ++i) {
          if (u < cum[i]) {
            pick = i;
            break;
          }
        }
        return draw(p.children[pick]);
      }
      default:
        return ar(id);
    }
  }
};

void sample_1d(const Model& m, int id, const double* theta, long long n, std::uint64_t seed,
               double* out, SampleStats& stats) {
  if (m.pdfs[id].obs < 0) usage_error("sampling needs a one-dimensional pdf per factor");
  Sampler s{m, theta, Rng(seed), std::vector<double>(m.pdfs.size(), 0.0), {}};
  if (s.direct(id)) {
    s.prepare(id);
    for (long long i = 0; i < n; ++i) out[i] = s.draw(id);
  } else {
    s.bound[id] = m.max_hint(id, theta);
    if (s.bound[id] == 0.0) {
      numeric_error("cannot sample '" + m.pdfs[id].name + "': pdf is zero over the whole range");
    }
    for (long long i = 0; i < n; ++i) out[i] = s.ar(id);
  }
  stats.proposed += s.stats.proposed;
  stats.accepted += s.stats.accepted;
}

}  // namespace

std::vector<std::vector<double>> sample(const Model& m, long long n, std::uint64_t seed,
                                        SampleStats* stats) {
  if (n < 0) usage_error("sample size must be >= 0");
  const std::vector<double> theta = m.theta();
  m.check_params(m.root, theta.data());
  std::vector<std::vector<double>> cols(m.observables.size());
  SampleStats st;
  const Pdf& root = m.pdfs[m.root];
  if (root.kind == Kind::ProdPdf) {
    std::vector<int> fs;
    std::function<void(int)> flat = [&](int id) {
      if (m.pdfs[id].kind == Kind::ProdPdf) {
        for (const int c : m.pdfs[id].children) flat(c);
      } else {
        fs.push_back(id);
      }
    };
    flat(m.root);
    for (std::size_t k = 0; k < fs.size(); ++k) {
      auto& col = cols[m.pdfs[fs[k]].obs];
      col.resize(static_cast<std::size_t>(n));
      sample_1d(m, fs[k], theta.data(), n, seed + 10ull * k, col.data(), st);
    }
  } else {
    auto& col = cols[root.obs < 0 ? 0 : root.obs];
    col.resize(static_cast<std::size_t>(n));
    sample_1d(m, m.root, theta.data(), n, seed, col.data(), st);
  }
  for (auto& c : cols) c.resize(static_cast<std::size_t>(n), 0.0);
  if (stats) *stats = st;
  return cols;
}

}  // namespace ffb
