#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "model.hpp"

namespace ffb {

// xoshiro256++ seeded through splitmix64 (proj/include/ffit/sampling.hpp:13-31).
class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  std::uint64_t next();
  double uniform();  // [0, 1)
  double gauss();    // Box-Muller, second value cached

 private:
  std::array<std::uint64_t, 4> s_{};
  double spare_ = 0.0;
  bool have_spare_ = false;
};

struct SampleStats {
  unsigned long long proposed = 0;  // accept/reject proposals (0: only direct samplers ran)
  unsigned long long accepted = 0;
};

// n events from the model at its current parameter values; one column per
// model observable (declaration order).
std::vector<std::vector<double>> sample(const Model& m, long long n, std::uint64_t seed,
                                        SampleStats* stats);

}  // namespace ffb
