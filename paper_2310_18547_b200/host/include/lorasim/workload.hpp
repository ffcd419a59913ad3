// lorasim/workload.hpp -- B200 drop-in, the batch-composition part of the
// reference's workload generators (proj/core/include/lorasim/workload.hpp):
// the seeded RNG, stream splitting and the Distinct / Uniform / Skewed /
// Identical adapter assignment that decides the SGMV segment layout.  Arrival
// processes and length tables (serving traffic) are out of scope.
#pragma once

#include <cstdint>
#include <random>
#include <vector>

namespace lorasim {

// mt19937_64 with portable, hand-written distributions (the std:: distribution
// objects are implementation-defined, the engine is not).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}

  std::uint64_t next() { return engine_(); }
  double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53;  }  // 53-bit [0,1)
  double exponential(double rate);
  std::uint64_t uniform_index(std::uint64_t n);  // exact uniform in [0, n)
  int uniform_int(int lo, int hi);               // inclusive
  std::size_t discrete(const std::vector<double>& cumulative, double total);

  template <typename T>
  void shuffle(std::vector<T>& items) {
    for (std::size_t i = items.size(); i > 1; --i) std::swap(items[i - 1], items[uniform_index(i)]);
  }

 private:
  std::mt19937_64 engine_;
};

std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream);

enum class Popularity { Distinct, Uniform, Skewed, Identical };

int model_count_for(int n, Popularity popularity);
std::vector<std::int64_t> assign_models(int n, Popularity popularity, double alpha, std::uint64_t seed);
const char* to_string(Popularity p);

}  // namespace lorasim
