// workload.cpp -- batch-composition generators (reference: workload.cpp:11-44, 92-143).
#include "lorasim/workload.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace lorasim {

double Rng::exponential(double rate) {
  if (rate <= 0.0) throw std::invalid_argument("Rng::exponential: rate must be > 0");
  return -std::log1p(-uniform01()) / rate;
}

std::uint64_t Rng::uniform_index(std::uint64_t n) {
  if (n == 0) throw std::invalid_argument("Rng::uniform_index: n must be > 0");
  // reject the top partial block so that x % n is exactly uniform
  const std::uint64_t bound = UINT64_MAX - UINT64_MAX % n;
  for (;;) {
    const std::uint64_t x = next();
    if (x < bound) return x % n;
  }
}

int Rng::uniform_int(int lo, int hi) {
  if (hi < lo) throw std::invalid_argument("Rng::uniform_int: empty range");
  return lo + static_cast<int>(uniform_index(static_cast<std::uint64_t>(hi - lo) + 1));
}

std::size_t Rng::discrete(const std::vector<double>& cumulative, double total) {
  const double u = uniform01() * total;
  const auto it = std::upper_bound(cumulative.begin(), cumulative.end(), u);
  return it == cumulative.end() ? cumulative.size() - 1 : static_cast<std::size_t>(it - cumulative.begin());
}

std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t z = seed + 0x9E3779B97F4A7C15ull * (stream + 1);  // splitmix64 step + finaliser
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int model_count_for(int n, Popularity popularity) {
  if (n <= 0) return 0;
  if (popularity == Popularity::Distinct) return n;
  if (popularity == Popularity::Identical) return 1;
  return static_cast<int>(std::ceil(std::sqrt(static_cast<double>(n))));
}

std::vector<std::int64_t> assign_models(int n, Popularity popularity, double alpha, std::uint64_t seed) {
  if (n < 0) throw std::invalid_argument("assign_models: negative request count");
  std::vector<std::int64_t> ids(static_cast<std::size_t>(n), 0);
  if (n == 0) return ids;
  Rng rng(seed);
  const int m = model_count_for(n, popularity);
  if (popularity == Popularity::Distinct) {
    for (int i = 0; i < n; ++i) ids[static_cast<std::size_t>(i)] = i;
  } else if (popularity == Popularity::Uniform) {
    for (int i = 0; i < n; ++i) ids[static_cast<std::size_t>(i)] = i % m;
    rng.shuffle(ids);
  } else if (popularity == Popularity::Skewed) {
    if (alpha <= 1.0) throw std::invalid_argument("assign_models: Skewed needs alpha > 1");
    std::vector<double> cumulative;
    cumulative.reserve(static_cast<std::size_t>(m));
    // adjacent-rank popularity ratio alpha: weights 1, 1/alpha, 1/alpha^2, ... (by repeated division)
    double total = 0.0, w = 1.0;
    for (int i = 0; i < m; ++i) {
      total += w;
      cumulative.push_back(total);
      w /= alpha;
    }
    for (int i = 0; i < n; ++i) ids[static_cast<std::size_t>(i)] = static_cast<std::int64_t>(rng.discrete(cumulative, total));
  }
  return ids;
}

const char* to_string(Popularity p) {
  switch (p) {
    case Popularity::Distinct: return "distinct";
    case Popularity::Uniform: return "uniform";
    case Popularity::Skewed: return "skewed";
    case Popularity::Identical: return "identical";
  }
  return "?";
}

}  // namespace lorasim
