// janus/rng.hpp — the pinned splitmix64 generator.
//
// Drop-in for reference proj/include/janus/rng.hpp:11-38: identical next()
// sequence (Steele/Lea/Flood constants), `next() % n` bounded draws, 53-bit
// doubles and the descending Fisher–Yates shuffle, so every seeded artefact
// (GARS shuffles, synthetic cells, parameters, targets) reproduces across C,
// C++, Python and CUDA.  The extra members below (normal(), derive()) are the
// synthetic-data helpers the training path needs; they only consume next().
#pragma once

#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

namespace janus {

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}

  std::uint64_t next() {
    state_ += kGamma;
    std::uint64_t x = state_;
    x = (x ^ (x >> 30)) * kMix1;
    x = (x ^ (x >> 27)) * kMix2;
    return x ^ (x >> 31);
  }

  /// Uniform integer in [0, n); n <= 1 yields 0 without consuming a draw.
  std::uint64_t next_below(std::uint64_t n) {
    if (n <= 1) return 0;
    return next() % n;
  }

  /// Uniform double in [0, 1) built from the top 53 bits.
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

  /// Descending Fisher–Yates: for i = size..2, swap v[i-1] with v[next_below(i)].
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t i = v.size(); i >= 2; --i) {
      const auto j = static_cast<std::size_t>(next_below(i));
      using std::swap;
      swap(v[i - 1], v[j]);
    }
  }

  /// Standard normal via Box–Muller on two uniforms (u1 mapped to (0,1]).
  /// Pinned: consumes exactly two draws, returns the cosine branch.
  double normal() {
    const double u1 = 1.0 - next_double();
    const double u2 = next_double();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }

  /// Independent stream for a named tensor: seed ^ (tag * golden-ratio).
  static SplitMix64 derive(std::uint64_t seed, std::uint64_t tag) {
    return SplitMix64(seed ^ (tag * kGamma));
  }

 private:
  static constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
  static constexpr std::uint64_t kMix1 = 0xbf58476d1ce4e5b9ULL;
  static constexpr std::uint64_t kMix2 = 0x94d049bb133111ebULL;
  std::uint64_t state_;
};

}  // namespace janus
