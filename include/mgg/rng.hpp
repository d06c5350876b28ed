// SplitMix64 (Steele, Lea & Flood 2014), the generator the reference pins all
// synthetic inputs to (R:proj/include/pipeshard/rng.hpp:26-54): the same
// stream gives bit-identical graphs, so the reference library and this one
// can be fed the same workload from a seed alone.
#pragma once

#include <cstdint>

namespace mgg {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}

  std::uint64_t next_u64() {
    std::uint64_t z = (s_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }

  /// Uniform in [0, n), n > 0; unbiased by rejecting the top partial bucket
  /// (same acceptance region as R:proj/include/pipeshard/rng.hpp:39-45, so
  /// the stream positions match draw for draw).
  std::uint64_t next_below(std::uint64_t n) {
    const std::uint64_t reject_from = ~0ull - (~0ull % n);
    std::uint64_t v;
    do v = next_u64();
    while (v >= reject_from);
    return v % n;
  }

  /// Uniform in [0, 1) from the top 53 bits.
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

 private:
  std::uint64_t s_;
};

}  // namespace mgg
