// semikern/rng.hpp (B200 shim) -- SplitMix64, the counter-addressable generator
// every reference generator draws from (proj/include/semikern/rng.hpp:22-62).
// The device generators (sk_gen_*) evaluate the same function per element.
#pragma once

#include <cstdint>

namespace semikern {

class SplitMix64 {
 public:
  explicit constexpr SplitMix64(std::uint64_t seed) noexcept : state_(seed) {}

  constexpr std::uint64_t next() noexcept { return finalize(state_ += kIncrement); }
  /// Uniform double in [0, 1) from the top 53 bits.
  double next_unit() noexcept { return to_unit(next()); }
  /// The value the (index+1)-th next() of a generator seeded with `seed` returns.
  static constexpr std::uint64_t at(std::uint64_t seed, std::uint64_t index) noexcept {
    return finalize(seed + (index + 1) * kIncrement);
  }
  static constexpr double to_unit(std::uint64_t bits) noexcept {
    return static_cast<double>(bits >> 11) * 0x1.0p-53;
  }

 private:
  static constexpr std::uint64_t kIncrement = 0x9E3779B97F4A7C15ull;  // golden-ratio step
  static constexpr std::uint64_t finalize(std::uint64_t x) noexcept {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  std::uint64_t state_;
};

}  // namespace semikern
