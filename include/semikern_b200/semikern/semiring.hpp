// semikern/semiring.hpp (B200 shim) -- semirings, scalar operators and the law
// checker (proj/include/semikern/semiring.hpp:32-203, src/semiring.cpp).
// The scalar operators are the host twins of the device op tables in
// csrc/sk_common.cuh; check_laws evaluates every law on the DEVICE, through
// the element-wise kernels the library's mxm/ewise paths share.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <string>
#include <string_view>
#include <vector>

#include "error.hpp"

namespace semikern {

using Scalar = float;
enum class SemiringKind : std::uint8_t { arithmetic, max_plus, min_max, gf2 };

inline constexpr float kRelTol = 1e-5f;
inline constexpr float kAbsTol = 1e-6f;

inline bool approx_equal(Scalar x, Scalar y) noexcept {
  if (x == y) return true;
  return std::fabs(x - y) <= std::max(kAbsTol, kRelTol * std::max(std::fabs(x), std::fabs(y)));
}
inline bool approx_equal_scaled(Scalar x, Scalar y, float scale) noexcept {
  if (x == y) return true;
  return std::fabs(x - y) <= std::max(kAbsTol, kRelTol * scale);
}

namespace ops {
// One tag type per semiring (semiring.hpp:57-110); the device kernels carry the
// same four as OpArith / OpMaxPlus / OpMinMax / OpGf2.
struct Arithmetic {
  static constexpr SemiringKind kind = SemiringKind::arithmetic;
  static constexpr Scalar zero = 0.0f;
  static constexpr Scalar one = 1.0f;
  static Scalar add(Scalar a, Scalar b) noexcept { return a + b; }
  static Scalar mul(Scalar a, Scalar b) noexcept { return a * b; }
};
struct MaxPlus {
  static constexpr SemiringKind kind = SemiringKind::max_plus;
  static constexpr Scalar zero = -std::numeric_limits<Scalar>::infinity();
  static constexpr Scalar one = 0.0f;
  static Scalar add(Scalar a, Scalar b) noexcept { return a < b ? b : a; }
  static Scalar mul(Scalar a, Scalar b) noexcept { return a + b; }
};
struct MinMax {
  static constexpr SemiringKind kind = SemiringKind::min_max;
  static constexpr Scalar zero = std::numeric_limits<Scalar>::infinity();
  static constexpr Scalar one = 0.0f;
  static Scalar add(Scalar a, Scalar b) noexcept { return b < a ? b : a; }
  static Scalar mul(Scalar a, Scalar b) noexcept { return a < b ? b : a; }
};
struct Gf2 {
  static constexpr SemiringKind kind = SemiringKind::gf2;
  static constexpr Scalar zero = 0.0f;
  static constexpr Scalar one = 1.0f;
  static void require(Scalar v) {
    if (v != 0.0f && v != 1.0f)
      throw DomainError("GF(2) scalar must be 0 or 1, got " + std::to_string(v));
  }
  static Scalar add(Scalar a, Scalar b) {
    require(a);
    require(b);
    return a != b ? 1.0f : 0.0f;
  }
  static Scalar mul(Scalar a, Scalar b) {
    require(a);
    require(b);
    return a == 1.0f && b == 1.0f ? 1.0f : 0.0f;
  }
};
}  // namespace ops

template <typename F>
decltype(auto) dispatch(SemiringKind kind, F&& f) {
  switch (kind) {
    case SemiringKind::arithmetic: return f(ops::Arithmetic{});
    case SemiringKind::max_plus: return f(ops::MaxPlus{});
    case SemiringKind::min_max: return f(ops::MinMax{});
    case SemiringKind::gf2: return f(ops::Gf2{});
  }
  throw Error("unknown semiring kind");
}

struct Semiring {
  SemiringKind kind;
  std::string_view name;
  Scalar zero;  // additive identity, multiplicative annihilator
  Scalar one;   // multiplicative identity
  Scalar add(Scalar a, Scalar b) const {
    return dispatch(kind, [&](auto o) { return decltype(o)::add(a, b); });
  }
  Scalar mul(Scalar a, Scalar b) const {
    return dispatch(kind, [&](auto o) { return decltype(o)::mul(a, b); });
  }
};

inline Semiring arithmetic_semiring() noexcept {
  return {SemiringKind::arithmetic, "arithmetic", ops::Arithmetic::zero, ops::Arithmetic::one};
}
inline Semiring max_plus_semiring() noexcept {
  return {SemiringKind::max_plus, "maxplus", ops::MaxPlus::zero, ops::MaxPlus::one};
}
inline Semiring min_max_semiring() noexcept {
  return {SemiringKind::min_max, "minmax", ops::MinMax::zero, ops::MinMax::one};
}
inline Semiring gf2_semiring() noexcept {
  return {SemiringKind::gf2, "gf2", ops::Gf2::zero, ops::Gf2::one};
}
inline Semiring semiring_by_name(std::string_view name) {
  for (const Semiring& s :
       {arithmetic_semiring(), max_plus_semiring(), min_max_semiring(), gf2_semiring()})
    if (s.name == name) return s;
  throw InvalidArgument("unknown semiring '" + std::string(name) +
                        "' (expected arithmetic|maxplus|minmax|gf2)");
}

// ---- law checker (semiring.hpp:165-203) -------------------------------------------------
struct LawResult {
  std::string_view law;
  bool passed = true;
  std::size_t failures = 0;
  std::array<Scalar, 3> witness{};  // first failing (a, b, c)
  Scalar lhs = 0;
  Scalar rhs = 0;
};
struct LawReport {
  std::string_view semiring;
  std::size_t samples = 0;
  bool exact = true;  // compared bit for bit (tolerance for arithmetic)
  std::vector<LawResult> laws;
  bool all_passed() const {
    for (const LawResult& l : laws)
      if (!l.passed) return false;
    return true;
  }
};

/// Defined in semikern/matrix.hpp (the laws run through the device kernels).
inline LawReport check_laws(const Semiring& s, std::size_t samples, std::uint64_t seed);

}  // namespace semikern

#include "matrix.hpp"  // check_laws' definition needs DenseMatrix
