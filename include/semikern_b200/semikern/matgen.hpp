// semikern/matgen.hpp (B200 shim) -- the paper-sweep generators
// (proj/include/semikern/matgen.hpp:26-52, src/matgen.cpp).  Weights and
// inputs are generated on the device (sk_gen_weight / sk_gen_input_dense,
// bitwise equal to the reference); the m-element bias is drawn here.
#pragma once

#include <cstdint>
#include <vector>

#include "matrix.hpp"

namespace semikern {

struct GenSpec {
  index_t m = 0;
  double inverse_sparsity = 1.0;
  index_t batch = 64;
  std::uint64_t seed = 0;

  /// InvalidArgument unless m >= 1, batch >= 1, inverse_sparsity >= 1.
  void validate() const {
    if (m < 1) throw InvalidArgument("GenSpec: m must be >= 1");
    if (batch < 1) throw InvalidArgument("GenSpec: batch must be >= 1");
    if (!(inverse_sparsity >= 1.0))
      throw InvalidArgument("GenSpec: inverse_sparsity must be >= 1");
  }
};

enum class BiasMode { zero, uniform01 };

/// m x m, entry (i, j) kept with probability 1/inverse_sparsity.
inline CsrMatrix gen_weight(const GenSpec& spec) {
  spec.validate();
  sk_csr* h = nullptr;
  detail::check(sk_gen_weight(detail::ctx(), spec.m, spec.inverse_sparsity, spec.seed, &h));
  return CsrMatrix::from_handle(h);
}

/// m x batch, U[0, 1).
inline DenseMatrix gen_input(const GenSpec& spec) {
  spec.validate();
  sk_dense* h = nullptr;
  detail::check(sk_gen_input_dense(detail::ctx(), spec.m, spec.batch, spec.seed, &h));
  return DenseMatrix::from_handle(h);
}

/// zero, or U[0, 1) from the bias stream (stream 3 of the spec's seed).
inline std::vector<Scalar> gen_bias(const GenSpec& spec, BiasMode mode = BiasMode::zero) {
  spec.validate();
  std::vector<Scalar> b(spec.m, 0.0f);
  if (mode == BiasMode::uniform01) {
    const std::uint64_t stream = SplitMix64::at(spec.seed, 3);
    for (index_t i = 0; i < spec.m; ++i)
      b[i] = static_cast<Scalar>(SplitMix64::to_unit(SplitMix64::at(stream, i)));
  }
  return b;
}

}  // namespace semikern
