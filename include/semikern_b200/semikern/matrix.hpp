// semikern/matrix.hpp (B200 shim) -- the matrix value types and kernels
// (proj/include/semikern/matrix.hpp:29-218) over the C-ABI.
//
// Storage: every matrix owns a device object (sk_dense / sk_csr).  A
// DenseMatrix also keeps a host mirror, filled on the first element access and
// kept coherent both ways: writes through operator()/row()/data() land in the
// mirror and are uploaded before the next kernel reads the matrix; copies share
// storage until one of them is written (copy on write), so the reference's
// value semantics hold.  CsrMatrix is immutable (as in the reference): its
// spans view a host copy fetched once.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include "error.hpp"
#include "rng.hpp"
#include "semiring.hpp"
#include "sk_api.h"

namespace semikern {

namespace detail {
/// Status -> the reference's exception classes (error.hpp); parse errors carry
/// the line the library reports ("line N: ...").
inline void check(sk_status s) {
  if (s == SK_OK) return;
  const std::string msg = sk_last_error();
  switch (s) {
    case SK_ERR_DIMENSION: throw DimensionError(msg);
    case SK_ERR_DOMAIN: throw DomainError(msg);
    case SK_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case SK_ERR_PARSE: {
      std::size_t line = 0, pos = 5;
      if (msg.rfind("line ", 0) == 0) {
        while (pos < msg.size() && msg[pos] >= '0' && msg[pos] <= '9')
          line = line * 10 + static_cast<std::size_t>(msg[pos++] - '0');
        if (pos + 1 < msg.size() && msg[pos] == ':' && line > 0)
          throw ParseError(line, msg.substr(pos + 2));
      }
      throw ParseError(line, msg);
    }
    case SK_ERR_OOM: throw OutOfMemory(msg);
    default: throw Error(msg);
  }
}

/// Process-wide context of device 0 (one CUDA stream).
inline sk_ctx* ctx() {
  static std::shared_ptr<sk_ctx> c = [] {
    sk_ctx* h = nullptr;
    check(sk_ctx_create(0, &h));
    return std::shared_ptr<sk_ctx>(h, [](sk_ctx* p) { sk_ctx_destroy(p); });
  }();
  return c.get();
}
}  // namespace detail

using index_t = std::uint32_t;
inline constexpr std::size_t kIndexWidth = sizeof(index_t);

struct Triple {
  index_t row;
  index_t col;
  Scalar value;
};

class DenseMatrix {
 public:
  DenseMatrix() : s_(std::make_shared<State>()) {}
  DenseMatrix(index_t rows, index_t cols, Scalar fill = 0.0f) : DenseMatrix() {
    s_->rows = rows;
    s_->cols = cols;
    s_->host.assign(static_cast<std::size_t>(rows) * cols, fill);
  }
  /// Adopts `data` (row-major); InvalidArgument on a size mismatch.
  DenseMatrix(index_t rows, index_t cols, std::vector<Scalar> data) : DenseMatrix() {
    if (data.size() != static_cast<std::size_t>(rows) * cols)
      throw InvalidArgument("dense data length " + std::to_string(data.size()) +
                            " does not equal rows*cols for " + std::to_string(rows) + "x" +
                            std::to_string(cols));
    s_->rows = rows;
    s_->cols = cols;
    s_->host = std::move(data);
  }
  static DenseMatrix identity(index_t n) {
    sk_dense* h = nullptr;
    detail::check(sk_dense_identity(detail::ctx(), n, &h));
    return from_handle(h);
  }
  /// Takes ownership of a device matrix (the C-ABI's results).
  static DenseMatrix from_handle(sk_dense* h) {
    DenseMatrix d;
    d.s_->dev.reset(h, [](sk_dense* p) { sk_dense_free(p); });
    detail::check(sk_dense_shape(h, &d.s_->rows, &d.s_->cols));
    d.s_->host_ok = false;
    d.s_->dev_ok = true;
    return d;
  }

  index_t rows() const noexcept { return s_->rows; }
  index_t cols() const noexcept { return s_->cols; }

  Scalar operator()(index_t i, index_t j) const { return host()[at(i, j)]; }
  Scalar& operator()(index_t i, index_t j) { return writable()[at(i, j)]; }
  std::span<const Scalar> row(index_t i) const { return {host().data() + at(i, 0), cols()}; }
  std::span<Scalar> row(index_t i) { return {writable().data() + at(i, 0), cols()}; }
  std::span<const Scalar> data() const { return host(); }
  std::span<Scalar> data() { return writable(); }

  /// The device object, uploaded first if the host mirror was written.
  /// nullptr for a default-constructed (0 x 0) matrix.
  sk_dense* handle() const {
    State& s = *s_;
    if (!s.dev_ok) {
      if (!s.dev && s.rows == 0 && s.cols == 0) return nullptr;
      if (!s.dev) {
        sk_dense* h = nullptr;
        detail::check(sk_dense_upload(detail::ctx(), s.rows, s.cols, s.host.data(), &h));
        s.dev.reset(h, [](sk_dense* p) { sk_dense_free(p); });
      } else {
        detail::check(sk_dense_write(detail::ctx(), s.dev.get(), s.host.data()));
      }
      s.dev_ok = true;
    }
    return s.dev.get();
  }

 private:
  struct State {
    index_t rows = 0, cols = 0;
    std::shared_ptr<sk_dense> dev;
    std::vector<Scalar> host;
    bool host_ok = true;  // host mirror current
    bool dev_ok = false;  // device object current
  };
  std::size_t at(index_t i, index_t j) const { return static_cast<std::size_t>(i) * cols() + j; }
  const std::vector<Scalar>& host() const {
    State& s = *s_;
    if (!s.host_ok) {
      s.host.resize(static_cast<std::size_t>(s.rows) * s.cols);
      if (!s.host.empty())
        detail::check(sk_dense_download(detail::ctx(), s.dev.get(), s.host.data()));
      s.host_ok = true;
    }
    return s.host;
  }
  std::vector<Scalar>& writable() {
    host();
    if (s_.use_count() > 1) {  // copy on write
      auto own = std::make_shared<State>();
      own->rows = s_->rows;
      own->cols = s_->cols;
      own->host = s_->host;
      s_ = std::move(own);
    }
    s_->dev_ok = false;
    return s_->host;
  }
  std::shared_ptr<State> s_;
};

class CsrMatrix {
 public:
  CsrMatrix() : CsrMatrix(0, 0, std::vector<index_t>{0}, {}, {}) {}
  /// Validating constructor (matrix.cpp:89-119): the row_ptr/col_idx
  /// invariants are checked on the device, the first violation reported with
  /// the reference's message.  Stored values are not inspected.
  CsrMatrix(index_t rows, index_t cols, std::vector<index_t> row_ptr,
            std::vector<index_t> col_idx, std::vector<Scalar> values) {
    if (row_ptr.size() != static_cast<std::size_t>(rows) + 1)
      throw InvalidArgument("row_ptr length must be rows+1");
    if (row_ptr.front() != 0) throw InvalidArgument("row_ptr[0] must be 0");
    if (row_ptr.back() != col_idx.size() || col_idx.size() != values.size())
      throw InvalidArgument("row_ptr[rows], col_idx and values disagree on nnz");
    sk_csr* h = nullptr;
    detail::check(sk_csr_from_parts(detail::ctx(), rows, cols, row_ptr.data(), col_idx.data(),
                                    values.data(), 1, &h));
    adopt(h);
  }
  /// Trusted constructor for outputs that are valid by construction.
  static CsrMatrix from_parts_unchecked(index_t rows, index_t cols, std::vector<index_t> row_ptr,
                                        std::vector<index_t> col_idx,
                                        std::vector<Scalar> values) {
    sk_csr* h = nullptr;
    detail::check(sk_csr_from_parts(detail::ctx(), rows, cols, row_ptr.data(), col_idx.data(),
                                    values.data(), 0, &h));
    return from_handle(h);
  }
  static CsrMatrix from_handle(sk_csr* h) {
    CsrMatrix m(Tag{});
    m.adopt(h);
    return m;
  }

  index_t rows() const noexcept { return rows_; }
  index_t cols() const noexcept { return cols_; }
  std::size_t nnz() const noexcept { return nnz_; }
  /// extractTuples (matrix.hpp:99-108): views of a host copy fetched once.
  std::span<const index_t> row_ptr() const { return fetch().rp; }
  std::span<const index_t> col_idx() const { return fetch().ci; }
  std::span<const Scalar> values() const { return fetch().v; }
  std::span<const index_t> row_cols(index_t i) const {
    const Host& f = fetch();
    return {f.ci.data() + f.rp[i], f.rp[i + 1] - f.rp[i]};
  }
  std::span<const Scalar> row_values(index_t i) const {
    const Host& f = fetch();
    return {f.v.data() + f.rp[i], f.rp[i + 1] - f.rp[i]};
  }
  sk_csr* handle() const noexcept { return h_.get(); }

 private:
  struct Tag {};
  explicit CsrMatrix(Tag) {}
  struct Host {
    std::vector<index_t> rp, ci;
    std::vector<Scalar> v;
  };
  const Host& fetch() const {
    if (!host_) {
      auto h = std::make_shared<Host>();
      h->rp.resize(static_cast<std::size_t>(rows_) + 1);
      h->ci.resize(nnz_);
      h->v.resize(nnz_);
      detail::check(sk_csr_extract(detail::ctx(), h_.get(), h->rp.data(),
                                   nnz_ ? h->ci.data() : nullptr, nnz_ ? h->v.data() : nullptr));
      host_ = h;
    }
    return *host_;
  }
  void adopt(sk_csr* h) {
    h_.reset(h, [](sk_csr* p) { sk_csr_free(p); });
    detail::check(sk_csr_shape(h, &rows_, &cols_, &nnz_));
  }
  index_t rows_ = 0, cols_ = 0;
  std::size_t nnz_ = 0;
  std::shared_ptr<sk_csr> h_;
  mutable std::shared_ptr<Host> host_;
};

class Matrix {
 public:
  Matrix(CsrMatrix m) : rep_(std::move(m)) {}
  Matrix(DenseMatrix m) : rep_(std::move(m)) {}
  bool is_sparse() const noexcept { return std::holds_alternative<CsrMatrix>(rep_); }
  index_t rows() const noexcept {
    return is_sparse() ? std::get<CsrMatrix>(rep_).rows() : std::get<DenseMatrix>(rep_).rows();
  }
  index_t cols() const noexcept {
    return is_sparse() ? std::get<CsrMatrix>(rep_).cols() : std::get<DenseMatrix>(rep_).cols();
  }
  const CsrMatrix& csr() const {
    if (!is_sparse()) throw Error("matrix holds a dense representation");
    return std::get<CsrMatrix>(rep_);
  }
  const DenseMatrix& dense() const {
    if (is_sparse()) throw Error("matrix holds a sparse representation");
    return std::get<DenseMatrix>(rep_);
  }

 private:
  std::variant<CsrMatrix, DenseMatrix> rep_;
};

// ---- construction and conversion (matrix.cpp:145-260) --------------------------------------
inline CsrMatrix csr_from_triples(index_t rows, index_t cols, std::span<const Triple> t) {
  std::vector<index_t> r(t.size()), c(t.size());
  std::vector<Scalar> v(t.size());
  for (std::size_t i = 0; i < t.size(); ++i) {
    r[i] = t[i].row;
    c[i] = t[i].col;
    v[i] = t[i].value;
  }
  sk_csr* h = nullptr;
  detail::check(sk_csr_from_triples(detail::ctx(), rows, cols, r.data(), c.data(), v.data(),
                                    t.size(), &h));
  return CsrMatrix::from_handle(h);
}
inline CsrMatrix csr_from_triples(index_t rows, index_t cols,
                                  std::initializer_list<Triple> triples) {
  return csr_from_triples(rows, cols, std::span<const Triple>(triples.begin(), triples.size()));
}
inline DenseMatrix to_dense(const CsrMatrix& a, Scalar ambient_zero) {
  sk_dense* h = nullptr;
  detail::check(sk_to_dense(detail::ctx(), a.handle(), ambient_zero, &h));
  return DenseMatrix::from_handle(h);
}
inline DenseMatrix to_dense(const Matrix& a, Scalar ambient_zero) {
  return a.is_sparse() ? to_dense(a.csr(), ambient_zero) : a.dense();
}
inline CsrMatrix from_dense(const DenseMatrix& d) {
  sk_csr* h = nullptr;
  detail::check(sk_from_dense(detail::ctx(), d.handle(), &h));
  return CsrMatrix::from_handle(h);
}
inline std::size_t nnz(const Matrix& a) {
  if (a.is_sparse()) return a.csr().nnz();
  std::size_t n = 0;
  detail::check(sk_dense_nnz(detail::ctx(), a.dense().handle(), &n));
  return n;
}
constexpr std::size_t csr_storage_bytes(index_t rows, std::size_t nnz_count) {
  return (static_cast<std::size_t>(rows) + 1) * kIndexWidth +
         nnz_count * (kIndexWidth + sizeof(Scalar));
}
constexpr std::size_t dense_storage_bytes(index_t rows, index_t cols) {
  return static_cast<std::size_t>(rows) * cols * sizeof(Scalar);
}
inline std::size_t storage_bytes(const Matrix& a) {
  return a.is_sparse() ? csr_storage_bytes(a.rows(), a.csr().nnz())
                       : dense_storage_bytes(a.rows(), a.cols());
}

// ---- element-wise and products (matrix.cpp:262-447) ---------------------------------------
namespace detail {
inline sk_semiring kind(const Semiring& s) { return static_cast<sk_semiring>(s.kind); }
inline Matrix ewise(int mul, const Matrix& a, const Matrix& b, const Semiring& s) {
  if (a.is_sparse() && b.is_sparse()) {
    sk_csr* h = nullptr;
    check(sk_ewise_csr(ctx(), mul, a.csr().handle(), b.csr().handle(), kind(s), &h));
    return Matrix(CsrMatrix::from_handle(h));
  }
  sk_dense* h = nullptr;
  if (!a.is_sparse() && !b.is_sparse())
    check(sk_ewise_dense(ctx(), mul, a.dense().handle(), b.dense().handle(), kind(s), &h));
  else if (a.is_sparse())
    check(sk_ewise_mixed(ctx(), mul, a.csr().handle(), b.dense().handle(), 1, kind(s), &h));
  else
    check(sk_ewise_mixed(ctx(), mul, b.csr().handle(), a.dense().handle(), 0, kind(s), &h));
  return Matrix(DenseMatrix::from_handle(h));
}
inline void workers_ok(int workers) {
  if (workers < 1) throw InvalidArgument("workers must be >= 1");
}
}  // namespace detail

inline Matrix ewise_add(const Matrix& a, const Matrix& b, const Semiring& s) {
  return detail::ewise(0, a, b, s);
}
inline Matrix ewise_mul(const Matrix& a, const Matrix& b, const Semiring& s) {
  return detail::ewise(1, a, b, s);
}
inline DenseMatrix ewise_add(const DenseMatrix& a, const DenseMatrix& b, const Semiring& s) {
  return detail::ewise(0, Matrix(a), Matrix(b), s).dense();
}
inline DenseMatrix ewise_mul(const DenseMatrix& a, const DenseMatrix& b, const Semiring& s) {
  return detail::ewise(1, Matrix(a), Matrix(b), s).dense();
}

inline DenseMatrix mxm(const CsrMatrix& a, const DenseMatrix& b, const Semiring& s,
                       int workers = 1) {
  detail::workers_ok(workers);
  sk_dense* h = nullptr;
  detail::check(sk_mxm_csr_dense(detail::ctx(), a.handle(), b.handle(), detail::kind(s), &h));
  return DenseMatrix::from_handle(h);
}
inline DenseMatrix mxm(const DenseMatrix& a, const DenseMatrix& b, const Semiring& s,
                       int workers = 1) {
  detail::workers_ok(workers);
  sk_dense* h = nullptr;
  detail::check(sk_mxm_dense_dense(detail::ctx(), a.handle(), b.handle(), detail::kind(s), &h));
  return DenseMatrix::from_handle(h);
}
inline CsrMatrix mxm(const CsrMatrix& a, const CsrMatrix& b, const Semiring& s,
                     int workers = 1) {
  detail::workers_ok(workers);
  sk_csr* h = nullptr;
  detail::check(sk_mxm_csr_csr(detail::ctx(), a.handle(), b.handle(), detail::kind(s), &h));
  return CsrMatrix::from_handle(h);
}
inline DenseMatrix mxm(const Matrix& a, const DenseMatrix& b, const Semiring& s,
                       int workers = 1) {
  return a.is_sparse() ? mxm(a.csr(), b, s, workers) : mxm(a.dense(), b, s, workers);
}
inline Matrix mxm(const Matrix& a, const Matrix& b, const Semiring& s, int workers = 1) {
  if (a.is_sparse() && b.is_sparse()) return Matrix(mxm(a.csr(), b.csr(), s, workers));
  if (a.is_sparse()) return Matrix(mxm(a.csr(), b.dense(), s, workers));
  if (!b.is_sparse()) return Matrix(mxm(a.dense(), b.dense(), s, workers));
  throw Error("mxm: dense-by-sparse is not supported; densify the right operand");
}
/// The dense comparator (K4: tcgen05 3xTF32, within approx_equal_scaled).
inline DenseMatrix dense_mxm_baseline(const DenseMatrix& a, const DenseMatrix& b,
                                      int workers = 1) {
  detail::workers_ok(workers);
  sk_dense* h = nullptr;
  detail::check(sk_dense_mxm_baseline(detail::ctx(), a.handle(), b.handle(), &h));
  return DenseMatrix::from_handle(h);
}

// ---- check_laws (semiring.cpp:87-176) ------------------------------------------------------
// Samples per semiring as the reference draws them (finite values plus the
// semiring's infinities); the same (a, b, c) triples feed every law.  Each side
// of each law is evaluated for all samples at once by the device element-wise
// kernels on 1 x samples rows; comparison bit-exact, or approx_equal_scaled by
// max(|a|, |b|, |c|) for arithmetic.
namespace detail {
inline Scalar law_sample(SemiringKind kind, SplitMix64& rng) {
  switch (kind) {
    case SemiringKind::arithmetic:
      return static_cast<Scalar>(20.0 * rng.next_unit() - 10.0);
    case SemiringKind::max_plus: {
      const std::uint64_t r = rng.next();
      if (r % 8 == 0) return ops::MaxPlus::zero;
      return static_cast<Scalar>(static_cast<long>((r >> 3) & 1023) - 512) / 64.0f;
    }
    case SemiringKind::min_max: {
      const std::uint64_t r = rng.next();
      if (r % 8 == 0) return ops::MinMax::zero;
      return static_cast<Scalar>(10.0 * SplitMix64::to_unit(r));
    }
    case SemiringKind::gf2:
      return static_cast<Scalar>(rng.next() & 1);
  }
  throw Error("unknown semiring kind");
}
}  // namespace detail

inline LawReport check_laws(const Semiring& s, std::size_t samples, std::uint64_t seed) {
  if (samples < 1) throw InvalidArgument("check_laws: samples must be >= 1");
  LawReport rep;
  rep.semiring = s.name;
  rep.samples = samples;
  rep.exact = s.kind != SemiringKind::arithmetic;
  const auto n = static_cast<index_t>(samples);
  std::vector<Scalar> ha(samples), hb(samples), hc(samples);
  SplitMix64 rng(seed);
  for (std::size_t i = 0; i < samples; ++i) {
    ha[i] = detail::law_sample(s.kind, rng);
    hb[i] = detail::law_sample(s.kind, rng);
    hc[i] = detail::law_sample(s.kind, rng);
  }
  const DenseMatrix a(1, n, ha), b(1, n, hb), c(1, n, hc);
  const DenseMatrix zero(1, n, s.zero), one(1, n, s.one);
  const auto add = [&](const DenseMatrix& x, const DenseMatrix& y) { return ewise_add(x, y, s); };
  const auto mul = [&](const DenseMatrix& x, const DenseMatrix& y) { return ewise_mul(x, y, s); };
  struct Law {
    std::string_view name;
    DenseMatrix lhs, rhs;
  };
  const Law laws[] = {
      {"additive commutativity", add(a, b), add(b, a)},
      {"additive associativity", add(add(a, b), c), add(a, add(b, c))},
      {"multiplicative associativity", mul(mul(a, b), c), mul(a, mul(b, c))},
      {"left distributivity", mul(a, add(b, c)), add(mul(a, b), mul(a, c))},
      {"right distributivity", mul(add(a, b), c), add(mul(a, c), mul(b, c))},
      {"additive identity", add(a, zero), a},
      {"multiplicative identity", mul(a, one), a},
      {"multiplicative annihilator", mul(a, zero), zero},
  };
  for (const Law& law : laws) {
    LawResult r;
    r.law = law.name;
    const auto l = law.lhs.data(), x = law.rhs.data();
    for (std::size_t i = 0; i < samples; ++i) {
      const float scale = std::max({std::fabs(ha[i]), std::fabs(hb[i]), std::fabs(hc[i])});
      const bool ok = rep.exact ? l[i] == x[i] : approx_equal_scaled(l[i], x[i], scale);
      if (ok) continue;
      if (r.passed) {
        r.passed = false;
        r.witness = {ha[i], hb[i], hc[i]};
        r.lhs = l[i];
        r.rhs = x[i];
      }
      ++r.failures;
    }
    rep.laws.push_back(r);
  }
  return rep;
}

}  // namespace semikern
