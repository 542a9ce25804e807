// semikern_b200/semikern.hpp -- header-only C++ shim that re-exposes the
// reference library's hot-path API (namespace semikern, /root/reference/proj/
// include/semikern/{error,semiring,matrix,dnn}.hpp) on top of the C-ABI in
// sk_api.h, so a reference call site compiles against the B200 engine:
//
//   #include "semikern_b200/semikern.hpp"      // instead of semikern/dnn.hpp
//   using namespace semikern;
//   CsrMatrix w = csr_from_triples(m, m, triples);
//   Batch y = relu_forward(DnnModel({Matrix(w)}, {bias}), input);
//
// Differences a caller can observe, all deliberate:
//  * Matrices live in device memory.  Element access (operator(), row(),
//    data(), row_ptr() ...) copies to the host; results are identical.
//  * Handles are shared and immutable (the reference's value types are never
//    mutated after construction on the hot path), so copies are cheap.
//  * `workers` is accepted and ignored; results are bitwise independent of it,
//    as the reference guarantees (dnn.hpp:75-76).
//  * ForwardOptions gains `clip` (BASELINE cfg3-5); relu_forward_sparse() and
//    categories() are extensions for the sparse-activation workloads.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

#include "sk_api.h"

namespace semikern {

// ---- error.hpp:24-58 -----------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
class DomainError : public Error {
 public:
  using Error::Error;
};
class InvalidArgument : public Error {
 public:
  using Error::Error;
};
class ParseError : public Error {
 public:
  ParseError(std::size_t line, const std::string& message)
      : Error("line " + std::to_string(line) + ": " + message), line_(line) {}
  std::size_t line() const noexcept { return line_; }

 private:
  std::size_t line_;
};
/// Device allocation failed (the reference reports this as a SkippedRun).
class OutOfMemory : public Error {
 public:
  using Error::Error;
};

namespace detail {
inline void check(sk_status s) {
  if (s == SK_OK) return;
  const std::string msg = sk_last_error();
  switch (s) {
    case SK_ERR_DIMENSION: throw DimensionError(msg);
    case SK_ERR_DOMAIN: throw DomainError(msg);
    case SK_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case SK_ERR_PARSE: throw ParseError(0, msg);
    case SK_ERR_OOM: throw OutOfMemory(msg);
    default: throw Error(msg);
  }
}

/// Process-wide context of the current device (one CUDA stream).
inline sk_ctx* ctx() {
  static std::shared_ptr<sk_ctx> c = [] {
    sk_ctx* h = nullptr;
    check(sk_ctx_create(0, &h));
    return std::shared_ptr<sk_ctx>(h, [](sk_ctx* p) { sk_ctx_destroy(p); });
  }();
  return c.get();
}
}  // namespace detail

// ---- semiring.hpp:32-153 ----------------------------------------------------------
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

struct Semiring {
  SemiringKind kind;
  std::string_view name;
  Scalar zero;
  Scalar one;
};
inline Semiring arithmetic_semiring() noexcept {
  return {SemiringKind::arithmetic, "arithmetic", 0.0f, 1.0f};
}
inline Semiring max_plus_semiring() noexcept {
  return {SemiringKind::max_plus, "maxplus", -std::numeric_limits<Scalar>::infinity(), 0.0f};
}
inline Semiring min_max_semiring() noexcept {
  return {SemiringKind::min_max, "minmax", std::numeric_limits<Scalar>::infinity(), 0.0f};
}
inline Semiring gf2_semiring() noexcept { return {SemiringKind::gf2, "gf2", 0.0f, 1.0f}; }

// ---- matrix.hpp:29-218 --------------------------------------------------------------
using index_t = std::uint32_t;
inline constexpr std::size_t kIndexWidth = sizeof(index_t);

struct Triple {
  index_t row;
  index_t col;
  Scalar value;
};

class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(index_t rows, index_t cols, Scalar fill = 0.0f) {
    sk_dense* h = nullptr;
    detail::check(sk_dense_create(detail::ctx(), rows, cols, fill, &h));
    adopt(h);
  }
  DenseMatrix(index_t rows, index_t cols, std::vector<Scalar> data) {
    if (data.size() != static_cast<std::size_t>(rows) * cols)
      throw InvalidArgument("dense data length " + std::to_string(data.size()) +
                            " does not equal rows*cols for " + std::to_string(rows) + "x" +
                            std::to_string(cols));
    sk_dense* h = nullptr;
    detail::check(sk_dense_upload(detail::ctx(), rows, cols, data.data(), &h));
    adopt(h);
  }
  static DenseMatrix identity(index_t n) {
    sk_dense* h = nullptr;
    detail::check(sk_dense_identity(detail::ctx(), n, &h));
    DenseMatrix d;
    d.adopt(h);
    return d;
  }
  static DenseMatrix from_handle(sk_dense* h) {
    DenseMatrix d;
    d.adopt(h);
    return d;
  }

  index_t rows() const noexcept { return rows_; }
  index_t cols() const noexcept { return cols_; }
  /// Host copy of the row-major data.
  std::vector<Scalar> data() const {
    std::vector<Scalar> out(static_cast<std::size_t>(rows_) * cols_);
    if (!out.empty()) detail::check(sk_dense_download(detail::ctx(), h_.get(), out.data()));
    return out;
  }
  Scalar operator()(index_t i, index_t j) const {
    return data()[static_cast<std::size_t>(i) * cols_ + j];
  }
  std::vector<Scalar> row(index_t i) const {
    const auto d = data();
    return {d.begin() + static_cast<std::ptrdiff_t>(i) * cols_,
            d.begin() + static_cast<std::ptrdiff_t>(i + 1) * cols_};
  }
  sk_dense* handle() const noexcept { return h_.get(); }

 private:
  void adopt(sk_dense* h) {
    h_.reset(h, [](sk_dense* p) { sk_dense_free(p); });
    detail::check(sk_dense_shape(h, &rows_, &cols_));
  }
  index_t rows_ = 0, cols_ = 0;
  std::shared_ptr<sk_dense> h_;
};

class CsrMatrix {
 public:
  CsrMatrix() : CsrMatrix(0, 0, std::vector<index_t>{0}, {}, {}) {}
  /// Validating constructor (matrix.cpp:89-119).
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
  /// extractTuples: host copies of the three arrays (matrix.hpp:99-108).
  std::vector<index_t> row_ptr() const { return fetch().rp; }
  std::vector<index_t> col_idx() const { return fetch().ci; }
  std::vector<Scalar> values() const { return fetch().v; }
  std::vector<index_t> row_cols(index_t i) const {
    const auto& f = fetch();
    return {f.ci.begin() + f.rp[i], f.ci.begin() + f.rp[i + 1]};
  }
  std::vector<Scalar> row_values(index_t i) const {
    const auto& f = fetch();
    return {f.v.begin() + f.rp[i], f.v.begin() + f.rp[i + 1]};
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
      h->rp.resize(rows_ + 1);
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
  return (static_cast<std::size_t>(rows) + 1) * kIndexWidth + nnz_count * (kIndexWidth + 4);
}
constexpr std::size_t dense_storage_bytes(index_t rows, index_t cols) {
  return static_cast<std::size_t>(rows) * cols * sizeof(Scalar);
}
inline std::size_t storage_bytes(const Matrix& a) {
  return a.is_sparse() ? csr_storage_bytes(a.rows(), a.csr().nnz())
                       : dense_storage_bytes(a.rows(), a.cols());
}

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
  if (workers < 1) throw InvalidArgument("workers must be >= 1");
  sk_dense* h = nullptr;
  detail::check(sk_mxm_csr_dense(detail::ctx(), a.handle(), b.handle(), detail::kind(s), &h));
  return DenseMatrix::from_handle(h);
}
inline DenseMatrix mxm(const DenseMatrix& a, const DenseMatrix& b, const Semiring& s,
                       int workers = 1) {
  if (workers < 1) throw InvalidArgument("workers must be >= 1");
  sk_dense* h = nullptr;
  detail::check(sk_mxm_dense_dense(detail::ctx(), a.handle(), b.handle(), detail::kind(s), &h));
  return DenseMatrix::from_handle(h);
}
inline CsrMatrix mxm(const CsrMatrix& a, const CsrMatrix& b, const Semiring& s,
                     int workers = 1) {
  if (workers < 1) throw InvalidArgument("workers must be >= 1");
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
inline DenseMatrix dense_mxm_baseline(const DenseMatrix& a, const DenseMatrix& b,
                                      int workers = 1) {
  (void)workers;
  sk_dense* h = nullptr;
  detail::check(sk_dense_mxm_baseline(detail::ctx(), a.handle(), b.handle(), &h));
  return DenseMatrix::from_handle(h);
}

// ---- dnn.hpp:22-89 ----------------------------------------------------------------------
using Batch = DenseMatrix;

namespace detail {
// Dense weights keep every entry (explicit zeros too), so the fold is exactly
// the dense kernel's (matrix.cpp:426-447).
inline CsrMatrix dense_as_csr(const DenseMatrix& d) {
  const auto v = d.data();
  std::vector<index_t> rp(d.rows() + 1), ci(v.size());
  for (index_t i = 0; i <= d.rows(); ++i) rp[i] = i * d.cols();
  for (std::size_t e = 0; e < v.size(); ++e) ci[e] = static_cast<index_t>(e % d.cols());
  return CsrMatrix::from_parts_unchecked(d.rows(), d.cols(), rp, ci, v);
}
inline CsrMatrix as_csr(const Matrix& w) { return w.is_sparse() ? w.csr() : dense_as_csr(w.dense()); }
}  // namespace detail

class DnnModel {
 public:
  DnnModel(std::vector<Matrix> weights, std::vector<std::vector<Scalar>> biases)
      : weights_(std::move(weights)), biases_(std::move(biases)) {
    if (weights_.empty()) throw InvalidArgument("model must have at least one layer");
    if (weights_.size() != biases_.size())
      throw InvalidArgument("model has " + std::to_string(weights_.size()) +
                            " weight matrices but " + std::to_string(biases_.size()) +
                            " bias vectors");
    neurons_ = weights_.front().rows();
    std::vector<const sk_csr*> hs;
    std::vector<const float*> bs;
    for (std::size_t k = 0; k < weights_.size(); ++k) {
      const Matrix& w = weights_[k];
      if (w.rows() != neurons_ || w.cols() != neurons_)
        throw DimensionError("layer " + std::to_string(k) + " weight is " +
                             std::to_string(w.rows()) + "x" + std::to_string(w.cols()) +
                             "; all layers must be " + std::to_string(neurons_) + "x" +
                             std::to_string(neurons_));
      if (biases_[k].size() != neurons_)
        throw DimensionError("layer " + std::to_string(k) + " bias length " +
                             std::to_string(biases_[k].size()) + " does not match " +
                             std::to_string(neurons_) + " neurons");
      csr_.push_back(detail::as_csr(w));
      hs.push_back(csr_.back().handle());
      bs.push_back(biases_[k].data());
    }
    sk_model* h = nullptr;
    detail::check(sk_model_create(detail::ctx(), static_cast<uint32_t>(hs.size()), hs.data(),
                                  bs.data(), &h));
    h_.reset(h, [](sk_model* p) { sk_model_free(p); });
  }
  index_t num_layers() const noexcept { return static_cast<index_t>(weights_.size()); }
  index_t neurons() const noexcept { return neurons_; }
  const Matrix& weight(index_t k) const { return weights_[k]; }
  std::span<const Scalar> bias(index_t k) const { return biases_[k]; }
  sk_model* handle() const noexcept { return h_.get(); }

 private:
  index_t neurons_ = 0;
  std::vector<Matrix> weights_;
  std::vector<std::vector<Scalar>> biases_;
  std::vector<CsrMatrix> csr_;
  std::shared_ptr<sk_model> h_;
};

struct ForwardOptions {
  int workers = 1;
  bool materialize_bias = false;
  float clip = 0.0f;  // extension: BASELINE cfg3-5 (0 = none, as the reference)
};

namespace detail {
inline sk_fwd_opts opts(const ForwardOptions& o) {
  if (o.workers < 1) throw InvalidArgument("workers must be >= 1");
  return sk_fwd_opts{o.workers, o.materialize_bias ? 1 : 0, o.clip};
}
}  // namespace detail

inline DenseMatrix layer_step(const Matrix& w, std::span<const Scalar> bias,
                              const DenseMatrix& y, const DenseMatrix& relu_zero,
                              const ForwardOptions& opt = {}) {
  (void)relu_zero;  // the fused kernel never materialises the zero matrix
  if (w.cols() != y.rows())
    throw DimensionError("weight is " + std::to_string(w.rows()) + "x" +
                         std::to_string(w.cols()) + " but input has " +
                         std::to_string(y.rows()) + " rows");
  if (bias.size() != w.rows())
    throw DimensionError("bias length " + std::to_string(bias.size()) + " does not match " +
                         std::to_string(w.rows()) + " output rows");
  const CsrMatrix wc = detail::as_csr(w);
  const sk_fwd_opts o = detail::opts(opt);
  sk_dense* h = nullptr;
  detail::check(sk_layer_step(detail::ctx(), wc.handle(), bias.data(), y.handle(), &o, &h));
  return DenseMatrix::from_handle(h);
}
inline DenseMatrix layer_step(const Matrix& w, std::span<const Scalar> bias,
                              const DenseMatrix& y, const ForwardOptions& opt = {}) {
  return layer_step(w, bias, y, DenseMatrix(), opt);
}

inline Batch relu_forward(const DnnModel& model, const Batch& input,
                          const ForwardOptions& opt = {}) {
  const sk_fwd_opts o = detail::opts(opt);
  sk_dense* h = nullptr;
  detail::check(sk_relu_forward(detail::ctx(), model.handle(), input.handle(), &o, &h));
  return DenseMatrix::from_handle(h);
}
inline DenseMatrix dense_layer_step(const DenseMatrix& w, std::span<const Scalar> bias,
                                    const DenseMatrix& y, int workers = 1) {
  (void)workers;
  if (bias.size() != w.rows())
    throw DimensionError("bias length " + std::to_string(bias.size()) + " does not match " +
                         std::to_string(w.rows()) + " output rows");
  sk_dense* h = nullptr;
  detail::check(sk_dense_layer_step(detail::ctx(), w.handle(), bias.data(), y.handle(), &h));
  return DenseMatrix::from_handle(h);
}
inline Batch dense_relu_forward(const DnnModel& model, const Batch& input) {
  sk_dense* h = nullptr;
  detail::check(sk_dense_relu_forward(detail::ctx(), model.handle(), input.handle(), &h));
  return DenseMatrix::from_handle(h);
}

// ---- extensions ----------------------------------------------------------------------------
/// Sparse-activation forward pass (BASELINE cfg3-5); trace gets nnz(Y_k), k=0..L.
inline CsrMatrix relu_forward_sparse(const DnnModel& model, const CsrMatrix& y0,
                                     const ForwardOptions& opt = {},
                                     std::vector<std::uint64_t>* trace = nullptr) {
  const sk_fwd_opts o = detail::opts(opt);
  std::vector<std::uint64_t> t(model.num_layers() + 1);
  sk_csr* h = nullptr;
  detail::check(sk_relu_forward_sparse(detail::ctx(), model.handle(), y0.handle(), &o, &h,
                                       t.data()));
  if (trace) *trace = std::move(t);
  return CsrMatrix::from_handle(h);
}
/// Sorted indices of samples (columns) with any nonzero activation.
inline std::vector<index_t> categories(const CsrMatrix& y) {
  std::size_t n = 0;
  std::vector<index_t> out(y.cols());
  detail::check(sk_categories_csr(detail::ctx(), y.handle(), out.data(), out.size(), &n));
  out.resize(n);
  return out;
}
inline std::vector<index_t> categories(const DenseMatrix& y) {
  std::size_t n = 0;
  std::vector<index_t> out(y.cols());
  detail::check(sk_categories_dense(detail::ctx(), y.handle(), out.data(), out.size(), &n));
  out.resize(n);
  return out;
}

}  // namespace semikern
