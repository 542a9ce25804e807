// semikern/dnn.hpp (B200 shim) -- the sparse ReLU DNN recurrence
// (proj/include/semikern/dnn.hpp:22-89, src/dnn.cpp:65-121): the hot path.
// relu_forward runs the whole L-layer chain inside the library (exact layer /
// windowed engine / ESC / dense engine per layer); outputs are
// bitwise the reference's.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "matrix.hpp"

namespace semikern {

using Batch = DenseMatrix;

namespace detail {
// Dense weights keep every entry (explicit zeros too), so the fold is exactly
// the dense kernel's (matrix.cpp:426-447).
inline CsrMatrix dense_as_csr(const DenseMatrix& d) {
  const auto v = d.data();
  std::vector<index_t> rp(static_cast<std::size_t>(d.rows()) + 1), ci(v.size());
  for (index_t i = 0; i <= d.rows(); ++i) rp[i] = i * d.cols();
  for (std::size_t e = 0; e < v.size(); ++e) ci[e] = static_cast<index_t>(e % d.cols());
  return CsrMatrix::from_parts_unchecked(d.rows(), d.cols(), std::move(rp), std::move(ci),
                                         std::vector<Scalar>(v.begin(), v.end()));
}
inline CsrMatrix as_csr(const Matrix& w) {
  return w.is_sparse() ? w.csr() : dense_as_csr(w.dense());
}
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
  int workers = 1;                // accepted; results never depend on it (dnn.hpp:75-76)
  bool materialize_bias = false;  // both bias paths give identical output
  float clip = 0.0f;              // extension: BASELINE cfg3-5 (0 = none, as the reference)
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
  (void)relu_zero;  // the fused epilogue never materialises the zero matrix
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
  detail::workers_ok(workers);
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
