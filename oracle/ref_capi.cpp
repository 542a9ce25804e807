// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (semikern, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// exists so that Python tests, the golden-fixture generator and bench.py's
// reference arm can call the reference's own hot-path functions through
// ctypes.  Every function below forwards to the reference API named in its
// comment; the one exception is skref_layer_sparse_h, which follows the
// reference's mxm(CsrMatrix, CsrMatrix) with the sparse-activation layer
// epilogue the reference has no function for (restated exactly as
// oracle/sk_oracle.c sko_sparse_epilogue: z = Z + b_i -> ReLU select -> clip ->
// prune, untouched positions give epilogue(0 + b_i)).
//
// Reference interfaces wrapped (paths relative to /root/reference):
//   csr_from_triples            proj/include/semikern/matrix.hpp:144-150
//   CsrMatrix validating ctor   proj/include/semikern/matrix.hpp:84-89
//   from_dense / to_dense       proj/include/semikern/matrix.hpp:154-159
//   mxm (4 overloads)           proj/include/semikern/matrix.hpp:202-211
//   ewise_add / ewise_mul       proj/include/semikern/matrix.hpp:186-191
//   dense_mxm_baseline          proj/include/semikern/matrix.hpp:217-218
//   layer_step / relu_forward   proj/include/semikern/dnn.hpp:66-78
//   dense_layer_step / dense_relu_forward  proj/include/semikern/dnn.hpp:85-89
//   gen_weight / gen_input / gen_bias      proj/include/semikern/matgen.hpp:46-52
//   SplitMix64::at              proj/include/semikern/rng.hpp:43-46

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <sstream>

#include "semikern/bench.hpp"
#include "semikern/matio.hpp"
#include "semikern/dnn.hpp"
#include "semikern/error.hpp"
#include "semikern/matgen.hpp"
#include "semikern/matrix.hpp"
#include "semikern/rng.hpp"
#include "semikern/semiring.hpp"

using namespace semikern;

namespace {

thread_local std::string g_msg;

// Status codes shared with include/sk_api.h (SK_OK ... SK_ERR_PARSE).
enum : int {
  kOk = 0,
  kErr = 1,
  kDim = 2,
  kDomain = 3,
  kInvalid = 4,
  kParse = 5,
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const DimensionError& e) {
    g_msg = e.what();
    return kDim;
  } catch (const DomainError& e) {
    g_msg = e.what();
    return kDomain;
  } catch (const InvalidArgument& e) {
    g_msg = e.what();
    return kInvalid;
  } catch (const ParseError& e) {
    g_msg = e.what();
    return kParse;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return kErr;
  }
}

Semiring semiring_of(int kind) {
  switch (kind) {
    case 0: return arithmetic_semiring();
    case 1: return max_plus_semiring();
    case 2: return min_max_semiring();
    case 3: return gf2_semiring();
  }
  throw InvalidArgument("unknown semiring kind " + std::to_string(kind));
}

CsrMatrix csr_of(uint32_t rows, uint32_t cols, const uint32_t* rp,
                 const uint32_t* ci, const float* v) {
  const std::size_t nnz = rp[rows];
  return CsrMatrix(rows, cols, std::vector<index_t>(rp, rp + rows + 1),
                   std::vector<index_t>(ci, ci + nnz),
                   std::vector<Scalar>(v, v + nnz));
}

DenseMatrix dense_of(uint32_t rows, uint32_t cols, const float* d) {
  return DenseMatrix(rows, cols,
                     std::vector<Scalar>(d, d + std::size_t(rows) * cols));
}

void copy_out(const DenseMatrix& m, float* out) {
  std::memcpy(out, m.data().data(), m.data().size_bytes());
}

}  // namespace

/// Opaque owner of a reference CsrMatrix result.
struct skref_csr {
  CsrMatrix m;
};

extern "C" {

const char* skref_last_error(void) { return g_msg.c_str(); }

// --- rng -------------------------------------------------------------------
uint64_t skref_splitmix_at(uint64_t seed, uint64_t idx) {
  return SplitMix64::at(seed, idx);
}

// --- CSR handles --------------------------------------------------------------
int skref_csr_from_triples(uint32_t rows, uint32_t cols, const uint32_t* r,
                           const uint32_t* c, const float* v, size_t n,
                           skref_csr** out) {
  return guarded([&] {
    std::vector<Triple> t(n);
    for (size_t i = 0; i < n; ++i) t[i] = Triple{r[i], c[i], v[i]};
    *out = new skref_csr{csr_from_triples(rows, cols, t)};
  });
}

int skref_csr_from_parts(uint32_t rows, uint32_t cols, const uint32_t* rp,
                         const uint32_t* ci, const float* v, skref_csr** out) {
  return guarded([&] { *out = new skref_csr{csr_of(rows, cols, rp, ci, v)}; });
}

int skref_csr_from_dense(uint32_t rows, uint32_t cols, const float* d,
                         skref_csr** out) {
  return guarded(
      [&] { *out = new skref_csr{from_dense(dense_of(rows, cols, d))}; });
}

size_t skref_csr_nnz(const skref_csr* a) { return a->m.nnz(); }
uint32_t skref_csr_rows(const skref_csr* a) { return a->m.rows(); }
uint32_t skref_csr_cols(const skref_csr* a) { return a->m.cols(); }

void skref_csr_extract(const skref_csr* a, uint32_t* rp, uint32_t* ci,
                       float* v) {
  const auto r = a->m.row_ptr();
  const auto c = a->m.col_idx();
  const auto x = a->m.values();
  if (rp) std::memcpy(rp, r.data(), r.size_bytes());
  if (ci) std::memcpy(ci, c.data(), c.size_bytes());
  if (v) std::memcpy(v, x.data(), x.size_bytes());
}

void skref_csr_free(skref_csr* a) { delete a; }

int skref_to_dense(const skref_csr* a, float ambient_zero, float* out) {
  return guarded([&] { copy_out(to_dense(a->m, ambient_zero), out); });
}

// --- mxm ------------------------------------------------------------------------
int skref_mxm_csr_dense(const skref_csr* a, uint32_t brows, uint32_t bcols,
                        const float* b, int semiring, int workers, float* out) {
  return guarded([&] {
    copy_out(mxm(a->m, dense_of(brows, bcols, b), semiring_of(semiring), workers),
             out);
  });
}

int skref_mxm_dense_dense(uint32_t arows, uint32_t acols, const float* a,
                          uint32_t brows, uint32_t bcols, const float* b,
                          int semiring, int workers, float* out) {
  return guarded([&] {
    copy_out(mxm(dense_of(arows, acols, a), dense_of(brows, bcols, b),
                 semiring_of(semiring), workers),
             out);
  });
}

int skref_mxm_csr_csr(const skref_csr* a, const skref_csr* b, int semiring,
                      int workers, skref_csr** out) {
  return guarded([&] {
    *out = new skref_csr{mxm(a->m, b->m, semiring_of(semiring), workers)};
  });
}

// One sparse-activation layer on reference handles (bench.py's reference arm):
// Z = mxm(W_ref, Y_ref) (proj/src/matrix.cpp:541-547 -> 452-521, the
// reference's own Gustavson SpGEMM, `workers` threads), then the restated
// epilogue; the result is a reference CsrMatrix (validating constructor,
// matrix.hpp:84-89) so layers chain without leaving the reference's types.
int skref_layer_sparse_h(const skref_csr* w, const skref_csr* y, const float* bias,
                         float clip, int workers, skref_csr** out) {
  return guarded([&] {
    const CsrMatrix z = mxm(w->m, y->m, arithmetic_semiring(), workers);
    const uint32_t m = z.rows(), n = z.cols();
    auto epi = [clip](float acc, float b) {
      float v = acc + b;
      v = (v < 0.0f) ? 0.0f : v;
      if (clip > 0.0f) v = (v > clip) ? clip : v;
      return v;
    };
    std::vector<index_t> rp(size_t(m) + 1, 0), ci;
    std::vector<Scalar> v;
    const auto zrp = z.row_ptr();
    const auto zci = z.col_idx();
    const auto zv = z.values();
    for (uint32_t i = 0; i < m; ++i) {
      const float untouched = epi(0.0f, bias[i]);
      size_t q = zrp[i];
      const size_t qe = zrp[i + 1];
      if (untouched == 0.0f) {
        for (; q < qe; ++q) {
          const float o = epi(zv[q], bias[i]);
          if (o != 0.0f) {
            ci.push_back(zci[q]);
            v.push_back(o);
          }
        }
      } else {
        for (uint32_t s = 0; s < n; ++s) {
          const float o = (q < qe && zci[q] == s) ? epi(zv[q++], bias[i]) : untouched;
          if (o != 0.0f) {
            ci.push_back(s);
            v.push_back(o);
          }
        }
      }
      rp[i + 1] = index_t(ci.size());
    }
    *out = new skref_csr{CsrMatrix(m, n, std::move(rp), std::move(ci), std::move(v))};
  });
}

int skref_dense_mxm_baseline(uint32_t arows, uint32_t acols, const float* a,
                             uint32_t brows, uint32_t bcols, const float* b,
                             int workers, float* out) {
  return guarded([&] {
    copy_out(dense_mxm_baseline(dense_of(arows, acols, a),
                                dense_of(brows, bcols, b), workers),
             out);
  });
}

// --- element-wise -------------------------------------------------------------
int skref_ewise_dense(int mul, uint32_t rows, uint32_t cols, const float* a,
                      const float* b, int semiring, float* out) {
  return guarded([&] {
    const DenseMatrix da = dense_of(rows, cols, a);
    const DenseMatrix db = dense_of(rows, cols, b);
    const Semiring s = semiring_of(semiring);
    copy_out(mul ? ewise_mul(da, db, s) : ewise_add(da, db, s), out);
  });
}

// Sparse (+) sparse keeps union semantics (matrix.cpp:253-290).
int skref_ewise_csr(int mul, const skref_csr* a, const skref_csr* b,
                    int semiring, skref_csr** out) {
  return guarded([&] {
    const Semiring s = semiring_of(semiring);
    Matrix r = mul ? ewise_mul(Matrix(a->m), Matrix(b->m), s)
                   : ewise_add(Matrix(a->m), Matrix(b->m), s);
    *out = new skref_csr{r.csr()};
  });
}

// --- DNN ----------------------------------------------------------------------------
// Layers are given in the reference orientation: W_ref[k] is m-by-m CSR with
// row i = in-edges of output neuron i; Y is m-by-n neuron-major.
static DnnModel model_of(uint32_t m, uint32_t layers, const skref_csr* const* w,
                         const float* const* bias, int dense_weights) {
  std::vector<Matrix> ws;
  std::vector<std::vector<Scalar>> bs;
  for (uint32_t k = 0; k < layers; ++k) {
    if (dense_weights)
      ws.emplace_back(to_dense(w[k]->m, 0.0f));
    else
      ws.emplace_back(w[k]->m);
    bs.emplace_back(bias[k], bias[k] + m);
  }
  return DnnModel(std::move(ws), std::move(bs));
}

int skref_relu_forward(uint32_t m, uint32_t layers, const skref_csr* const* w,
                       const float* const* bias, uint32_t n, const float* y0,
                       int workers, int materialize_bias, float* out) {
  return guarded([&] {
    const DnnModel model = model_of(m, layers, w, bias, 0);
    ForwardOptions opt;
    opt.workers = workers;
    opt.materialize_bias = materialize_bias != 0;
    copy_out(relu_forward(model, dense_of(m, n, y0), opt), out);
  });
}

int skref_dense_relu_forward(uint32_t m, uint32_t layers,
                             const skref_csr* const* w, const float* const* bias,
                             uint32_t n, const float* y0, float* out) {
  return guarded([&] {
    const DnnModel model = model_of(m, layers, w, bias, 0);
    copy_out(dense_relu_forward(model, dense_of(m, n, y0)), out);
  });
}

int skref_layer_step(const skref_csr* w, const float* bias, uint32_t n,
                     const float* y, int workers, float* out) {
  return guarded([&] {
    const uint32_t m = w->m.rows();
    ForwardOptions opt;
    opt.workers = workers;
    copy_out(layer_step(Matrix(w->m), std::span<const Scalar>(bias, m),
                        dense_of(w->m.cols(), n, y), opt),
             out);
  });
}

int skref_dense_layer_step(uint32_t m, uint32_t l, const float* wd,
                           const float* bias, uint32_t n, const float* y,
                           int workers, float* out) {
  return guarded([&] {
    copy_out(dense_layer_step(dense_of(m, l, wd), std::span<const Scalar>(bias, m),
                              dense_of(l, n, y), workers),
             out);
  });
}

// --- generators (matgen.cpp) --------------------------------------------------------
int skref_gen_weight(uint32_t m, double inverse_sparsity, uint64_t seed,
                     skref_csr** out) {
  return guarded([&] {
    *out = new skref_csr{gen_weight(GenSpec{m, inverse_sparsity, 1, seed})};
  });
}

int skref_gen_input(uint32_t m, uint32_t batch, uint64_t seed, float* out) {
  return guarded([&] { copy_out(gen_input(GenSpec{m, 1.0, batch, seed}), out); });
}

int skref_gen_bias(uint32_t m, uint64_t seed, int uniform01, float* out) {
  return guarded([&] {
    const auto b = gen_bias(GenSpec{m, 1.0, 1, seed},
                            uniform01 ? BiasMode::uniform01 : BiasMode::zero);
    std::memcpy(out, b.data(), b.size() * sizeof(float));
  });
}

static void text_out(const std::string& t, char* buf, size_t cap, size_t* len);

// ---- Matrix Market (proj/include/semikern/matio.hpp) ------------------------------

/* read_matrix(std::istream&): *kind 0 = coordinate (CSR in *csr), 1 = array
 * (dense copied into `dense` when *rows * *cols <= cap). */
int skref_read_matrix_text(const char* text, int* kind, uint32_t* rows, uint32_t* cols,
                           skref_csr** csr, float* dense, size_t cap) {
  return guarded([&] {
    std::istringstream in{std::string(text)};
    Matrix m = read_matrix(in);
    *rows = m.rows();
    *cols = m.cols();
    if (m.is_sparse()) {
      *kind = 0;
      *csr = new skref_csr{m.csr()};
    } else {
      *kind = 1;
      const auto d = m.dense().data();
      if (d.size() <= cap) std::memcpy(dense, d.data(), d.size_bytes());
    }
  });
}

/* write_matrix(Matrix, std::ostream&) of a CSR (csr != null) or a dense matrix. */
int skref_format_matrix(const skref_csr* csr, uint32_t rows, uint32_t cols, const float* dense,
                        char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::ostringstream o;
    if (csr)
      write_matrix(Matrix(csr->m), o);
    else
      write_matrix(Matrix(dense_of(rows, cols, dense)), o);
    text_out(o.str(), buf, cap, len);
  });
}

// ---- benchmark sweep analysis and CSV (proj/include/semikern/bench.hpp) -----------

static std::vector<BenchRecord> records_of(size_t n, const uint32_t* m, const double* is,
                                           const int* impl, const int* workers,
                                           const double* mean, const double* sd,
                                           const uint64_t* nnz, const uint64_t* bytes) {
  std::vector<BenchRecord> r(n);
  for (size_t i = 0; i < n; ++i) {
    r[i].m = m[i];
    r[i].inverse_sparsity = is[i];
    r[i].implementation = impl[i] ? Impl::dense : Impl::sparse;
    r[i].workers = workers[i];
    r[i].mean_layer_seconds = mean[i];
    r[i].stddev_seconds = sd ? sd[i] : 0.0;
    r[i].nnz = nnz ? nnz[i] : 0;
    r[i].matrix_bytes = bytes ? bytes[i] : 0;
  }
  return r;
}

static void text_out(const std::string& t, char* buf, size_t cap, size_t* len) {
  *len = t.size();
  if (buf && cap) {
    const size_t k = std::min(cap - 1, t.size());
    std::memcpy(buf, t.data(), k);
    buf[k] = 0;
  }
}

/* analyze (bench.cpp): out[9*j..] = m, ratio_dense, slope, saturation,
 * blas_per_element, and the four normalized values, per size. */
int skref_bench_analyze(size_t n, const uint32_t* m, const double* is, const int* impl,
                        const int* workers, const double* mean, uint32_t ref_m, size_t cap,
                        double* out, size_t* count) {
  return guarded([&] {
    const auto rec = records_of(n, m, is, impl, workers, mean, nullptr, nullptr, nullptr);
    const auto p = analyze(rec, ref_m);
    *count = p.size();
    for (size_t j = 0; j < p.size() && j < cap; ++j) {
      const double v[9] = {double(p[j].m), p[j].ratio_dense, p[j].slope, p[j].saturation,
                           p[j].blas_per_element, p[j].ratio_dense_normalized,
                           p[j].slope_normalized, p[j].saturation_normalized,
                           p[j].blas_per_element_normalized};
      std::memcpy(out + 9 * j, v, sizeof v);
    }
  });
}

int skref_bench_records_csv(size_t n, const uint32_t* m, const double* is, const int* impl,
                            const int* workers, const double* mean, const double* sd,
                            const uint64_t* nnz, const uint64_t* bytes, char* buf, size_t cap,
                            size_t* len) {
  return guarded([&] {
    std::ostringstream o;
    write_records_csv(records_of(n, m, is, impl, workers, mean, sd, nnz, bytes), o);
    text_out(o.str(), buf, cap, len);
  });
}

int skref_bench_params_csv(size_t n, const uint32_t* m, const double* is, const int* impl,
                           const int* workers, const double* mean, uint32_t ref_m, char* buf,
                           size_t cap, size_t* len) {
  return guarded([&] {
    const auto p = analyze(records_of(n, m, is, impl, workers, mean, nullptr, nullptr, nullptr),
                           ref_m);
    std::ostringstream o;
    write_params_csv(p, o);
    text_out(o.str(), buf, cap, len);
  });
}

/* read_records_csv: parsed fields (cap records) or the ParseError message. */
int skref_bench_read_csv(const char* text, size_t cap, uint32_t* m, double* is, int* impl,
                         int* workers, double* mean, double* sd, uint64_t* nnz, uint64_t* bytes,
                         size_t* count) {
  return guarded([&] {
    std::istringstream in{std::string(text)};
    const auto r = read_records_csv(in);
    *count = r.size();
    for (size_t i = 0; i < r.size() && i < cap; ++i) {
      m[i] = r[i].m;
      is[i] = r[i].inverse_sparsity;
      impl[i] = r[i].implementation == Impl::dense;
      workers[i] = r[i].workers;
      mean[i] = r[i].mean_layer_seconds;
      sd[i] = r[i].stddev_seconds;
      nnz[i] = r[i].nnz;
      bytes[i] = r[i].matrix_bytes;
    }
  });
}

/* BenchConfig::validate on the given fields (bench.cpp). */
int skref_bench_validate(size_t nsizes, const uint32_t* sizes, size_t nis, const double* is,
                         uint32_t batch, uint32_t layers, size_t nworkers, const int* workers,
                         int repetitions, int warmup) {
  return guarded([&] {
    BenchConfig c;
    c.sizes.assign(sizes, sizes + nsizes);
    c.inverse_sparsities.assign(is, is + nis);
    c.batch = batch;
    c.layers = layers;
    c.workers.assign(workers, workers + nworkers);
    c.repetitions = repetitions;
    c.warmup = warmup;
    c.validate();
  });
}

}  // extern "C"
