// Reference hot-path test cases, restated, run through the C++ shim
// (include/semikern_b200/semikern.hpp) and therefore through the C-ABI and
// the CUDA kernels.  Each case cites the reference test it mirrors.  Built and
// run by tests/test_cpp_shim.py; prints one line per case, exits nonzero on
// any failure.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "semikern_b200/semikern.hpp"

using namespace semikern;

namespace {

int g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++g_fail;                                                                  \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, Exc)          \
  do {                                      \
    bool ok_ = false;                       \
    try {                                   \
      (void)(expr);                         \
    } catch (const Exc&) {                  \
      ok_ = true;                           \
    } catch (...) {                         \
    }                                       \
    CHECK(ok_ && "throws " #Exc);           \
  } while (0)

struct Rng {  // SplitMix64, same construction as proj/include/semikern/rng.hpp
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double unit() { return double(next() >> 11) * 0x1.0p-53; }
};

CsrMatrix random_csr(index_t rows, index_t cols, double density, Rng& r) {
  std::vector<Triple> t;
  for (index_t i = 0; i < rows; ++i)
    for (index_t j = 0; j < cols; ++j)
      if (r.unit() < density) t.push_back({i, j, float(-1.0 + 2.0 * r.unit())});
  return csr_from_triples(rows, cols, t);
}

DenseMatrix random_dense(index_t rows, index_t cols, Rng& r) {
  std::vector<Scalar> v(size_t(rows) * cols);
  for (auto& x : v) x = float(r.unit());
  return DenseMatrix(rows, cols, v);
}

bool bitwise(std::span<const Scalar> a, std::span<const Scalar> b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

// Host copy of a (possibly temporary) matrix: data() views the matrix's own
// storage, as in the reference, so a temporary's view must not outlive it.
std::vector<Scalar> host(const DenseMatrix& d) {
  const auto v = d.data();
  return {v.begin(), v.end()};
}

}  // namespace

int main() {
  std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"identity weights clamp the negative entry (test_dnn.cpp:85-93)",
       [] {
         const DnnModel model({Matrix(DenseMatrix::identity(2))}, {{0.0f, 0.0f}});
         const Batch input(2, 1, std::vector<Scalar>{3.0f, -2.0f});
         for (const Batch& out : {relu_forward(model, input), dense_relu_forward(model, input)}) {
           CHECK(out(0, 0) == 3.0f);
           CHECK(out(1, 0) == 0.0f);
         }
       }},
      {"hand-computed single layer (test_dnn.cpp:95-105)",
       [] {
         const DenseMatrix w(2, 2, std::vector<Scalar>{1, 2, 3, 4});
         const DnnModel model({Matrix(w)}, {{1.0f, -100.0f}});
         const Batch input(2, 1, std::vector<Scalar>{1.0f, 1.0f});
         for (const Batch& out : {relu_forward(model, input), dense_relu_forward(model, input)}) {
           CHECK(out(0, 0) == 4.0f);
           CHECK(out(1, 0) == 0.0f);
         }
       }},
      {"mxm 2x2 arithmetic and max-plus (test_matrix.cpp:230-243)",
       [] {
         const DenseMatrix a(2, 2, std::vector<Scalar>{1, 2, 3, 4});
         const DenseMatrix b(2, 1, std::vector<Scalar>{5, 6});
         const DenseMatrix c = mxm(a, b, arithmetic_semiring());
         CHECK(c(0, 0) == 17.0f && c(1, 0) == 39.0f);
         const DenseMatrix d = mxm(a, b, max_plus_semiring());
         CHECK(d(0, 0) == 8.0f && d(1, 0) == 10.0f);
       }},
      {"csr_from_triples basics (test_matrix.cpp:39-78)",
       [] {
         const CsrMatrix m = csr_from_triples(1, 3, {{0, 2, 3.0f}, {0, 0, 1.0f}, {0, 1, 2.0f}});
         CHECK(m.row_cols(0)[0] == 0 && m.row_cols(0)[2] == 2 && m.row_values(0)[0] == 1.0f);
         CHECK(csr_from_triples(2, 2, {{0, 0, 0.0f}, {1, 1, 2.0f}}).nnz() == 1);
         const CsrMatrix e = csr_from_triples(2, 2, {});
         CHECK(e.nnz() == 0 && e.row_ptr().size() == 3);
         CHECK_THROWS_AS(csr_from_triples(2, 2, {{2, 0, 1.0f}}), InvalidArgument);
         CHECK_THROWS_AS(csr_from_triples(2, 2, {{0, 1, 1.0f}, {0, 1, 2.0f}}), InvalidArgument);
       }},
      {"validating constructor (test_matrix.cpp:80-88)",
       [] {
         CHECK_THROWS_AS(CsrMatrix(2, 2, {0, 1}, {0}, {1.0f}), InvalidArgument);
         CHECK_THROWS_AS(CsrMatrix(1, 2, {0, 2}, {1, 0}, {1.0f, 2.0f}), InvalidArgument);
         CHECK_THROWS_AS(CsrMatrix(1, 2, {0, 1}, {5}, {1.0f}), InvalidArgument);
         CHECK(CsrMatrix(1, 2, {0, 2}, {0, 1}, {0.0f, 2.0f}).nnz() == 2);
       }},
      {"layer_step edge cases (test_dnn.cpp:115-151)",
       [] {
         const std::vector<Scalar> b3(3, 0.0f);
         for (Scalar v : host(layer_step(Matrix(csr_from_triples(3, 3, {})), b3, DenseMatrix(3, 2, 1.0f))))
           CHECK(v == 0.0f);
         const std::vector<Scalar> m1(4, -1.0f);
         for (Scalar v : host(layer_step(Matrix(DenseMatrix::identity(4)), m1, DenseMatrix(4, 3, 1.0f))))
           CHECK(v == 0.0f);
         CHECK_THROWS_AS(layer_step(Matrix(DenseMatrix::identity(3)), b3, DenseMatrix(2, 2, 1.0f)),
                         DimensionError);
         const std::vector<Scalar> b2(2, 0.0f);
         CHECK_THROWS_AS(layer_step(Matrix(DenseMatrix::identity(3)), b2, DenseMatrix(3, 2, 1.0f)),
                         DimensionError);
       }},
      {"model construction is validated (test_dnn.cpp:67-83)",
       [] {
         const CsrMatrix w2 = csr_from_triples(2, 2, {{0, 0, 1.0f}});
         CHECK_THROWS_AS(DnnModel({}, {}), InvalidArgument);
         CHECK_THROWS_AS(DnnModel({Matrix(w2)}, {}), InvalidArgument);
         CHECK_THROWS_AS(DnnModel({Matrix(csr_from_triples(2, 3, {}))}, {{0.0f, 0.0f}}),
                         DimensionError);
         CHECK_THROWS_AS(DnnModel({Matrix(w2)}, {{0.0f}}), DimensionError);
         const DnnModel ok({Matrix(w2)}, {{0.0f, 0.0f}});
         CHECK(ok.num_layers() == 1 && ok.neurons() == 2);
       }},
      {"semiring path equals the dense reference on 50 random models (acceptance.cpp:60-90 "
       "criterion 1; test_dnn.cpp:153-172)",
       // The dense leg runs on tensor cores (3xTF32), so it is compared with the
       // reference's magnitude-scaled criterion (approx_equal_scaled,
       // semiring.hpp:50-55), scale = sum_k |w||y| propagated layer by layer.
       [] {
         Rng r{101};
         for (int trial = 0; trial < 50; ++trial) {
           const index_t m = 4 + r.next() % 61, layers = 1 + r.next() % 4, n = 1 + r.next() % 8;
           const double density = std::vector<double>{1.0, 0.25, 1.0 / 64}[r.next() % 3];
           std::vector<Matrix> ws;
           std::vector<std::vector<Scalar>> bs;
           for (index_t k = 0; k < layers; ++k) {
             ws.emplace_back(random_csr(m, m, density, r));
             std::vector<Scalar> b(m);
             for (auto& x : b) x = float(r.unit()) - 0.5f;
             bs.push_back(b);
           }
           const DnnModel model(ws, bs);
           const Batch input = random_dense(m, n, r);
           const auto a = host(relu_forward(model, input));
           const auto d = host(dense_relu_forward(model, input));
           const auto x0 = input.data();
           std::vector<double> y(x0.begin(), x0.end()), sc(y.size());
           for (auto& v : y) v = std::fabs(v);
           for (index_t k = 0; k < layers; ++k) {  // |W| |Y| + |b|, host double
             const auto rp = ws[k].csr().row_ptr();
             const auto ci = ws[k].csr().col_idx();
             const auto vv = ws[k].csr().values();
             std::fill(sc.begin(), sc.end(), 0.0);
             for (index_t i = 0; i < m; ++i)
               for (index_t e = rp[i]; e < rp[i + 1]; ++e)
                 for (index_t j = 0; j < n; ++j) sc[i * n + j] += std::fabs(vv[e]) * y[ci[e] * n + j];
             for (index_t i = 0; i < m; ++i)
               for (index_t j = 0; j < n; ++j) sc[i * n + j] += std::fabs(bs[k][i]);
             y = sc;
           }
           for (size_t q = 0; q < a.size(); ++q)
             CHECK(approx_equal_scaled(a[q], d[q], float(sc[q])));
           for (Scalar v : a) CHECK(v >= 0.0f);
         }
       }},
      {"stored semiring zeros never change results, 20 instances x 4 semirings "
       "(acceptance.cpp:147-180 criterion 4)",
       [] {
         Rng r{11};
         const Semiring all[] = {arithmetic_semiring(), max_plus_semiring(), min_max_semiring(),
                                 gf2_semiring()};
         auto rnd = [&](index_t rows, index_t cols, const Semiring& s) {
           std::vector<Triple> t;
           for (index_t i = 0; i < rows; ++i)
             for (index_t j = 0; j < cols; ++j)
               if (r.unit() < 0.35) {
                 float v = s.kind == SemiringKind::gf2 ? 1.0f : float(-4.0 + 8.0 * r.unit());
                 t.push_back({i, j, v});
               }
           return csr_from_triples(rows, cols, t);
         };
         auto inject = [&](const CsrMatrix& a, Scalar zero) {  // validating ctor, zeros kept
           std::vector<index_t> rp{0}, ci;
           std::vector<Scalar> v;
           for (index_t i = 0; i < a.rows(); ++i) {
             const auto cols = a.row_cols(i);
             const auto vals = a.row_values(i);
             size_t k = 0;
             for (index_t j = 0; j < a.cols(); ++j) {
               if (k < cols.size() && cols[k] == j) {
                 ci.push_back(j);
                 v.push_back(vals[k++]);
               } else if (r.unit() < 0.4) {
                 ci.push_back(j);
                 v.push_back(zero);
               }
             }
             rp.push_back(index_t(ci.size()));
           }
           return CsrMatrix(a.rows(), a.cols(), rp, ci, v);
         };
         auto same = [](const DenseMatrix& x, const DenseMatrix& y) {
           return x.rows() == y.rows() && x.cols() == y.cols() && bitwise(x.data(), y.data());
         };
         for (int trial = 0; trial < 20; ++trial) {
           const Semiring& s = all[trial % 4];
           const index_t m = 2 + r.next() % 8, l = 2 + r.next() % 8, n = 2 + r.next() % 8;
           const CsrMatrix a = rnd(m, l, s), b = rnd(l, n, s), e = rnd(m, l, s);
           const CsrMatrix az = inject(a, s.zero), bz = inject(b, s.zero), ez = inject(e, s.zero);
           CHECK(same(to_dense(mxm(a, b, s), s.zero), to_dense(mxm(az, bz, s), s.zero)));
           CHECK(same(mxm(a, to_dense(b, s.zero), s), mxm(az, to_dense(b, s.zero), s)));
           CHECK(same(to_dense(ewise_add(Matrix(a), Matrix(e), s), s.zero),
                      to_dense(ewise_add(Matrix(az), Matrix(ez), s), s.zero)));
           CHECK(same(to_dense(ewise_mul(Matrix(a), Matrix(e), s), s.zero),
                      to_dense(ewise_mul(Matrix(az), Matrix(ez), s), s.zero)));
         }
       }},
      {"zero bias reduces the layer to max(W*Y, 0) exactly (test_dnn.cpp:174-185)",
       [] {
         Rng r{31};
         const CsrMatrix w = random_csr(20, 20, 0.25, r);
         const DenseMatrix y = random_dense(20, 6, r);
         const auto got = host(layer_step(Matrix(w), std::vector<Scalar>(20, 0.0f), y));
         const auto prod = host(mxm(w, y, arithmetic_semiring()));
         for (size_t i = 0; i < got.size(); ++i) CHECK(got[i] == std::max(prod[i], 0.0f));
       }},
      {"forward output is bitwise identical across worker counts (acceptance.cpp:318-349 "
       "criterion 10; test_dnn.cpp:197-204)",
       [] {
         Rng r{1234};
         std::vector<Matrix> ws;
         std::vector<std::vector<Scalar>> bs;
         for (int k = 0; k < 3; ++k) {
           ws.emplace_back(random_csr(32, 32, 0.125, r));
           bs.emplace_back(32, 0.1f);
         }
         const DnnModel model(ws, bs);
         const Batch input = random_dense(32, 8, r);
         const auto base = host(relu_forward(model, input, {1, false}));
         for (int w : {2, 4}) CHECK(bitwise(host(relu_forward(model, input, {w, false})), base));
       }},
      {"sparse-activation route equals the dense route",
       [] {
         Rng r{77};
         std::vector<Matrix> ws;
         std::vector<std::vector<Scalar>> bs;
         for (int k = 0; k < 3; ++k) {
           ws.emplace_back(random_csr(64, 64, 0.25, r));
           bs.emplace_back(64, -0.05f);
         }
         const DnnModel model(ws, bs);
         const Batch input = random_dense(64, 40, r);
         const auto dense = host(relu_forward(model, input));
         std::vector<std::uint64_t> trace;
         const CsrMatrix sp = relu_forward_sparse(model, from_dense(input), {}, &trace);
         CHECK(bitwise(host(to_dense(sp, 0.0f)), dense));
         CHECK(trace.size() == 4 && trace[0] == 64u * 40u);
       }},
      {"gf2 domain violations surface from kernels (test_matrix.cpp:353-358)",
       [] {
         const CsrMatrix a = csr_from_triples(1, 1, {{0, 0, 2.0f}});
         const DenseMatrix b(1, 1, 1.0f);
         CHECK_THROWS_AS(mxm(a, b, gf2_semiring()), DomainError);
         CHECK_THROWS_AS(mxm(a, b, gf2_semiring(), 4), DomainError);
       }},
      {"nnz and storage bytes (test_matrix.cpp:112-128)",
       [] {
         const CsrMatrix empty = csr_from_triples(5, 4, {});
         CHECK(storage_bytes(Matrix(empty)) == 6 * kIndexWidth);
         DenseMatrix d(4, 4, std::vector<Scalar>(16, 0.0f));
         CHECK(nnz(Matrix(d)) == 0);
         CHECK(storage_bytes(Matrix(d)) == 64);
         CHECK(dense_storage_bytes(32768, 32768) == std::size_t{4} * 1024 * 1024 * 1024);
       }},
  };
  int failed_cases = 0;
  for (auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      std::printf("    exception: %s\n", e.what());
      ++g_fail;
    }
    const bool ok = g_fail == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
  }
  std::printf("%d of %zu cases failed\n", failed_cases, cases.size());
  return failed_cases ? 1 : 0;
}
