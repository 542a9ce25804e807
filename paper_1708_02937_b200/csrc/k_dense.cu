// Dense comparator leg: dense_mxm_baseline / dense_layer_step /
// dense_relu_forward (proj/src/matrix.cpp:564-585, proj/src/dnn.cpp:123-149).
//
// launch_dense_gemm_tc() is the entry used by the C-ABI; the tensor-core
// implementation lives in k_dense_tc.cu.
#include "sk_common.cuh"

namespace sk {

void launch_mxm_dense_dense(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K,
                            uint32_t N, sk_semiring s, float* c);
sk_csr* csr_transpose(sk_ctx* ctx, const sk_csr* a);

// Below this many multiply-adds the dense comparator runs the CUDA-core GEMM
// in the reference's own order (c = 0, c += a_ik b_kj for ascending k, no FMA:
// matrix.cpp:564-585), so its results are bitwise the reference's.  A 128 x 256
// tcgen05 tile would be mostly padding there; above it K4 (3xTF32) runs, within
// approx_equal_scaled of the reference (K4).
constexpr uint64_t kExactDenseMacs = uint64_t(1) << 22;

__global__ void k_bias_relu(float* __restrict__ c, const float* __restrict__ bias, uint32_t M,
                            uint32_t N) {
  const size_t total = size_t(M) * N;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const float z = __fadd_rn(c[e], bias[e / N]);
    c[e] = z < 0.0f ? 0.0f : z;  // std::max(z, 0.0f) (dnn.cpp:135)
  }
}

// The dense comparator's GEMM (+ bias + ReLU when bias != nullptr).
void dense_gemm(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K, uint32_t N,
                const float* bias, float* c, PackCache* cache, uint64_t version) {
  if (uint64_t(M) * K * N <= kExactDenseMacs) {
    launch_mxm_dense_dense(ctx, a, b, M, K, N, SK_ARITHMETIC, c);
    if (bias && M && N)
      SK_LAUNCH(k_bias_relu, unsigned(std::min<uint64_t>((uint64_t(M) * N + 255) / 256,
                                                         uint64_t(ctx->num_sms) * 8)),
                256, 0, ctx->stream, c, bias, M, N);
    return;
  }
  launch_dense_gemm_tc(ctx, a, b, M, K, N, bias, bias ? 1 : 0, c, cache, version);
}

bool dense_gemm_exact(uint32_t M, uint32_t K, uint32_t N) {
  return uint64_t(M) * K * N <= kExactDenseMacs;
}

}  // namespace sk

using namespace sk;

extern "C" sk_status sk_dense_mxm_baseline(sk_ctx* ctx, const sk_dense* a, const sk_dense* b,
                                           sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    if (a->cols != b->rows)
      fail(SK_ERR_DIMENSION, "dense_mxm_baseline: inner dimensions " + std::to_string(a->cols) +
                                 " and " + std::to_string(b->rows) + " do not match");
    sk_dense* o = new_dense(ctx, a->rows, b->cols);
    dense_gemm(ctx, a->d, b->d, a->rows, a->cols, b->cols, nullptr, o->d,
               const_cast<PackCache*>(&a->pack), a->version);
    *out = o;
  });
}

extern "C" sk_status sk_dense_layer_step(sk_ctx* ctx, const sk_dense* w, const float* bias,
                                         const sk_dense* y, sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    if (!bias)
      fail(SK_ERR_DIMENSION, "bias length 0 does not match " + std::to_string(w->rows) +
                                 " output rows");
    if (w->cols != y->rows)
      fail(SK_ERR_DIMENSION, "dense_mxm_baseline: inner dimensions " + std::to_string(w->cols) +
                                 " and " + std::to_string(y->rows) + " do not match");
    float* db = dalloc<float>(ctx, w->rows);
    upload_staged(ctx, db, bias, size_t(w->rows) * 4);  // the host bias is only lent
    sk_dense* o = new_dense(ctx, w->rows, y->cols);
    dense_gemm(ctx, w->d, y->d, w->rows, w->cols, y->cols, db, o->d,
               const_cast<PackCache*>(&w->pack), w->version);
    dfree(ctx, db);
    *out = o;
  });
}

extern "C" sk_status sk_dense_relu_forward(sk_ctx* ctx, const sk_model* m, const sk_dense* y0,
                                           sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    if (y0->rows != m->neurons || y0->cols < 1)
      fail(SK_ERR_DIMENSION, "input batch is " + dim_string(y0->rows, y0->cols) + ", expected " +
                                 std::to_string(m->neurons) + " rows and n >= 1 columns");
    const uint32_t nn = m->neurons, n = y0->cols;
    sk_dense* wd = nullptr;
    SK_CUDA(cudaSuccess);
    // dnn.cpp:141-149: re-densify each layer's weights, then the dense step.
    sk_dense* bufs[2] = {new_dense(ctx, nn, n), new_dense(ctx, nn, n)};
    const float* src = y0->d;
    int cur = 0;
    for (uint32_t k = 0; k < m->layers; ++k) {
      // the densified weights are only needed to (re)build the packed copy cached
      // on the immutable CSR handle (dnn.cpp:145 re-densifies every layer; the
      // split / pack of a layer's weights happens once per model here)
      PackCache* pc = &const_cast<sk_csr*>(m->w[k])->pack;
      const bool cached = pc->buf && pc->version == 0 && !dense_gemm_exact(nn, nn, n);
      if (!cached) {
        sk_status st = sk_to_dense(ctx, m->w[k], 0.0f, &wd);
        if (st != SK_OK) fail(st, sk_last_error());
      }
      dense_gemm(ctx, cached ? nullptr : wd->d, src, nn, nn, n, m->bias + size_t(k) * nn,
                 bufs[cur]->d, pc, 0);
      if (!cached) sk_dense_free(wd);
      src = bufs[cur]->d;
      cur ^= 1;
    }
    sk_dense_free(bufs[cur]);
    *out = bufs[cur ^ 1];
  });
}
