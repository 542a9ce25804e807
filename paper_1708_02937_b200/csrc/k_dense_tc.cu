// Dense GEMM for the comparator leg, C[M,N] = A[M,K] . B[K,N] (+ bias, ReLU).
//
// Interim CUDA-core implementation (exact ascending-k fold, bitwise equal to
// the reference's dense_mxm_baseline, matrix.cpp:564-585).  The tcgen05
// tensor-core kernel replaces it; see DESIGN.md "K4".
#include "sk_common.cuh"

namespace sk {

__global__ void __launch_bounds__(256)
    k_gemm_cuda_core(const float* __restrict__ a, const float* __restrict__ b, uint32_t M,
                     uint32_t K, uint32_t N, const float* __restrict__ bias, int relu,
                     float* __restrict__ c) {
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t row0 = blockIdx.y * 32, col = blockIdx.x * 32 + tx;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (uint32_t k0 = 0; k0 < K; k0 += 32) {
    for (uint32_t r = ty; r < 32; r += 8) {
      const uint32_t gi = row0 + r, gk = k0 + tx;
      As[r][tx] = (gi < M && gk < K) ? a[size_t(gi) * K + gk] : 0.0f;
      const uint32_t bk = k0 + r;
      Bs[r][tx] = (bk < K && col < N) ? b[size_t(bk) * N + col] : 0.0f;
    }
    __syncthreads();
    const uint32_t kmax = min(32u, K - k0);
    for (uint32_t kk = 0; kk < kmax; ++kk) {
      const float bv = Bs[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(As[ty + 8 * q][kk], bv));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t gi = row0 + ty + 8 * q;
    if (gi < M && col < N) {
      float z = acc[q];
      if (bias) z = __fadd_rn(z, bias[gi]);
      if (relu) z = (z < 0.0f) ? 0.0f : z;
      c[size_t(gi) * N + col] = z;
    }
  }
}

void launch_dense_gemm_tc(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K,
                          uint32_t N, const float* bias, int relu, float* c) {
  if (M == 0 || N == 0) return;
  dim3 grid(ceil_div(N, 32), ceil_div(M, 32));
  SK_LAUNCH(k_gemm_cuda_core, grid, 256, 0, ctx->stream, a, b, M, K, N, bias, relu, c);
}

}  // namespace sk
