// K1: CSR x dense SpMM on neuron-major activations, with the layer epilogue
// fused (proj/src/matrix.cpp:403-424 + proj/src/dnn.cpp:65-103).
//
// Bitwise contract (SURVEY §8a "Op order"): every output (i, j) is a LEFT FOLD
// over the stored entries of W_ref row i in ascending column order, starting
// from the semiring zero, with separately rounded multiply and add
// (__fmul_rn/__fadd_rn -- never contracted to FMA).  Each output element has
// exactly one owner lane, so there is no split-K and no atomic anywhere.
//
// Mapping: one warp owns (row i, 128-column chunk c); each lane owns 4
// consecutive columns and streams float4 rows of Y.  The warp loads 32 (k, w)
// pairs of W row i cooperatively and broadcasts them with shuffles, so the
// inner loop issues only the Y loads.  Tasks are ordered chunk-major so the
// live Y panel (m x 128 floats) stays L2-resident while every row that
// touches it runs.
#include <cooperative_groups.h>

#include "sk_common.cuh"

namespace cg = cooperative_groups;

namespace sk {

enum EpiMode { kEpiNone = 0, kEpiLayer = 1 };

// kU: 128-column chunks per task (a lane owns 4 columns of each).  Light rows
// (few stored entries) take kU = 4: the row's (k, w) pairs are loaded once for
// 512 columns and every entry issues four independent float4 loads, so a task
// is not a chain of dependent round trips per 128 columns.
template <typename Ops, int kEpi, bool kVec4, int kU = 1>
__device__ __forceinline__ void spmm_tasks(const uint32_t* __restrict__ rp,
                                           const uint32_t* __restrict__ ci,
                                           const float* __restrict__ wv,
                                           const float* __restrict__ bias,
                                           const float* __restrict__ y, uint32_t m, uint32_t n,
                                           float clip, float* __restrict__ out, int* err,
                                           unsigned long long* nz_count = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t nz = 0;  // nonzero outputs written by this lane (only when nz_count)
  const uint32_t chunks = (n + 128 * kU - 1) / (128 * kU);
  const uint64_t tasks = uint64_t(chunks) * m;
  for (uint64_t task = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; task < tasks;
       task += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t c = uint32_t(task / m);
    const uint32_t i = uint32_t(task % m);
    float acc[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[u][q] = Ops::zero();
    const uint32_t eb = rp[i], ee = rp[i + 1];
    for (uint32_t e0 = eb; e0 < ee; e0 += 32) {
      const uint32_t cnt = min(32u, ee - e0);
      uint32_t kk = 0;
      float aa = 0.0f;
      if (uint32_t(lane) < cnt) {
        kk = ci[e0 + lane];
        aa = wv[e0 + lane];
      }
#pragma unroll 4
      for (uint32_t t = 0; t < cnt; ++t) {
        const uint32_t k = __shfl_sync(0xffffffffu, kk, t);
        const float a = __shfl_sync(0xffffffffu, aa, t);
        const float* yr = y + size_t(k) * n;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t col0 = (c * kU + u) * 128 + lane * 4;
          if (kVec4) {
            if (col0 < n) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(yr + col0));
              acc[u][0] = Ops::add(acc[u][0], Ops::mul(a, v.x, err), err);
              acc[u][1] = Ops::add(acc[u][1], Ops::mul(a, v.y, err), err);
              acc[u][2] = Ops::add(acc[u][2], Ops::mul(a, v.z, err), err);
              acc[u][3] = Ops::add(acc[u][3], Ops::mul(a, v.w, err), err);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (col0 + q < n) acc[u][q] = Ops::add(acc[u][q], Ops::mul(a, yr[col0 + q], err), err);
          }
        }
      }
    }
    float b = 0.0f;
    if (kEpi == kEpiLayer) b = bias[i];
    float* orow = out + size_t(i) * n;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t col0 = (c * kU + u) * 128 + lane * 4;
      if (kEpi == kEpiLayer)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[u][q] = layer_epilogue(acc[u][q], b, clip);
      if (nz_count)
#pragma unroll
        for (int q = 0; q < 4; ++q) nz += (col0 + q < n && acc[u][q] != 0.0f) ? 1u : 0u;
      if (kVec4) {
        if (col0 < n)
          *reinterpret_cast<float4*>(orow + col0) =
              make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (col0 + q < n) orow[col0 + q] = acc[u][q];
      }
    }
  }
  if (nz_count) {  // warp-uniform: nz_count is a kernel argument
#pragma unroll
    for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    if (lane == 0 && nz) atomicAdd(nz_count, (unsigned long long)nz);
  }
}

template <typename Ops, int kEpi, bool kVec4, int kU = 1>
__global__ void __launch_bounds__(256)
    k_spmm_rows(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                const float* __restrict__ wv, const float* __restrict__ bias,
                const float* __restrict__ y, uint32_t m, uint32_t n, float clip,
                float* __restrict__ out, int* err) {
  spmm_tasks<Ops, kEpi, kVec4, kU>(rp, ci, wv, bias, y, m, n, clip, out, err);
}

// The whole dense-activation forward in ONE persistent cooperative launch: each
// layer is the K1 task loop, layers are separated by a grid barrier (every
// output column of layer k+1 needs the whole of Y_k).  Removes the per-layer
// launch latency that dominates small models (BASELINE cfg1).
//
// Density-adaptive mode (nnz != nullptr): every layer also counts its nonzero
// outputs; when a layer's count drops below stop_below the engine stops after
// that layer (every block reads the same count after the barrier, so the
// decision is uniform) and the host continues on the sparse engine.
struct DenseEngineArgs {
  const uint32_t* const* w_rp;
  const uint32_t* const* w_ci;
  const float* const* w_v;
  const float* bias;
  uint32_t m, n, L;
  float clip;
  const float* y0;
  float* buf[2];
  int* err;
  unsigned long long* nnz;         // L counters, zeroed (optional)
  unsigned long long stop_below;   // 0 = never stop early
  int* layers_done;                // written when stopping early
};

template <bool kVec4>
__global__ void __launch_bounds__(256) k_dense_engine(DenseEngineArgs p) {
  cg::grid_group grid = cg::this_grid();
  for (uint32_t k = 0; k < p.L; ++k) {
    const float* src = k == 0 ? p.y0 : p.buf[(k - 1) & 1];
    float* dst = p.buf[k & 1];
    spmm_tasks<OpArith, kEpiLayer, kVec4>(p.w_rp[k], p.w_ci[k], p.w_v[k], p.bias + size_t(k) * p.m,
                                          src, p.m, p.n, p.clip, dst, p.err,
                                          p.nnz ? p.nnz + k : nullptr);
    if (k + 1 < p.L) {
      grid.sync();
      if (p.stop_below && *(volatile unsigned long long*)(p.nnz + k) < p.stop_below) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *p.layers_done = int(k + 1);
        return;
      }
    }
  }
}

static unsigned spmm_grid(sk_ctx* ctx, uint32_t m, uint32_t n, int U = 1) {
  const uint64_t warps = uint64_t((n + 128 * U - 1) / (128 * U)) * m;
  const uint64_t blocks = (warps + 7) / 8;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(ctx->num_sms) * 16)));
}

// Dense forward over layers [k0, L) of a model (layer k0 + j writes buffer j & 1).
// With nnz != nullptr (L - k0 zeroed device counters) each layer's nonzero count
// is recorded and the engine stops after the first layer whose count is below
// stop_below (> 0); *d_done (device) then holds the number of layers run.
void dense_forward_engine(sk_ctx* ctx, const sk_model* md, uint32_t k0, const float* y0,
                          uint32_t n, float clip, float* buf0, float* buf1,
                          unsigned long long* nnz, unsigned long long stop_below, int* d_done) {
  auto* mm = const_cast<sk_model*>(md);
  const uint32_t L = md->layers, m = md->neurons;
  ensure_model_tables(ctx, mm);
  DenseEngineArgs p;
  p.w_rp = reinterpret_cast<const uint32_t* const*>(mm->d_wptr) + k0;
  p.w_ci = reinterpret_cast<const uint32_t* const*>(mm->d_wptr + L) + k0;
  p.w_v = reinterpret_cast<const float* const*>(mm->d_wptr + 2 * L) + k0;
  p.bias = md->bias + size_t(k0) * m;
  p.m = m;
  p.n = n;
  p.L = L - k0;
  p.clip = clip;
  p.y0 = y0;
  p.buf[0] = buf0;
  p.buf[1] = buf1;
  p.err = ctx->d_err;
  p.nnz = nnz;
  p.stop_below = nnz ? stop_below : 0;
  p.layers_done = d_done;
  const bool vec = (n % 4) == 0;
  const void* fn = vec ? (const void*)k_dense_engine<true> : (const void*)k_dense_engine<false>;
  const int per_sm = kernel_occupancy(ctx, fn, 256, 0);  // cached per device
  const uint64_t warps = uint64_t((n + 127) / 128) * m;
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((warps + 7) / 8, uint64_t(ctx->num_sms) * std::max(per_sm, 1))));
  void* args[] = {&p};
  timing_mark(ctx, SK_KT_DENSE_ENGINE);
  SK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, ctx->stream));
  g_launches.fetch_add(1);
  timing_mark(ctx);
}

void launch_layer_dense(sk_ctx* ctx, const sk_csr* w, const float* d_bias, const float* y,
                        uint32_t n, float clip, float* out) {
  if (w->rows == 0 || n == 0) return;
  const bool vec = (n % 4 == 0);
  // light rows (<= 16 stored entries on average) and wide activations: four
  // 128-column chunks per task
  const bool light = vec && n >= 512 && w->nnz <= size_t(16) * w->rows;
  if (light)
    SK_LAUNCH((k_spmm_rows<OpArith, kEpiLayer, true, 4>), spmm_grid(ctx, w->rows, n, 4), 256, 0,
              ctx->stream, w->rp, w->ci, w->v, d_bias, y, w->rows, n, clip, out, ctx->d_err);
  else if (vec)
    SK_LAUNCH((k_spmm_rows<OpArith, kEpiLayer, true>), spmm_grid(ctx, w->rows, n), 256, 0,
              ctx->stream, w->rp, w->ci, w->v, d_bias, y, w->rows, n, clip, out, ctx->d_err);
  else
    SK_LAUNCH((k_spmm_rows<OpArith, kEpiLayer, false>), spmm_grid(ctx, w->rows, n), 256, 0,
              ctx->stream, w->rp, w->ci, w->v, d_bias, y, w->rows, n, clip, out, ctx->d_err);
}

void launch_mxm_csr_dense(sk_ctx* ctx, const sk_csr* a, const float* b, uint32_t n,
                          sk_semiring s, float* out) {
  if (a->rows == 0 || n == 0) return;
  dispatch_semiring(s, [&](auto ops) {
    using Ops = decltype(ops);
    if (n % 4 == 0)
      SK_LAUNCH((k_spmm_rows<Ops, kEpiNone, true>), spmm_grid(ctx, a->rows, n), 256, 0,
                ctx->stream, a->rp, a->ci, a->v, nullptr, b, a->rows, n, 0.0f, out, ctx->d_err);
    else
      SK_LAUNCH((k_spmm_rows<Ops, kEpiNone, false>), spmm_grid(ctx, a->rows, n), 256, 0,
                ctx->stream, a->rp, a->ci, a->v, nullptr, b, a->rows, n, 0.0f, out, ctx->d_err);
  });
}

// ---- dense x dense over a semiring (matrix.cpp:426-447), exact ascending-k fold ----
// 32x32 output tile per block; K staged through shared memory in 32-wide slabs.
template <typename Ops>
__global__ void __launch_bounds__(256)
    k_mxm_dense_dense(const float* __restrict__ a, const float* __restrict__ b, uint32_t M,
                      uint32_t K, uint32_t N, float* __restrict__ c, int* err) {
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const uint32_t row0 = blockIdx.y * 32, col = blockIdx.x * 32 + tx;
  float acc[4] = {Ops::zero(), Ops::zero(), Ops::zero(), Ops::zero()};
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
      for (int q = 0; q < 4; ++q) acc[q] = Ops::add(acc[q], Ops::mul(As[ty + 8 * q][kk], bv, err), err);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t gi = row0 + ty + 8 * q;
    if (gi < M && col < N) c[size_t(gi) * N + col] = acc[q];
  }
}

void launch_mxm_dense_dense(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K,
                            uint32_t N, sk_semiring s, float* c) {
  if (M == 0 || N == 0) return;
  dim3 grid(ceil_div(N, 32), ceil_div(M, 32));
  dispatch_semiring(s, [&](auto ops) {
    using Ops = decltype(ops);
    SK_LAUNCH(k_mxm_dense_dense<Ops>, grid, 256, 0, ctx->stream, a, b, M, K, N, c, ctx->d_err);
  });
}

}  // namespace sk

using namespace sk;

static void require_inner(const char* op, uint32_t ac, uint32_t br) {
  // matrix.cpp:40-46
  if (ac != br)
    fail(SK_ERR_DIMENSION, std::string(op) + ": inner dimensions " + std::to_string(ac) +
                               " and " + std::to_string(br) + " do not match");
}

extern "C" sk_status sk_mxm_csr_dense(sk_ctx* ctx, const sk_csr* a, const sk_dense* b,
                                      sk_semiring s, sk_dense** out) {
  return guarded([&] {
    csr_ready(ctx, a);
    SK_CUDA(cudaSetDevice(ctx->device));
    require_inner("mxm", a->cols, b->rows);
    sk_dense* o = new_dense(ctx, a->rows, b->cols);
    launch_mxm_csr_dense(ctx, a, b->d, b->cols, s, o->d);
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, "mxm");
      } catch (...) {
        sk_dense_free(o);
        throw;
      }
    }
    *out = o;
  });
}

extern "C" sk_status sk_mxm_dense_dense(sk_ctx* ctx, const sk_dense* a, const sk_dense* b,
                                        sk_semiring s, sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    require_inner("mxm", a->cols, b->rows);
    sk_dense* o = new_dense(ctx, a->rows, b->cols);
    launch_mxm_dense_dense(ctx, a->d, b->d, a->rows, a->cols, b->cols, s, o->d);
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, "mxm");
      } catch (...) {
        sk_dense_free(o);
        throw;
      }
    }
    *out = o;
  });
}

extern "C" sk_status sk_mxm_csr_csr(sk_ctx* ctx, const sk_csr* a, const sk_csr* b,
                                    sk_semiring s, sk_csr** out) {
  return guarded([&] {
    csr_ready(ctx, a);
    csr_ready(ctx, b);
    SK_CUDA(cudaSetDevice(ctx->device));
    require_inner("mxm", a->cols, b->rows);
    sk_csr* o = mxm_csr_csr_impl(ctx, a, b, s);
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, "mxm");
      } catch (...) {
        csr_release(o);
        throw;
      }
    }
    *out = o;
  });
}
