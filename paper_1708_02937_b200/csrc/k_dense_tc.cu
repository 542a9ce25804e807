// K4: dense GEMM on the 5th-generation tensor cores for the dense comparator
// leg -- dense_mxm_baseline / dense_layer_step / dense_relu_forward
// (proj/src/matrix.cpp:564-585, proj/src/dnn.cpp:123-149):
//     C[M,N] = A[M,K] . B[K,N]  (+ bias[M], ReLU)      all fp32, row-major.
//
// Precision: fp32-class via 3xTF32.  Every operand x is split into
// hi = rna_tf32(x) and lo = x - hi (exact), and the tile product is
// hi.hi + hi.lo + lo.hi accumulated in fp32 in TMEM (the dropped lo.lo term
// and lo's own tf32 truncation are ~2^-21 relative).  The result is therefore
// within kRelTol of the reference's scalar fold when measured against the
// magnitude sum_k |a||b| (approx_equal_scaled, semiring.hpp:50-55) -- the
// tensor core can never reproduce the fp32 fold bitwise, which is why the
// sparse leg (K1/K3) is the bitwise path and this leg is tolerance-checked.
//
// Structure (one CTA = one 128x128 output tile, 4 warps):
//  * mainloop over K in 32-wide slabs, two smem stages.  All 128 threads load
//    the A (128x32) and B (32x128, staged transposed) slabs, both K-major,
//    split them, and store hi/lo copies in the no-swizzle canonical UMMA
//    layouts (8-row x 16-byte core matrices); fence.proxy.async makes the
//    generic-proxy writes visible to the tensor core;
//  * one elected thread issues 3 x 4 tcgen05.mma.cta_group::1.kind::tf32
//    (M=128, N=128, K=8) per slab and tcgen05.commit's them to the stage's
//    mbarrier, so loading slab t+1 overlaps the MMAs of slab t;
//  * epilogue: each warp reads its 32 TMEM lanes (= 32 output rows) with
//    tcgen05.ld.32x32b.x32, adds the bias, applies the ReLU select, stores.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "sk_common.cuh"

namespace sk {
namespace tc {

constexpr int BM = 128, BN = 128;
constexpr int kThreads = 128;
template <int BK>
struct Cfg {
  static constexpr uint32_t kTileBytes = BM * BK * 4;      // A (128 x BK) and B (BK x 128)
  static constexpr uint32_t kStageBytes = 4 * kTileBytes;  // A_hi, A_lo, B_hi, B_lo
  static constexpr uint32_t kSmemBytes = 2 * kStageBytes + 64;
  static constexpr uint32_t KC = BK / 4;                   // 16-byte k-chunks per row
  static constexpr uint32_t KC_LOG = KC == 8 ? 3 : (KC == 4 ? 2 : 1);
  // core matrix (kc, row group) = 8 rows x 4 k at group*SBO + kc*LBO; B is staged
  // K-major as well (B^T tile: n rows x k).  An MN-major fp32/tf32 operand would
  // need the 128B_BASE32B swizzle.
  static constexpr uint32_t LBO = 128, SBO = KC * 128;
};
constexpr uint32_t kA_LBO = 128, kA_SBO = 1024, kB_LBO = 128, kB_SBO = 1024;  // BK = 32

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // descriptor version 1 (sm_100); base offset 0; no swizzle
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                 // c_format = F32
         | (2u << 7)               // a_format = TF32
         | (2u << 10)              // b_format = TF32
         | (0u << 15)              // a_major = K
         | (0u << 16)              // b_major = K
         | (uint32_t(n >> 3) << 17)
         | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = rna_tf32(x);
  lo = __fsub_rn(x, hi);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

struct TcParams {  // descriptor fields, overridable for bring-up (SK_TC_DBG)
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo, idesc;
  uint32_t mode;  // 0 normal; 1 TMEM st/ld self-test (no MMA); 2 delay after wait
};

template <int BK>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tf32x3(const float* __restrict__ A, const float* __restrict__ B, uint32_t M,
                  uint32_t K, uint32_t N, const float* __restrict__ bias, int relu,
                  float* __restrict__ C, TcParams tp) {
  using G = Cfg<BK>;
  constexpr uint32_t kTileBytes = G::kTileBytes, kStageBytes = G::kStageBytes;
  constexpr uint32_t KC = G::KC, KC_LOG = G::KC_LOG;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const uint32_t sbase = smem_u32(smem);

  if (warp == 0) {
    // 128 fp32 accumulator columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(&tmem_base_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_slot;
  const uint32_t idesc = tp.idesc;

  const uint32_t nk = tp.mode == 1 ? 0u : (K + BK - 1) / BK;
  if (tp.mode == 1) {
    for (uint32_t c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = __float_as_uint(float((warp * 32 + lane) * 1000 + c0 + q));
      const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + c0;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\t"
          "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
          "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
          "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
          "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
    }
  }
  // Register double buffering: the global loads of slab t+1 are issued before
  // slab t is split/stored and its MMAs run, so their latency overlaps the
  // tensor-core work instead of being exposed once per slab.
  constexpr int NJ = int(KC);  // 16-byte chunks per thread per operand (128*KC/128)
  float4 ra[NJ];
  float rb[NJ][4];
  auto load_slab = [&](uint32_t t) {
    const uint32_t k0 = t * BK;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint32_t c = uint32_t(j) * kThreads + tid;
      const uint32_t kc = (c >> 3) & (KC - 1), r = (c >> (3 + KC_LOG)) * 8 + (c & 7);
      const uint32_t gr = m0 + r, gk = k0 + kc * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < M) {
        const float* src = A + size_t(gr) * K + gk;
        if (gk + 3 < K && (K & 3) == 0) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (gk + 0 < K) v.x = __ldg(src + 0);
          if (gk + 1 < K) v.y = __ldg(src + 1);
          if (gk + 2 < K) v.z = __ldg(src + 2);
          if (gk + 3 < K) v.w = __ldg(src + 3);
        }
      }
      ra[j] = v;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint32_t c = uint32_t(j) * kThreads + tid;
      const uint32_t nr = (c & 31) + 32 * ((c >> 5) & 3);
      const uint32_t kc = c >> 7;
      const uint32_t gn = n0 + nr, gk = k0 + kc * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        rb[j][q] = (gn < N && gk + q < K) ? __ldg(B + size_t(gk + q) * N + gn) : 0.0f;
    }
  };
  auto store_slab = [&](uint32_t st) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint32_t c = uint32_t(j) * kThreads + tid;
      const uint32_t kc = (c >> 3) & (KC - 1), r = (c >> (3 + KC_LOG)) * 8 + (c & 7);
      float h[4], l[4];
      split(ra[j].x, h[0], l[0]);
      split(ra[j].y, h[1], l[1]);
      split(ra[j].z, h[2], l[2]);
      split(ra[j].w, h[3], l[3]);
      const uint32_t off = (r >> 3) * G::SBO + kc * G::LBO + (r & 7) * 16;
      st_shared_v4(st + off, h[0], h[1], h[2], h[3]);
      st_shared_v4(st + kTileBytes + off, l[0], l[1], l[2], l[3]);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint32_t c = uint32_t(j) * kThreads + tid;
      const uint32_t nr = (c & 31) + 32 * ((c >> 5) & 3);
      const uint32_t kc = c >> 7;
      float h[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split(rb[j][q], h[q], l[q]);
      const uint32_t off = (nr >> 3) * G::SBO + kc * G::LBO + (nr & 7) * 16;
      st_shared_v4(st + 2 * kTileBytes + off, h[0], h[1], h[2], h[3]);
      st_shared_v4(st + 3 * kTileBytes + off, l[0], l[1], l[2], l[3]);
    }
  };
  if (nk > 0) load_slab(0);
  for (uint32_t t = 0; t < nk; ++t) {
    const uint32_t s = t & 1;
    if (t >= 2) mbar_wait(smem_u32(&mbar[s]), ((t - 2) >> 1) & 1);
    const uint32_t st = sbase + s * kStageBytes;
    store_slab(st);
    if (t + 1 < nk) load_slab(t + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = st, a_lo = st + kTileBytes, b_hi = st + 2 * kTileBytes,
                     b_lo = st + 3 * kTileBytes;
#pragma unroll
      for (uint32_t kk = 0; kk < BK / 8; ++kk) {
        // K=8 is two 4-wide k-chunks (LBO apart) for both operands.
        const uint32_t ao = kk * 2 * kA_LBO, bo = kk * 2 * kB_LBO;
        const uint32_t acc0 = (t | kk) ? 1u : 0u;
        const uint32_t asbo = BK == 32 ? tp.a_sbo : G::SBO, bsbo = BK == 32 ? tp.b_sbo : G::SBO;
        mma_tf32(tmem, umma_desc(a_hi + ao, tp.a_lbo, asbo),
                 umma_desc(b_hi + bo, tp.b_lbo, bsbo), idesc, acc0);
        mma_tf32(tmem, umma_desc(a_hi + ao, tp.a_lbo, asbo),
                 umma_desc(b_lo + bo, tp.b_lbo, bsbo), idesc, 1u);
        mma_tf32(tmem, umma_desc(a_lo + ao, tp.a_lbo, asbo),
                 umma_desc(b_hi + bo, tp.b_lbo, bsbo), idesc, 1u);
      }
      mma_commit(smem_u32(&mbar[s]));
    }
  }
  if (nk > 0) mbar_wait(smem_u32(&mbar[(nk - 1) & 1]), ((nk - 1) >> 1) & 1);
  if (tp.mode == 2) {  // bring-up: long delay after the commit wait
    const long long t0 = clock64();
    while (clock64() - t0 < 20000000) {
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- epilogue: warp w owns TMEM lanes / output rows [32w, 32w+32) -------------------
  const uint32_t row = m0 + warp * 32 + lane;
  const float b = (bias && row < M) ? bias[row] : 0.0f;
#pragma unroll 1
  for (uint32_t c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    if (nk > 0 || tp.mode == 1) {
      const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + c0;
      // load and wait in ONE asm block: the destination registers are undefined
      // until tcgen05.wait::ld, so no use may be scheduled in between
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
          "tcgen05.wait::ld.sync.aligned;"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31])
          : "r"(taddr)
          : "memory");
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q) r[q] = 0u;
    }
    if (row < M) {
      float* dst = C + size_t(row) * N + n0 + c0;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t col = n0 + c0 + q;
        if (col < N) {
          float z = __uint_as_float(r[q]);
          if (bias) z = __fadd_rn(z, b);
          if (relu) z = (z < 0.0f) ? 0.0f : z;
          dst[q] = z;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

}  // namespace tc

void launch_dense_gemm_tc(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K,
                          uint32_t N, const float* bias, int relu, float* c) {
  if (M == 0 || N == 0) return;
  static bool attr = false;
  if (!attr) {
    SK_CUDA(cudaFuncSetAttribute(tc::k_gemm_tf32x3<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::Cfg<32>::kSmemBytes));
    SK_CUDA(cudaFuncSetAttribute(tc::k_gemm_tf32x3<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::Cfg<16>::kSmemBytes));
    attr = true;
  }
  static const int bk = [] {
    const char* e = getenv("SK_TC_BK");
    return (e && atoi(e) == 32) ? 32 : 16;
  }();
  dim3 grid(ceil_div(N, tc::BN), ceil_div(M, tc::BM));
  tc::TcParams tp{tc::kA_LBO, tc::kA_SBO, tc::kB_LBO, tc::kB_SBO,
                  tc::idesc_tf32(tc::BM, tc::BN), 0};
  if (const char* e = getenv("SK_TC_DBG")) {  // "a_lbo,a_sbo,b_lbo,b_sbo,idesc_hex,mode"
    unsigned v[6] = {0, 0, 0, 0, 0, 0};
    if (sscanf(e, "%u,%u,%u,%u,%x,%u", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5]) >= 5)
      tp = tc::TcParams{v[0], v[1], v[2], v[3], v[4], v[5]};
  }
  timing_mark(ctx);
  if (bk == 32)
    SK_LAUNCH(tc::k_gemm_tf32x3<32>, grid, tc::kThreads, tc::Cfg<32>::kSmemBytes, ctx->stream, a,
              b, M, K, N, bias, relu, c, tp);
  else
    SK_LAUNCH(tc::k_gemm_tf32x3<16>, grid, tc::kThreads, tc::Cfg<16>::kSmemBytes, ctx->stream, a,
              b, M, K, N, bias, relu, c, tp);
  timing_mark(ctx);
}

}  // namespace sk
