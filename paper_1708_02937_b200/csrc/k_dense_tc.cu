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
// Two kernels (SK_TC_VER selects; 3 is the default):
//  * v3 (k_pack_split + k_gemm_packed): each operand is split ONCE by a pack
//    kernel that writes hi/lo directly in the canonical K-major UMMA layout,
//    tile by tile; the GEMM is a pure pipeline -- one producer thread issues
//    four 1-D cp.async.bulk copies per 16-k stage into a 4-stage shared-memory
//    ring (completion counted on the stage mbarrier), one thread issues the
//    3 x 2 tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=256, K=8) and commits
//    to the stage's "empty" barrier, four warps drain the TMEM accumulator
//    (bias + ReLU fused).  Tensor pipe ~93 % active (profiles/r01/k4_packed_*).
//  * v1 (k_gemm_tf32x3, SK_TC_VER=1 or SK_TC_DBG): one CTA per 128x128 tile,
//    all threads load, split and store each slab (register double buffering),
//    one thread issues the MMAs; kept for bring-up/debug (descriptor overrides).
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "sk_async.cuh"
#include "sk_common.cuh"

namespace sk {
namespace tc {

using async::smem_u32;
using async::mbar_init;
using async::mbar_wait;
using async::mbar_expect_tx;
using async::bulk_g2s;


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

// ---- v3: pre-split operands, bulk-copy pipeline -----------------------------------------
// Splitting inside the GEMM repeats the work once per tile visit (every B tile
// is split M/128 times) and that staging, not the tensor core, bounds v1/v2.
// v3 splits each operand ONCE: a pack kernel writes hi and lo copies directly
// in the canonical K-major UMMA layout, tile by tile (tile = TR rows x 16 k,
// 8-row x 16-byte core matrices, LBO = 128 B, SBO = 512 B), so a stage of the
// GEMM is four contiguous 1-D bulk copies (cp.async.bulk, completion counted on
// the stage's mbarrier) and no thread touches the data on its way to the MMA.
// Warp roles: 0 producer (one thread), 1 MMA issuer (one thread), 2..5
// epilogue (TMEM lanes 32*(w%4)).
constexpr uint32_t kPK = 16;                // k per packed tile
constexpr uint32_t kPLBO = 128, kPSBO = 512;

// Packed tile of rows [tr*TR, tr*TR+TR) x k [tk*16, tk*16+16) at
// (tr * nkt + tk) * TR * 64 bytes.  src(r, k) = transposed ? X[k*ld + r] : X[r*ld + k].
// One warp = 32 rows x 16 k = a contiguous 2 KB span of one packed tile; lane =
// (8-row group g8, k-chunk kk, row half rg) owns a 4 x 4 block: four float4
// loads (along k, or along rows when transposed), an in-register transpose for
// the transposed source, and four consecutive 16-byte stores per copy.
__global__ void k_pack_split(const float* __restrict__ X, uint32_t rows, uint32_t K, uint32_t ld,
                             int transposed, uint32_t TR, uint32_t rows_pad, uint32_t K_pad,
                             float* __restrict__ hi, float* __restrict__ lo) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nkt = K_pad / kPK, nr32 = rows_pad / 32;
  const uint64_t units = uint64_t(nr32) * nkt;
  const uint64_t gw = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t g8 = lane >> 3, kk = (lane >> 1) & 3, rg = lane & 1;
  for (uint64_t u = gw; u < units; u += nw) {
    uint32_t r32, tk;
    if (transposed) {  // consecutive warps: consecutive rows (contiguous source rows)
      r32 = uint32_t(u % nr32);
      tk = uint32_t(u / nr32);
    } else {           // consecutive warps: consecutive k of the same rows
      tk = uint32_t(u % nkt);
      r32 = uint32_t(u / nkt);
    }
    const uint32_t r = r32 * 32 + g8 * 8 + rg * 4, k = tk * kPK + kk * 4;
    float v[4][4];  // v[i][q] = element (row r+i, k+q)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[i][q] = 0.0f;
    if (transposed) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (k + q < K) {
          const float* src = X + size_t(k + q) * ld + r;
          if (r + 3 < rows && (ld & 3) == 0) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(src));
            v[0][q] = t.x; v[1][q] = t.y; v[2][q] = t.z; v[3][q] = t.w;
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) if (r + i < rows) v[i][q] = __ldg(src + i);
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (r + i < rows) {
          const float* src = X + size_t(r + i) * ld + k;
          if (k + 3 < K && (ld & 3) == 0) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(src));
            v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) if (k + q < K) v[i][q] = __ldg(src + q);
          }
        }
      }
    }
    const uint32_t tr = r / TR, rr = r % TR;  // rr % 8 is 0 or 4: rows r..r+3 share a group
    const size_t off = (size_t(tr) * nkt + tk) * (TR * kPK) +
                       ((rr >> 3) * kPSBO + kk * kPLBO + (rr & 7) * 16) / 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float h[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split(v[i][q], h[q], l[q]);
      *reinterpret_cast<float4*>(hi + off + 4 * i) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(lo + off + 4 * i) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
}

template <int BN_, int NS>
struct Cfg3 {
  static constexpr uint32_t kA = BM * kPK * 4;    // 8 KB
  static constexpr uint32_t kB = BN_ * kPK * 4;   // 16 KB at BN = 256
  static constexpr uint32_t kStage = 2 * kA + 2 * kB;
  static constexpr uint32_t kSmem = NS * kStage + 1024;
  static constexpr uint32_t kTmemCols = BN_ <= 128 ? 128 : 256;
  static constexpr int kThreads = 6 * 32;
};

template <int BN_, int NS>
__global__ void __launch_bounds__(6 * 32, 1)
    k_gemm_packed(const float* __restrict__ a_hi, const float* __restrict__ a_lo,
                  const float* __restrict__ b_hi, const float* __restrict__ b_lo, uint32_t M,
                  uint32_t N, uint32_t nkt, const float* __restrict__ bias, int relu,
                  float* __restrict__ C) {
  using G = Cfg3<BN_, NS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[NS], empty[NS], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t mt = blockIdx.y, nt = blockIdx.x;
  const uint32_t m0 = mt * BM, n0 = nt * BN_;
  const uint32_t sbase = (smem_u32(smem) + 1023) & ~1023u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)), "r"(G::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer
      const float* ah = a_hi + size_t(mt) * nkt * (BM * kPK);
      const float* al = a_lo + size_t(mt) * nkt * (BM * kPK);
      const float* bh = b_hi + size_t(nt) * nkt * (BN_ * kPK);
      const float* bl = b_lo + size_t(nt) * nkt * (BN_ * kPK);
      for (uint32_t t = 0; t < nkt; ++t) {
        const uint32_t s = t % NS;
        if (t >= NS) mbar_wait(smem_u32(&empty[s]), ((t / NS) - 1) & 1);
        const uint32_t st = sbase + s * G::kStage, fb = smem_u32(&full[s]);
        mbar_expect_tx(fb, G::kStage);
        bulk_g2s(st, ah + size_t(t) * (BM * kPK), G::kA, fb);
        bulk_g2s(st + G::kA, al + size_t(t) * (BM * kPK), G::kA, fb);
        bulk_g2s(st + 2 * G::kA, bh + size_t(t) * (BN_ * kPK), G::kB, fb);
        bulk_g2s(st + 2 * G::kA + G::kB, bl + size_t(t) * (BN_ * kPK), G::kB, fb);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = idesc_tf32(BM, BN_);
      for (uint32_t t = 0; t < nkt; ++t) {
        const uint32_t s = t % NS;
        mbar_wait(smem_u32(&full[s]), (t / NS) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = sbase + s * G::kStage;
        const uint32_t ah = st, al = st + G::kA, bh = st + 2 * G::kA, bl = st + 2 * G::kA + G::kB;
#pragma unroll
        for (uint32_t kk = 0; kk < kPK / 8; ++kk) {
          const uint32_t o = kk * 2 * kPLBO;
          const uint32_t acc0 = (t | kk) ? 1u : 0u;
          mma_tf32(tmem, umma_desc(ah + o, kPLBO, kPSBO), umma_desc(bh + o, kPLBO, kPSBO), idesc,
                   acc0);
          mma_tf32(tmem, umma_desc(ah + o, kPLBO, kPSBO), umma_desc(bl + o, kPLBO, kPSBO), idesc,
                   1u);
          mma_tf32(tmem, umma_desc(al + o, kPLBO, kPSBO), umma_desc(bh + o, kPLBO, kPSBO), idesc,
                   1u);
        }
        mma_commit(smem_u32(&empty[s]));
      }
      mma_commit(smem_u32(&done));
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5: TMEM lanes 32*(warp%4)
    mbar_wait(smem_u32(&done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t quarter = uint32_t(warp & 3);
    const uint32_t row = m0 + quarter * 32 + lane;
    const float b = (bias && row < M) ? bias[row] : 0.0f;
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < uint32_t(BN_); c0 += 32) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((quarter * 32) << 16) + c0;
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
      if (row < M) {
        float* dst = C + size_t(row) * N + n0 + c0;
        const bool vec = (N & 3) == 0 && n0 + c0 + 32 <= N;
        float z[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          z[q] = __uint_as_float(r[q]);
          if (bias) z[q] = __fadd_rn(z[q], b);
          if (relu) z[q] = (z[q] < 0.0f) ? 0.0f : z[q];
        }
        if (vec) {
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            *reinterpret_cast<float4*>(dst + q) = make_float4(z[q], z[q + 1], z[q + 2], z[q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (n0 + c0 + q < N) dst[q] = z[q];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::kTmemCols)
                 : "memory");
}

}  // namespace tc

void launch_dense_gemm_tc(sk_ctx* ctx, const float* a, const float* b, uint32_t M, uint32_t K,
                          uint32_t N, const float* bias, int relu, float* c, PackCache* cache,
                          uint64_t version) {
  if (M == 0 || N == 0) return;
  {
    // v3 kernel: pack (split once) + bulk-copy pipeline
    constexpr int BNp = 256, NSp = 4;
    using G = tc::Cfg3<BNp, NSp>;
    const uint32_t Mp = ceil_div(M, tc::BM) * tc::BM, Np = ceil_div(N, BNp) * BNp;
    const uint32_t Kp = ceil_div(K, tc::kPK) * tc::kPK;
    // A's packed halves: from the owner's cache when it is current, else packed
    // here (and kept in the cache when there is one)
    const bool hit = cache && cache->buf && cache->version == version;
    if (cache && !hit && cache->buf) {
      dfree(ctx, cache->buf);
      cache->buf = nullptr;
    }
    float* abuf = hit ? cache->buf : dalloc<float>(ctx, 2 * size_t(Mp) * Kp);
    float* buf = dalloc<float>(ctx, 2 * size_t(Np) * Kp);
    float* ahi = abuf;
    float* alo = ahi + size_t(Mp) * Kp;
    float* bhi = buf;
    float* blo = bhi + size_t(Np) * Kp;
    smem_attr(ctx, tc::k_gemm_packed<BNp, NSp>, int(G::kSmem));
    timing_mark(ctx, SK_KT_GEMM_TC);
    const uint64_t wa = uint64_t(Mp / 32) * (Kp / tc::kPK), wb = uint64_t(Np / 32) * (Kp / tc::kPK);
    if (!hit)
      SK_LAUNCH(tc::k_pack_split,
                unsigned(std::min<uint64_t>((wa + 7) / 8, uint64_t(ctx->num_sms) * 16)), 256, 0,
                ctx->stream, a, M, K, K, 0, tc::BM, Mp, Kp, ahi, alo);
    if (cache && !hit) {
      cache->buf = abuf;
      cache->version = version;
    }
    SK_LAUNCH(tc::k_pack_split,
              unsigned(std::min<uint64_t>((wb + 7) / 8, uint64_t(ctx->num_sms) * 16)), 256, 0,
              ctx->stream, b, N, K, N, 1, uint32_t(BNp), Np, Kp, bhi, blo);
    dim3 g3(Np / BNp, Mp / tc::BM);
    SK_LAUNCH((tc::k_gemm_packed<BNp, NSp>), g3, G::kThreads, G::kSmem, ctx->stream, ahi, alo,
              bhi, blo, M, N, Kp / tc::kPK, bias, relu, c);
    timing_mark(ctx);
    dfree(ctx, buf);
    if (!cache) dfree(ctx, abuf);
  }
}

}  // namespace sk
