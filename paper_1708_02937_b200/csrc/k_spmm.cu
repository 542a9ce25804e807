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

#include <vector>

#include "sk_async.cuh"
#include "sk_common.cuh"

namespace cg = cooperative_groups;

namespace sk {

enum EpiMode { kEpiNone = 0, kEpiLayer = 1 };

// kU: 128-column chunks per task (a lane owns 4 columns of each).  Light rows
// (few stored entries) take kU = 4: the row's (k, w) pairs are loaded once for
// 512 columns and every entry issues four independent float4 loads, so a task
// is not a chain of dependent round trips per 128 columns.
// kBatch: in-edges whose Y loads are in flight together (registers: 4 kU kBatch)
// (light rows, kU = 4: the four chunks' loads are the batch).  Measured on
// B200 (tools/prof_dense.py, tools/cfg2_sweep.py): 4 in-edges per batch with
// 4 blocks of 256 per SM; 1, 2 and 8 were equal or slower.
#ifndef SK_SPMM_BATCH
#define SK_SPMM_BATCH 4
#endif
#ifndef SK_SPMM_MINB
#define SK_SPMM_MINB 4
#endif
template <typename Ops, int kEpi, bool kVec4, int kU = 1, int kBatch = (kU == 1 ? SK_SPMM_BATCH : 1)>
__device__ __forceinline__ void spmm_tasks(const uint32_t* __restrict__ rp,
                                           const uint32_t* __restrict__ ci,
                                           const float* __restrict__ wv,
                                           const float* __restrict__ bias,
                                           const float* __restrict__ y, uint32_t m, uint32_t n,
                                           float clip, float* __restrict__ out, int* err,
                                           unsigned long long* nz_count = nullptr,
                                           unsigned long long* work = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t nz = 0;  // nonzero outputs written by this lane (only when nz_count)
  const uint32_t chunks = (n + 128 * kU - 1) / (128 * kU);
  const uint64_t tasks = uint64_t(chunks) * m;
  // work (a zeroed counter): tasks claimed in order, one ahead (see K1b)
  const uint64_t stride = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t task = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (work) {
    if (lane == 0) task = atomicAdd(work, 1ull);
    task = __shfl_sync(0xffffffffu, task, 0);
  }
  for (; task < tasks;) {
    unsigned long long claimed = 0;
    if (work && lane == 0) claimed = atomicAdd(work, 1ull);
    // chunk-major: the live Y panel stays in L2 (a 32-bit divide where the
    // task count allows: the 64-bit one is ~100 instructions per task)
    uint32_t c, i;
    if (tasks <= 0xFFFFFFFFull) {
      c = uint32_t(task) / m;
      i = uint32_t(task) - c * m;
    } else {
      c = uint32_t(task / m);
      i = uint32_t(task - uint64_t(c) * m);
    }
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
      // Batches of kBatch in-edges: every Y load of the batch is issued before
      // the first fold step consumes one, so kBatch (x kU) 512-byte row segments
      // per warp are in flight instead of one (the fold itself stays strictly
      // in ascending k).
      for (uint32_t t0 = 0; t0 < cnt; t0 += kBatch) {
        float4 v[kBatch][kU];
        float a[kBatch];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          const uint32_t t = t0 + q;
          const uint32_t k = __shfl_sync(0xffffffffu, kk, t & 31);
          a[q] = __shfl_sync(0xffffffffu, aa, t & 31);
          const float* yr = y + size_t(k) * n;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const uint32_t col0 = (c * kU + u) * 128 + lane * 4;
            v[q][u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < cnt) {
              if (kVec4) {
                if (col0 < n) v[q][u] = __ldg(reinterpret_cast<const float4*>(yr + col0));
              } else {
                if (col0 < n) v[q][u].x = yr[col0];
                if (col0 + 1 < n) v[q][u].y = yr[col0 + 1];
                if (col0 + 2 < n) v[q][u].z = yr[col0 + 2];
                if (col0 + 3 < n) v[q][u].w = yr[col0 + 3];
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          if (t0 + q < cnt) {  // warp-uniform
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              acc[u][0] = Ops::add(acc[u][0], Ops::mul(a[q], v[q][u].x, err), err);
              acc[u][1] = Ops::add(acc[u][1], Ops::mul(a[q], v[q][u].y, err), err);
              acc[u][2] = Ops::add(acc[u][2], Ops::mul(a[q], v[q][u].z, err), err);
              acc[u][3] = Ops::add(acc[u][3], Ops::mul(a[q], v[q][u].w, err), err);
            }
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
    task = work ? __shfl_sync(0xffffffffu, claimed, 0) : task + stride;
  }
  if (nz_count) {  // warp-uniform: nz_count is a kernel argument
#pragma unroll
    for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    if (lane == 0 && nz) atomicAdd(nz_count, (unsigned long long)nz);
  }
}

// ---- K1b: the wide task with its activation segments staged through shared memory -----
// The register-staged wide task waits on its gathered loads with no unit busy
// (ncu: L2 36 %, 40 % of cycles without an eligible warp): what a warp keeps in
// flight is bounded by its registers (4 in-edges x 2 x 16 bytes per lane).  Here
// a lane copies its two 16-byte pieces of every in-edge's 1 KB segment (256
// columns of row k of Y) with cp.async into a warp-private ring of kS stages
// and reads back exactly the bytes it copied, so the pipeline is lane-local: one
// commit group per in-edge, cp.async.wait_group kS - 1 before the fold, no
// barrier and no cross-lane visibility to wait for; kS KB per warp are in flight
// whatever the register budget.  (The bulk-copy engine, one cp.async.bulk per
// segment on an mbarrier ring, measured 43 ms per saturated layer against 15:
// ~100 cycles per 1 KB copy and SM.)  n % 4 == 0 (16-byte aligned segments).
#ifndef SK_BULK_STAGES
#define SK_BULK_STAGES 4
#endif
#ifndef SK_BULK_MINB
#define SK_BULK_MINB 4
#endif
namespace bulk {
constexpr int kS = SK_BULK_STAGES;
constexpr int kWarps = 8;
constexpr size_t kSmem = size_t(kWarps) * kS * 1024;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_pending() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace bulk

template <typename Ops, int kEpi, bool kSrcBlk = false>
__device__ __forceinline__ void spmm_tasks_bulk(const uint32_t* __restrict__ rp,
                                                const uint32_t* __restrict__ ci,
                                                const float* __restrict__ wv,
                                                const float* __restrict__ bias,
                                                const float* __restrict__ y, uint32_t m,
                                                uint32_t n, float clip, float* __restrict__ out,
                                                int* err, unsigned long long* nz_count,
                                                uint8_t* smem, bool dst_blk = false,
                                                unsigned long long* work = nullptr) {
  // work (a zeroed counter): tasks are claimed in order, one ahead, instead of
  // strided statically.  A column panel is only m / (warps in flight) ~ 5 tasks
  // per warp, so statically strided warps drift panels apart within a layer
  // and the L2 stops holding "the" panel: ncu measured 351 GB of DRAM reads for
  // 15.7 GB of activations on four saturated 16384 x 60000 layers (5.8 TB/s:
  // DRAM-bound), 34 GB for 3.9 GB at 15000 samples.  Claimed in order, the
  // tasks in flight are always ~3500 consecutive rows of one panel.
  // kSrcBlk / dst_blk: the activations in PANEL-MAJOR layout -- element (row r,
  // column j) at ((j / 256) * m + r) * 256 + j % 256 -- so the 256-column panel
  // a task sweep gathers from is one contiguous m KB instead of m segments a row
  // pitch apart (16384 x 60000: 3.9 GB spanned per panel, and the gathers' rate
  // fell from 12.8 to 8.8 TB/s between 15000 and 60000 samples).  Square layers
  // only (Y has m rows); the engine keeps its intermediate activations this way.
  using namespace bulk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this lane's 16 bytes of the two halves of every stage
  const float* const mine = reinterpret_cast<const float*>(smem + size_t(warp) * kS * 1024) + lane * 4;
  const uint32_t mine_s = async::smem_u32(mine);
  uint32_t nz = 0;
  const uint32_t chunks = (n + 255) / 256;
  const uint64_t tasks = uint64_t(chunks) * m;
  const uint64_t stride = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t task = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (work) {
    if (lane == 0) task = atomicAdd(work, 1ull);
    task = __shfl_sync(0xffffffffu, task, 0);
  }
  while (task < tasks) {
    unsigned long long claimed = 0;
    if (work && lane == 0) claimed = atomicAdd(work, 1ull);  // consumed after this task
    uint32_t c, i;
    if (tasks <= 0xFFFFFFFFull) {
      c = uint32_t(task) / m;
      i = uint32_t(task) - c * m;
    } else {
      c = uint32_t(task / m);
      i = uint32_t(task - uint64_t(c) * m);
    }
    const uint32_t col0 = c * 256 + lane * 4;
    const bool in0 = col0 < n, in1 = col0 + 128 < n;  // the last chunk may be ragged
    float acc[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[u][q] = Ops::zero();
    const uint32_t eb = rp[i], ee = rp[i + 1];
    // this lane's first piece of row 0 of the task's panel
    const float* const ybase = kSrcBlk ? y + size_t(c) * m * 256 + lane * 4 : y + col0;
    const size_t pitch = kSrcBlk ? 256 : n;
    // One group of <= 32 in-edges.  kFull: the chunk has all 256 columns (no
    // column predicates); a group of exactly 32 runs without per-edge bounds.
    auto group = [&](auto full_tag, uint32_t e0) {
      constexpr bool kFull = decltype(full_tag)::value;
      const uint32_t cnt = min(32u, ee - e0);
      uint32_t kk = 0;
      float aa = 0.0f;
      if (uint32_t(lane) < cnt) {
        kk = ci[e0 + lane];
        aa = wv[e0 + lane];
      }
      // in-edge t into stage j (a compile-time index: the loops are unrolled by kS)
      auto issue = [&](uint32_t t, int j) {
        const uint32_t k = __shfl_sync(0xffffffffu, kk, t & 31);
        const float* src = ybase + size_t(k) * pitch;
        const uint32_t dst = mine_s + j * 1024;
        if (kFull || in0) cp16(dst, src);
        if (kFull || in1) cp16(dst + 512, src + 128);
      };
      auto fold = [&](uint32_t t, int j) {
        wait_pending<kS - 1>();
        const float* const seg = mine + j * 256;
        float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
        if (kFull || in0) v0 = *reinterpret_cast<const float4*>(seg);
        if (kFull || in1) v1 = *reinterpret_cast<const float4*>(seg + 128);
        const float a = __shfl_sync(0xffffffffu, aa, t);
        acc[0][0] = Ops::add(acc[0][0], Ops::mul(a, v0.x, err), err);
        acc[0][1] = Ops::add(acc[0][1], Ops::mul(a, v0.y, err), err);
        acc[0][2] = Ops::add(acc[0][2], Ops::mul(a, v0.z, err), err);
        acc[0][3] = Ops::add(acc[0][3], Ops::mul(a, v0.w, err), err);
        acc[1][0] = Ops::add(acc[1][0], Ops::mul(a, v1.x, err), err);
        acc[1][1] = Ops::add(acc[1][1], Ops::mul(a, v1.y, err), err);
        acc[1][2] = Ops::add(acc[1][2], Ops::mul(a, v1.z, err), err);
        acc[1][3] = Ops::add(acc[1][3], Ops::mul(a, v1.w, err), err);
      };
      // one commit group per step, empty past the end: the wait count stays fixed
      if (cnt == 32) {
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          issue(j, j);
          commit();
        }
#pragma unroll 1
        for (uint32_t t0 = 0; t0 < 32 - kS; t0 += kS) {
#pragma unroll
          for (int j = 0; j < kS; ++j) {
            fold(t0 + j, j);
            issue(t0 + j + kS, j);  // refills the stage just read (its values are in registers)
            commit();
          }
        }
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          fold(32 - kS + j, j);
          commit();
        }
      } else {
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          if (uint32_t(j) < cnt) issue(j, j);
          commit();
        }
        for (uint32_t t0 = 0; t0 < cnt; t0 += kS) {
#pragma unroll
          for (int j = 0; j < kS; ++j) {
            const uint32_t t = t0 + j;
            if (t < cnt) {  // warp-uniform
              fold(t, j);
              if (t + kS < cnt) issue(t + kS, j);
              commit();
            }
          }
        }
      }
    };
    static_assert(32 % kS == 0, "the 32-edge path unrolls whole rings");
    const bool full = c + 1 < chunks || (n & 255u) == 0;
    for (uint32_t e0 = eb; e0 < ee; e0 += 32) {
      if (full) group(std::true_type{}, e0);
      else group(std::false_type{}, e0);
    }
    float b = 0.0f;
    if (kEpi == kEpiLayer) b = bias[i];
    float* const orow = dst_blk ? out + (size_t(c) * m + i) * 256 - size_t(c) * 256
                                : out + size_t(i) * n;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t cu = col0 + u * 128;
      if (kEpi == kEpiLayer)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[u][q] = layer_epilogue(acc[u][q], b, clip);
      if (nz_count)
#pragma unroll
        for (int q = 0; q < 4; ++q) nz += (cu + q < n && acc[u][q] != 0.0f) ? 1u : 0u;
      if (cu < n)
        *reinterpret_cast<float4*>(orow + cu) =
            make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
    }
    task = work ? __shfl_sync(0xffffffffu, claimed, 0) : task + stride;
  }
  if (nz_count) {
#pragma unroll
    for (int o = 16; o; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    if (lane == 0 && nz) atomicAdd(nz_count, (unsigned long long)nz);
  }
}

template <typename Ops, int kEpi>
__global__ void __launch_bounds__(256, SK_BULK_MINB)
    k_spmm_rows_bulk(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                     const float* __restrict__ wv, const float* __restrict__ bias,
                     const float* __restrict__ y, uint32_t m, uint32_t n, float clip,
                     float* __restrict__ out, int* err, unsigned long long* work) {
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  spmm_tasks_bulk<Ops, kEpi>(rp, ci, wv, bias, y, m, n, clip, out, err, nullptr, bulk_smem, false,
                             work);
}

template <typename Ops, int kEpi, bool kVec4, int kU = 1>
__global__ void __launch_bounds__(256, SK_SPMM_MINB)
    k_spmm_rows(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                const float* __restrict__ wv, const float* __restrict__ bias,
                const float* __restrict__ y, uint32_t m, uint32_t n, float clip,
                float* __restrict__ out, int* err) {
  spmm_tasks<Ops, kEpi, kVec4, kU>(rp, ci, wv, bias, y, m, n, clip, out, err);
}

// Wide batches, rows of more than 16 entries: the engine's wide task (a row x
// 256 columns, 4 in-edges x 2 loads in flight per lane, 3 blocks per SM).
template <typename Ops, int kEpi>
__global__ void __launch_bounds__(256, 3)
    k_spmm_rows_wide(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                     const float* __restrict__ wv, const float* __restrict__ bias,
                     const float* __restrict__ y, uint32_t m, uint32_t n, float clip,
                     float* __restrict__ out, int* err) {
  spmm_tasks<Ops, kEpi, true, 2, 4>(rp, ci, wv, bias, y, m, n, clip, out, err);
}

// Narrow activations (n <= 64, n % 4 == 0): a group of G = n/4 lanes (rounded
// up to a power of two) owns one row and a lane owns 4 columns, so a warp
// folds 32/G rows at once instead of leaving 32 - n/4 lanes idle; every lane
// keeps kNB float4 Y loads in flight.  Rows of one warp may differ in length:
// the loop runs to the warp's longest row with the shorter ones predicated
// off, and each output still folds its row's entries strictly in ascending k.
// (A one-column-per-lane variant for long rows, kC = 1, measured 3-4x slower
// on the paper sweep's batch-64 shapes and is not dispatched.)
template <typename Ops, int kEpi, int G, int kC, int kNB>
__global__ void __launch_bounds__(256, kC == 1 ? 2 : 3)
    k_spmm_narrow(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                  const float* __restrict__ wv, const float* __restrict__ bias,
                  const float* __restrict__ y, uint32_t m, uint32_t n, float clip,
                  float* __restrict__ out, int* err) {
  static_assert(kC == 1 || kC == 4, "lane column width");
  constexpr int R = 32 / G;  // rows per warp
  const int lane = threadIdx.x & 31, sub = lane % G;
  const uint32_t chunks = (n + G * kC - 1) / (G * kC);
  const uint64_t row_groups = (uint64_t(m) + R - 1) / R;
  for (uint64_t task = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       task < row_groups * chunks; task += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t c = uint32_t(task / row_groups);
    const uint32_t i = uint32_t(task - uint64_t(c) * row_groups) * R + uint32_t(lane / G);
    const uint32_t col0 = (c * G + uint32_t(sub)) * kC;
    const bool live_row = i < m, live_col = col0 < n;
    const uint32_t eb = live_row ? rp[i] : 0u, ee = live_row ? rp[i + 1] : 0u;
    const uint32_t len = ee - eb;
    uint32_t wlen = len;
#pragma unroll
    for (int o = 16; o; o >>= 1) wlen = max(wlen, __shfl_xor_sync(0xffffffffu, wlen, o));
    float acc[kC];
#pragma unroll
    for (int q = 0; q < kC; ++q) acc[q] = Ops::zero();
    for (uint32_t e0 = 0; e0 < wlen; e0 += G) {
      uint32_t kk = 0;
      float aa = 0.0f;
      if (e0 + sub < len) {
        kk = ci[eb + e0 + sub];
        aa = wv[eb + e0 + sub];
      }
      for (uint32_t t0 = 0; t0 < uint32_t(G) && e0 + t0 < wlen; t0 += kNB) {
        float v[kNB][kC];
        float a[kNB];
#pragma unroll
        for (int q = 0; q < kNB; ++q) {
          const uint32_t t = t0 + q;
          const uint32_t k = __shfl_sync(0xffffffffu, kk, int(t % G), G);
          a[q] = __shfl_sync(0xffffffffu, aa, int(t % G), G);
#pragma unroll
          for (int u = 0; u < kC; ++u) v[q][u] = 0.0f;
          if (t < uint32_t(G) && e0 + t < len && live_col) {
            const float* yr = y + size_t(k) * n + col0;
            if (kC == 4) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(yr));
              v[q][0] = f.x;
              v[q][kC > 1 ? 1 : 0] = f.y;
              v[q][kC > 2 ? 2 : 0] = f.z;
              v[q][kC > 3 ? 3 : 0] = f.w;
            } else {
              v[q][0] = __ldg(yr);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kNB; ++q)
          if (t0 + q < uint32_t(G) && e0 + t0 + q < len)
#pragma unroll
            for (int u = 0; u < kC; ++u) acc[u] = Ops::add(acc[u], Ops::mul(a[q], v[q][u], err), err);
      }
    }
    if (live_row && live_col) {
      if (kEpi == kEpiLayer) {
        const float b = bias[i];
#pragma unroll
        for (int u = 0; u < kC; ++u) acc[u] = layer_epilogue(acc[u], b, clip);
      }
      float* o = out + size_t(i) * n + col0;
      if (kC == 4)
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[kC > 1 ? 1 : 0],
                                                    acc[kC > 2 ? 2 : 0], acc[kC > 3 ? 3 : 0]);
      else
        o[0] = acc[0];
    }
  }
}

template <typename Ops, int kEpi>
bool launch_narrow(sk_ctx* ctx, const sk_csr* w, const float* bias, const float* y, uint32_t n,
                   float clip, float* out) {
  if (n > 64 || n % 4 != 0 || w->rows == 0) return false;
  const uint32_t need = n / 4;  // lanes per row
  auto go = [&](auto g, auto c) {
    constexpr int G = decltype(g)::value, kC = decltype(c)::value;
    constexpr int kNB = kC == 1 ? 16 : 8;
    const uint64_t warps = (uint64_t(w->rows) + 32 / G - 1) / (32 / G) *
                           ((n + G * kC - 1) / (G * kC));
    const unsigned grid = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>((warps + 7) / 8, uint64_t(ctx->num_sms) * 16)));
    SK_LAUNCH((k_spmm_narrow<Ops, kEpi, G, kC, kNB>), grid, 256, 0, ctx->stream, w->rp, w->ci,
              w->v, bias, y, w->rows, n, clip, out, ctx->d_err);
  };
  using I1 = std::integral_constant<int, 1>;
  using I4 = std::integral_constant<int, 4>;
  if (need <= 1) go(I1{}, I4{});
  else if (need <= 2) go(std::integral_constant<int, 2>{}, I4{});
  else if (need <= 4) go(I4{}, I4{});
  else if (need <= 8) go(std::integral_constant<int, 8>{}, I4{});
  else go(std::integral_constant<int, 16>{}, I4{});
  return true;
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
  float* blk[2];                   // K1b: panel-major scratch of the intermediate layers (or null)
  unsigned long long* work;        // K1b: L zeroed task counters (or null: static striding)
};

// kU = 2 (wide batches, n >= 1024): a task is a row x 256 columns, so the (k, w)
// broadcasts, the row address and the loop overhead of an in-edge are paid once
// per two 16-byte loads (the saturated cfg3 layer ran ~36 instructions per
// in-edge and 128 columns, 8 of them the multiply-adds), and 4 in-edges x 2
// loads are in flight per lane at 3 blocks per SM.  Measured per saturated
// 16384 x 60000 layer (tools/prof_dense.py): 17.5 -> 15.0 ms; kU = 4 x batch 2
// 15.2, kU = 2 x batch 8 at 2 blocks 14.7 (15000 samples: 3.4 against 3.3),
// batch 2 at 4 blocks 16.2; L1::no_allocate loads 20.0 and an L2 bulk prefetch
// of the next column panel 16.7 -- both slower, removed.
#ifndef SK_ENG_KU
#define SK_ENG_KU 2
#endif
#ifndef SK_ENG_BATCH
#define SK_ENG_BATCH 4
#endif
#ifndef SK_ENG_MINB
#define SK_ENG_MINB 3
#endif
#ifndef SK_ENG_BULK
#define SK_ENG_BULK 1
#endif
#ifndef SK_ENG_BLOCKED
#define SK_ENG_BLOCKED 1
#endif
#ifndef SK_ENG_CLAIM
#define SK_ENG_CLAIM 1
#endif
#ifndef SK_ENG_CLAIM_REG
#define SK_ENG_CLAIM_REG 1
#endif
template <bool kVec4, int kU = 1>
__global__ void __launch_bounds__(256, kU == 1 ? SK_SPMM_MINB : SK_ENG_MINB)
    k_dense_engine(DenseEngineArgs p) {
  cg::grid_group grid = cg::this_grid();
  for (uint32_t k = 0; k < p.L; ++k) {
    const float* src = k == 0 ? p.y0 : (((k - 1) & 1) ? p.buf[1] : p.buf[0]);
    float* dst = (k & 1) ? p.buf[1] : p.buf[0];
    spmm_tasks<OpArith, kEpiLayer, kVec4, kU, (kU == 1 ? SK_SPMM_BATCH : SK_ENG_BATCH)>(
        p.w_rp[k], p.w_ci[k], p.w_v[k], p.bias + size_t(k) * p.m, src, p.m, p.n, p.clip, dst,
        p.err, p.nnz ? p.nnz + k : nullptr, p.work ? p.work + k : nullptr);
    if (k + 1 < p.L) {
      grid.sync();
      if (p.stop_below && *(volatile unsigned long long*)(p.nnz + k) < p.stop_below) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *p.layers_done = int(k + 1);
        return;
      }
    }
  }
}

// The engine over the shared-memory-staged wide task (K1b).  With p.blk the
// intermediate activations live in panel-major scratch: layer 0 reads the
// caller's row-major Y_0, the last layer writes the caller's row-major buffer;
// a density stop after layer k copies that layer's panels back into the
// row-major buffer the caller expects before the engine returns.
__global__ void __launch_bounds__(256, SK_BULK_MINB) k_dense_engine_bulk(DenseEngineArgs p) {
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  cg::grid_group grid = cg::this_grid();
  const bool blk = p.blk[0] != nullptr;
  for (uint32_t k = 0; k < p.L; ++k) {
    const bool last = k + 1 == p.L;
    const bool sb = blk && k > 0, db = blk && !last;
    const float* src = k == 0 ? p.y0 : sb ? p.blk[(k - 1) & 1] : p.buf[(k - 1) & 1];
    float* dst = db ? p.blk[k & 1] : p.buf[k & 1];
    if (sb)
      spmm_tasks_bulk<OpArith, kEpiLayer, true>(
          p.w_rp[k], p.w_ci[k], p.w_v[k], p.bias + size_t(k) * p.m, src, p.m, p.n, p.clip, dst,
          p.err, p.nnz ? p.nnz + k : nullptr, bulk_smem, db, p.work ? p.work + k : nullptr);
    else
      spmm_tasks_bulk<OpArith, kEpiLayer, false>(
          p.w_rp[k], p.w_ci[k], p.w_v[k], p.bias + size_t(k) * p.m, src, p.m, p.n, p.clip, dst,
          p.err, p.nnz ? p.nnz + k : nullptr, bulk_smem, db, p.work ? p.work + k : nullptr);
    if (!last) {
      grid.sync();
      if (p.stop_below && *(volatile unsigned long long*)(p.nnz + k) < p.stop_below) {
        if (db) {  // 16-byte units of the panels back to rows
          const uint32_t chunks = (p.n + 255) / 256;
          const uint64_t units = uint64_t(chunks) * p.m * 64;
          for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < units;
               t += uint64_t(gridDim.x) * blockDim.x) {
            const uint32_t q = uint32_t(t & 63);
            const uint64_t cr = t >> 6;  // c * m + row
            const uint32_t c = uint32_t(cr / p.m), r = uint32_t(cr - uint64_t(c) * p.m);
            const uint32_t col = c * 256 + q * 4;
            if (col < p.n)
              *reinterpret_cast<float4*>(p.buf[k & 1] + size_t(r) * p.n + col) =
                  *reinterpret_cast<const float4*>(dst + t * 4);
          }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) *p.layers_done = int(k + 1);
        return;
      }
    }
  }
}

// ---- K1t: register-tiled SpMM for weight rows with many entries ----------------------
//
// At high density (BASELINE cfg2, d >= 1/8) the row-per-warp K1 re-reads a
// 512-byte Y segment from L2 for every stored weight; here a CTA owns a
// (kWarps * kRW)-row x 256-column output tile and streams Y through shared memory
// in 32-row k-chunks (cp.async.bulk, one 1 KB row segment per copy,
// double-buffered on mbarriers).  A warp owns kRW rows x 256 columns (a lane:
// 8 columns of each row, fp32 accumulators in registers): each Y chunk row is
// read from shared memory once per warp and applied to every one of the warp's
// rows that stores a weight at that k.  Presence comes from a 32-bit mask per
// (row, chunk), so the fold is exactly the stored entries in ascending k (absent
// weights are skipped, never multiplied as zeros): bit-identical to K1 and to
// the reference's mxm_csr_dense (proj/src/matrix.cpp:403-424).
//
// The weights are repacked once per matrix (cached on the immutable handle)
// into the tile order: for every (64-row tile, 32-k chunk) a 64 x 32 value
// block (only present slots are written) and 64 masks, so each chunk's
// weights arrive with one more bulk copy.
#ifndef SK_TILE_PRED
#define SK_TILE_PRED 0
#endif
#ifndef SK_TILE_CB
#define SK_TILE_CB 2
#endif
#ifndef SK_TILE_PR
#define SK_TILE_PR 64
#endif
#ifndef SK_TILE_KC
#define SK_TILE_KC 32
#endif
namespace tile {
constexpr int kPR = SK_TILE_PR;        // rows per packed tile
constexpr int kCB = SK_TILE_CB;        // 256-column blocks per CTA (one 2-D TMA box each)
constexpr int kTC = 256 * kCB;         // columns per CTA (lane: 2 kCB x float4)
constexpr int kKC = SK_TILE_KC;        // k per chunk
constexpr int kStages = 2;
constexpr uint32_t kYBytes = uint32_t(kKC) * kTC * 4;      // 32 KB per column block
constexpr uint32_t kWBytes = uint32_t(kPR) * kKC * 4;      // 8 KB
constexpr uint32_t kMBytes = uint32_t(kPR) * 4;            // 256 B
constexpr uint32_t kStageBytes = kYBytes + kWBytes + kMBytes;
constexpr size_t kSmem = size_t(kStages) * kStageBytes + 64;
}  // namespace tile

// Pack (once per weight matrix): masks zeroed by the caller, then a thread per
// stored entry writes its value into its (tile, chunk) block and ORs its bit.
__global__ void k_tile_pack(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                            const float* __restrict__ v, uint32_t m, uint32_t nK,
                            float* __restrict__ vals, uint32_t* __restrict__ mask) {
  const int lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t rt = i / tile::kPR, r = i % tile::kPR;
    for (uint32_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
      const uint32_t k = ci[e], kc = k / tile::kKC, kk = k % tile::kKC;
      const size_t blk = size_t(rt) * nK + kc;
      vals[blk * (tile::kPR * tile::kKC) + r * tile::kKC + kk] = v[e];
      atomicOr(&mask[blk * tile::kPR + r], 1u << kk);
    }
  }
}

// kRW rows per warp, 64 / kRW warps per CTA (one packed tile per CTA)
template <int kEpi, int kRW>
__global__ void __launch_bounds__(tile::kPR / kRW * 32,
                                  tile::kCB * tile::kKC * tile::kStages <= 64 ? 2 : 1)
    k_spmm_tile(const __grid_constant__ CUtensorMap ymap, const float* __restrict__ wvals,
                const uint32_t* __restrict__ wmask, const float* __restrict__ bias, uint32_t m,
                uint32_t K, uint32_t n, float clip, float* __restrict__ out) {
  using namespace tile;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rt = blockIdx.y, c0 = blockIdx.x * kTC;
  const uint32_t nK = (K + kKC - 1) / kKC;
  const uint32_t ncols = min(uint32_t(kTC), n - c0);  // a multiple of 4 (n % 4 == 0)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  auto stage = [&](uint32_t s) { return smem + size_t(s) * kStageBytes; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) async::mbar_init(async::smem_u32(mbar + s), 1);
    async::fence_mbar_init();
  }
  __syncthreads();
  // producer (thread 0): chunk j's 32 x 256 Y box (one 2-D tensor copy; rows
  // past K and columns past n arrive as zeros and are never used) and its weight
  // block + masks into stage j % kStages
  auto issue = [&](uint32_t j) {
    const uint32_t s = j % kStages;
    const uint32_t mb = async::smem_u32(mbar + s);
    uint8_t* st = stage(s);
    async::mbar_expect_tx(mb, kYBytes + kWBytes + kMBytes);
    const size_t blk = size_t(rt) * nK + j;
#pragma unroll
    for (int h = 0; h < kCB; ++h)  // [kCB][kKC][256] in shared memory
      async::tma_2d_g2s(async::smem_u32(st + h * (kYBytes / kCB)), &ymap, int(c0 + 256 * h),
                        int(j * kKC), mb);
    async::bulk_g2s(async::smem_u32(st + kYBytes), wvals + blk * (kPR * kKC), kWBytes, mb);
    async::bulk_g2s(async::smem_u32(st + kYBytes + kWBytes), wmask + blk * kPR, kMBytes, mb);
  };
  if (threadIdx.x == 0)
    for (uint32_t j = 0; j < min(uint32_t(kStages), nK); ++j) issue(j);

  constexpr int kQ = 8 * kCB;  // columns per lane
  float acc[kRW][kQ];
#pragma unroll
  for (int r = 0; r < kRW; ++r)
#pragma unroll
    for (int q = 0; q < kQ; ++q) acc[r][q] = 0.0f;
  for (uint32_t j = 0; j < nK; ++j) {
    const uint32_t s = j % kStages;
    async::mbar_wait(async::smem_u32(mbar + s), (j / kStages) & 1u);
    const float* Yc = reinterpret_cast<const float*>(stage(s));
    const float* Wc = reinterpret_cast<const float*>(stage(s) + kYBytes) + warp * kRW * kKC;
    const uint32_t* Mc =
        reinterpret_cast<const uint32_t*>(stage(s) + kYBytes + kWBytes) + warp * kRW;
    uint32_t mask[kRW];
#pragma unroll
    for (int r = 0; r < kRW; ++r) mask[r] = Mc[r];  // warp-uniform (broadcast)
#pragma unroll 4
    for (int kk = 0; kk < kKC; ++kk) {
      float yv[kQ];
#pragma unroll
      for (int h = 0; h < kCB; ++h) {
        const float* yr = Yc + h * (kKC * 256) + kk * 256;
        const float4 a = *reinterpret_cast<const float4*>(yr + lane * 4);
        const float4 b4 = *reinterpret_cast<const float4*>(yr + 128 + lane * 4);
        yv[8 * h + 0] = a.x, yv[8 * h + 1] = a.y, yv[8 * h + 2] = a.z, yv[8 * h + 3] = a.w;
        yv[8 * h + 4] = b4.x, yv[8 * h + 5] = b4.y, yv[8 * h + 6] = b4.z, yv[8 * h + 7] = b4.w;
      }
#pragma unroll
      for (int r = 0; r < kRW; ++r) {
        if (mask[r] & (1u << kk)) {  // warp-uniform: the warp's lanes share the rows
          const float w = Wc[r * kKC + kk];
#pragma unroll
          for (int q = 0; q < kQ; ++q) acc[r][q] = __fadd_rn(acc[r][q], __fmul_rn(w, yv[q]));
        }
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && j + kStages < nK) issue(j + kStages);
  }
  // epilogue: bias + ReLU select (+ clip), 2 kCB float4 stores per row
#pragma unroll
  for (int r = 0; r < kRW; ++r) {
    const uint32_t i = rt * kPR + warp * kRW + r;
    if (i >= m) continue;
    const float b = kEpi == kEpiLayer ? bias[i] : 0.0f;
    float z[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) z[q] = kEpi == kEpiLayer ? layer_epilogue(acc[r][q], b, clip) : acc[r][q];
    float* orow = out + size_t(i) * n + c0;
#pragma unroll
    for (int h = 0; h < kCB; ++h) {
      const uint32_t ca = 256 * h + uint32_t(lane) * 4, cb = ca + 128;
      if (ca < ncols)
        *reinterpret_cast<float4*>(orow + ca) =
            make_float4(z[8 * h + 0], z[8 * h + 1], z[8 * h + 2], z[8 * h + 3]);
      if (cb < ncols)
        *reinterpret_cast<float4*>(orow + cb) =
            make_float4(z[8 * h + 4], z[8 * h + 5], z[8 * h + 6], z[8 * h + 7]);
    }
  }
}

// The tile-packed copy of W (built on first use, cached on the handle).
static void ensure_tile_pack(sk_ctx* ctx, const sk_csr* w) {
  auto* ww = const_cast<sk_csr*>(w);
  if (ww->tile_vals) return;
  const uint32_t nrt = (w->rows + tile::kPR - 1) / tile::kPR;
  const uint32_t nK = (w->cols + tile::kKC - 1) / tile::kKC;
  const size_t blocks = size_t(nrt) * nK;
  ww->tile_vals = dalloc<float>(ctx, blocks * tile::kPR * tile::kKC);
  ww->tile_mask = dalloc<uint32_t>(ctx, blocks * tile::kPR);
  SK_CUDA(cudaMemsetAsync(ww->tile_mask, 0, blocks * tile::kPR * 4, ctx->stream));
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t(w->rows) + 7) / 8, uint64_t(ctx->num_sms) * 16)));
  SK_LAUNCH(k_tile_pack, grid, 256, 0, ctx->stream, w->rp, w->ci, w->v, w->rows, nK,
            ww->tile_vals, ww->tile_mask);
}

#ifndef SK_TILE_RW
#define SK_TILE_RW 4
#endif
#ifndef SK_TILE_PRED
#define SK_TILE_PRED 0
#endif

// K1t applies when rows are heavy enough that a warp's rows share most k
// (mean stored entries per row >= cols / 8), the activations are 16-byte
// aligned rows (n % 4 == 0) and wide enough for the 256-column tiles, and the
// packed copy (dense-tile sized) stays small against the device.
static bool tile_applies(sk_ctx* ctx, const sk_csr* w, uint32_t n) {
  if (n % 4 != 0 || n < 128 || w->rows == 0 || w->cols == 0) return false;
  if (double(w->nnz) * 8.0 < double(w->rows) * double(w->cols)) return false;
  const double packed = double((w->rows + 63) / 64) * 64.0 * double((w->cols + 31) / 32) * 32.0 * 4.0;
  return packed < 0.05 * double(ctx->total_mem);
}

static void launch_tile(sk_ctx* ctx, const sk_csr* w, const float* d_bias, const float* y,
                        uint32_t n, float clip, float* out, bool layer) {
  constexpr int kRW = SK_TILE_RW;
  ensure_tile_pack(ctx, w);
  CUtensorMap ymap;
  if (!async::make_tmap_2d_f32(&ymap, y, w->cols, n, n, tile::kKC, 256))
    fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed for the activation tile map");
  dim3 grid(ceil_div(n, tile::kTC), ceil_div(w->rows, tile::kPR));
  const int threads = tile::kPR / kRW * 32;
  if (layer) {
    smem_attr(ctx, k_spmm_tile<kEpiLayer, kRW>, int(tile::kSmem));
    SK_LAUNCH((k_spmm_tile<kEpiLayer, kRW>), grid, threads, tile::kSmem, ctx->stream,
              ymap, w->tile_vals, w->tile_mask, d_bias, w->rows, w->cols, n, clip, out);
  } else {
    smem_attr(ctx, k_spmm_tile<kEpiNone, kRW>, int(tile::kSmem));
    SK_LAUNCH((k_spmm_tile<kEpiNone, kRW>), grid, threads, tile::kSmem, ctx->stream,
              ymap, w->tile_vals, w->tile_mask, nullptr, w->rows, w->cols, n, 0.0f, out);
  }
}

// ---- K1c: the whole forward of a small model, one thread-block cluster per ----------
//      32-sample column block, layers separated by cluster barriers
//
// Output column j of layer k+1 depends only on column j of layer k, so sample
// column blocks never need each other: a cluster of kCS CTAs owns 32 columns
// and runs EVERY layer on them, its CTAs splitting the output rows; no
// grid-wide barrier and no per-layer launch.  Per CTA:
//  * at start, every layer's weight rows of the CTA (row pointers, columns,
//    values) are copied into shared memory once;
//  * per layer, Y_k's 32-column panel (all m rows, 128 B per row) arrives in
//    shared memory by 2-D tensor copies (TMA), a warp folds one output row at a
//    time with lane = column (conflict-free shared loads, the row's (k, w)
//    broadcast), strictly in ascending k -- the reference's fold
//    (proj/src/matrix.cpp:403-424) -- and writes Y_{k+1} to global memory;
//  * a proxy fence + hardware cluster barrier (release / acquire) orders every
//    CTA's writes before the next layer's tensor copies read them.
// BASELINE cfg1 (m = 1024, 4 layers, 256 samples): 8 clusters x 8 CTAs.  (The
// clusters of one launch are placed on one die -- measured: 16 clusters of 8
// ran as two waves -- so the launch is kept to <= 9 clusters of 8.)
namespace clu {
constexpr int kCS = 8;        // CTAs per cluster
constexpr int kWarps = 32;    // warps per CTA
constexpr int kCols = 32;     // columns per cluster (kCols lanes fold one row)
constexpr int kBoxRows = 256; // tensor-copy box: 256 rows x kCols columns
}  // namespace clu

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

struct ClusterMaps {
  CUtensorMap y0, b0, b1;  // Y_0 and the two ping-pong buffers, box 256 x kCols
};

#ifdef SK_CLU_DEBUG
__device__ long long g_clu_ts[64];
#define CLU_TS(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_clu_ts[i] = t_; } } while (0)
__device__ unsigned long long g_clu_start[2];  // min / max CTA start
__device__ unsigned long long g_clu_end[2];
#else
#define CLU_TS(i) do {} while (0)
#endif
__global__ void __launch_bounds__(clu::kWarps * 32, 1)
    k_dense_cluster(const __grid_constant__ ClusterMaps maps, DenseEngineArgs p,
                    float* __restrict__ last, uint32_t wslice_entries) {
  using namespace clu;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank();
  constexpr int kGroups = 32 / kCols;  // row groups per warp
  const int h = lane / kCols, cl = lane % kCols;  // lane group, column within the block
  const uint32_t c0 = (blockIdx.x / kCS) * kCols, col = c0 + cl;
  const bool live = col < p.n;
  const uint32_t r0 = uint32_t(uint64_t(p.m) * crank / kCS);
  const uint32_t r1 = uint32_t(uint64_t(p.m) * (crank + 1) / kCS);
  const uint32_t nr = r1 - r0;
  // shared layout: Y panel (m x kCols floats, box-padded) | per layer: row
  // offsets (nr + 1) | (k, w) pairs (wslice_entries)
  const uint32_t mpad = (p.m + kBoxRows - 1) / kBoxRows * kBoxRows;
  float* Ys = reinterpret_cast<float*>(smem);
  uint32_t* roff = reinterpret_cast<uint32_t*>(Ys + size_t(mpad) * kCols);
  uint2* kw = reinterpret_cast<uint2*>(roff + ((size_t(p.L) * (nr + 1) + 1) & ~size_t(1)));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(kw + size_t(wslice_entries));
  CLU_TS(0);
#ifdef SK_CLU_DEBUG
  if (threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    atomicMin(&g_clu_start[0], t_);
    atomicMax(&g_clu_start[1], t_);
  }
#endif
  if (threadIdx.x == 0) {
    async::mbar_init(async::smem_u32(mbar), 1);
    async::fence_mbar_init();
  }
  // the CTA's weight rows of every layer in shared memory: slice bounds of all
  // layers first (one load each, in parallel); layer 0's entries before the
  // first fold, layer k+1's while the cluster waits at layer k's barrier
  uint32_t* bnd = reinterpret_cast<uint32_t*>(mbar + 1);  // 2 L + 1 words
  for (uint32_t q = threadIdx.x; q < 2 * p.L; q += blockDim.x)
    bnd[q] = p.w_rp[q >> 1][(q & 1) ? r1 : r0];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t base = 0;
    for (uint32_t k = 0; k < p.L; ++k) {
      const uint32_t eb = bnd[2 * k], ee = bnd[2 * k + 1];
      bnd[2 * k] = base;       // slice start in kw
      bnd[2 * k + 1] = eb;     // the layer's first entry in global memory
      base += ee - eb;
    }
    bnd[2 * p.L] = base;
  }
  __syncthreads();
  for (uint32_t k = 0; k < p.L; ++k) {
    const uint32_t* rp = p.w_rp[k];
    for (uint32_t q = threadIdx.x; q <= nr; q += blockDim.x)
      roff[k * (nr + 1) + q] = bnd[2 * k] + rp[r0 + q] - bnd[2 * k + 1];
  }
  float* bsh = reinterpret_cast<float*>(bnd + ((2 * p.L + 2) & ~1u));  // L x nr biases
  auto load_slice = [&](uint32_t k) {
    for (uint32_t q = threadIdx.x; q < nr; q += blockDim.x)
      bsh[k * nr + q] = p.bias[size_t(k) * p.m + r0 + q];
    const uint32_t* ci = p.w_ci[k];
    const float* wv = p.w_v[k];
    const uint32_t s0 = bnd[2 * k], cnt = bnd[2 * k + 2] - s0, g0 = bnd[2 * k + 1];
    constexpr int kU = 4;  // loads in flight per thread
    for (uint32_t t0 = threadIdx.x; t0 < cnt; t0 += blockDim.x * kU) {
      uint32_t cc[kU];
      float vv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t t = t0 + u * blockDim.x;
        if (t < cnt) {
          cc[u] = ci[g0 + t];
          vv[u] = wv[g0 + t];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t t = t0 + u * blockDim.x;
        if (t < cnt) kw[s0 + t] = make_uint2(cc[u], __float_as_uint(vv[u]));
      }
    }
  };
  load_slice(0);
  __syncthreads();
  const uint32_t nbox = mpad / kBoxRows;
  CLU_TS(1);
  for (uint32_t k = 0; k < p.L; ++k) {
    const CUtensorMap* src = k == 0 ? &maps.y0 : (((k - 1) & 1) ? &maps.b1 : &maps.b0);
    float* dst = k + 1 == p.L ? last : ((k & 1) ? p.buf[1] : p.buf[0]);
    if (threadIdx.x == 0) {
      const uint32_t mb = async::smem_u32(mbar);
      async::mbar_expect_tx(mb, nbox * kBoxRows * kCols * 4);
      for (uint32_t b = 0; b < nbox; ++b)
        async::tma_2d_g2s(async::smem_u32(Ys + size_t(b) * kBoxRows * kCols), src, int(c0),
                          int(b * kBoxRows), mb);
    }
    async::mbar_wait(async::smem_u32(mbar), k & 1u);
    CLU_TS(2 + 3 * k);
    const uint32_t* ro = roff + k * (nr + 1);
    const float* bias = bsh + size_t(k) * nr - r0;  // indexed by the global row
    // a lane group folds one row at a time: the row's entries in steps of 4
    // with every (k, w) and Y load of a step issued first, then the fold in
    // order; rows differ in length (W_ref's rows are W's columns), so there is
    // no guard inside a step -- the 0..3 leftover entries fold one by one
    const uint32_t vw = uint32_t(warp) * kGroups + h, nvw = kGroups * kWarps;
    for (uint32_t r = vw; r < nr; r += nvw) {
      float acc = 0.0f;
      const uint32_t e0 = ro[r], e1 = ro[r + 1];
      uint32_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        float yv[4], wv4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint2 kv = kw[e + u];  // broadcast within the lane group
          wv4[u] = __uint_as_float(kv.y);
          yv[u] = Ys[kv.x * kCols + cl];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = __fadd_rn(acc, __fmul_rn(wv4[u], yv[u]));
      }
      for (; e < e1; ++e) {
        const uint2 kv = kw[e];
        acc = __fadd_rn(acc, __fmul_rn(__uint_as_float(kv.y), Ys[kv.x * kCols + cl]));
      }
      if (live) {
        const uint32_t i = r0 + r;
        dst[size_t(i) * p.n + col] = layer_epilogue(acc, bias[i], p.clip);
      }
    }
    CLU_TS(3 + 3 * k);
    if (k + 1 < p.L) {
      // the generic-proxy stores above are read by the next layer's tensor copies
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      load_slice(k + 1);  // overlaps the wait for the slowest CTA of the cluster
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    CLU_TS(4 + 3 * k);
  }
#ifdef SK_CLU_DEBUG
  if (threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    atomicMin(&g_clu_end[0], t_);
    atomicMax(&g_clu_end[1], t_);
  }
#endif
}

// Shared memory K1c needs for a model and batch (0 = does not apply).
static size_t cluster_smem(sk_ctx* ctx, const sk_model* md, uint32_t n, uint32_t* wslice) {
  const uint32_t m = md->neurons;
  if (md->layers < 1 || m < clu::kCS || n % 4 != 0 ||
      size_t(m) * clu::kCols * 4 > 160 * 1024)
    return 0;
  auto* mm = const_cast<sk_model*>(md);
  if (mm->clu_worst == SIZE_MAX) {
    // the largest per-CTA weight slice over the cluster's row blocks (row
    // pointers at the block bounds; once per model)
    std::vector<uint32_t> bnd(size_t(md->layers) * (clu::kCS + 1));
    for (uint32_t k = 0; k < md->layers; ++k)
      for (uint32_t c = 0; c <= uint32_t(clu::kCS); ++c)
        SK_CUDA(cudaMemcpyAsync(&bnd[size_t(k) * (clu::kCS + 1) + c],
                                md->w[k]->rp + uint64_t(m) * c / clu::kCS, 4,
                                cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    size_t worst = 0;
    for (uint32_t c = 0; c < uint32_t(clu::kCS); ++c) {
      size_t tot = 0;
      for (uint32_t k = 0; k < md->layers; ++k)
        tot += bnd[size_t(k) * (clu::kCS + 1) + c + 1] - bnd[size_t(k) * (clu::kCS + 1) + c];
      worst = std::max(worst, tot);
    }
    mm->clu_worst = worst;
  }
  const size_t worst = mm->clu_worst;
  const size_t mpad = (m + clu::kBoxRows - 1) / clu::kBoxRows * clu::kBoxRows;
  const size_t nr = (m + clu::kCS - 1) / clu::kCS + 1;
  const size_t bytes = mpad * clu::kCols * 4 + ((size_t(md->layers) * (nr + 1) + 1) & ~size_t(1)) * 4 +
                       worst * 8 + 16 + (2 * size_t(md->layers) + 2) * 4 +
                       size_t(md->layers) * nr * 4;
  *wslice = uint32_t(worst);
  return bytes <= 200 * 1024 ? bytes : 0;
}

static void launch_cluster_forward(sk_ctx* ctx, const DenseEngineArgs& p, float* last,
                                   size_t smem, uint32_t wslice) {
  ClusterMaps maps;
  const uint64_t m = p.m, n = p.n;
  if (!async::make_tmap_2d_f32(&maps.y0, p.y0, m, n, n, clu::kBoxRows, clu::kCols) ||
      !async::make_tmap_2d_f32(&maps.b0, p.buf[0] ? p.buf[0] : last, m, n, n, clu::kBoxRows,
                               clu::kCols) ||
      !async::make_tmap_2d_f32(&maps.b1, p.buf[1] ? p.buf[1] : last, m, n, n, clu::kBoxRows,
                               clu::kCols))
    fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed for the dense forward");
  smem_attr(ctx, k_dense_cluster, int(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(((p.n + clu::kCols - 1) / clu::kCols) * clu::kCS));
  cfg.blockDim = dim3(clu::kWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = clu::kCS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  timing_mark(ctx, SK_KT_DENSE_ENGINE);  // (after the host-side map encoding)
  SK_CUDA(cudaLaunchKernelEx(&cfg, k_dense_cluster, maps, p, last, wslice));
  timing_mark(ctx);
  g_launches.fetch_add(1);
#ifdef SK_CLU_DEBUG
  {
    unsigned long long init[2] = {~0ull, 0ull};
    // (for the next call)
    unsigned long long st[2], en[2];
    SK_CUDA(cudaMemcpyFromSymbolAsync(st, g_clu_start, 16, 0, cudaMemcpyDeviceToHost, ctx->stream));
    SK_CUDA(cudaMemcpyFromSymbolAsync(en, g_clu_end, 16, 0, cudaMemcpyDeviceToHost, ctx->stream));
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
    fprintf(stderr, "[clu] CTA starts spread %.2f us, ends spread %.2f us, first start -> last end %.2f us\n",
            (st[1] - st[0]) / 1e3, (en[1] - en[0]) / 1e3, (en[1] - st[0]) / 1e3);
    SK_CUDA(cudaMemcpyToSymbolAsync(g_clu_start, init, 16, 0, cudaMemcpyHostToDevice, ctx->stream));
    SK_CUDA(cudaMemcpyToSymbolAsync(g_clu_end, init, 16, 0, cudaMemcpyHostToDevice, ctx->stream));
  }
  long long ts[64];
  SK_CUDA(cudaMemcpyFromSymbolAsync(ts, g_clu_ts, sizeof(ts), 0, cudaMemcpyDeviceToHost, ctx->stream));
  SK_CUDA(cudaStreamSynchronize(ctx->stream));
  fprintf(stderr, "[clu] prologue %.2f us |", (ts[1] - ts[0]) / 1e3);
  for (uint32_t k = 0; k < p.L; ++k)
    fprintf(stderr, " L%u tma %.2f fold %.2f bar %.2f |", k, (ts[2 + 3 * k] - (k ? ts[1 + 3 * k] : ts[1])) / 1e3,
            (ts[3 + 3 * k] - ts[2 + 3 * k]) / 1e3, (ts[4 + 3 * k] - ts[3 + 3 * k]) / 1e3);
  fprintf(stderr, "\n");
#endif
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
  p.blk[0] = p.blk[1] = nullptr;
  p.work = nullptr;
  uint32_t wslice = 0;
  const size_t csmem = (!nnz && k0 == 0 &&
                        uint64_t((n + clu::kCols - 1) / clu::kCols) * clu::kCS <= uint64_t(ctx->num_sms) / 2)
                           ? cluster_smem(ctx, md, n, &wslice) : 0;
  if (csmem) {
    // small model: one cluster-pipelined launch; the last layer writes the
    // buffer the caller reads ((L - 1) & 1), the others ping-pong as usual
    launch_cluster_forward(ctx, p, p.buf[(p.L - 1) & 1], csmem, wslice);
    return;
  }
  const bool vec = (n % 4) == 0;
  const bool wide = vec && n >= 1024 && SK_ENG_KU > 1;
  const bool staged = wide && SK_ENG_BULK != 0;
  const void* fn = staged ? (const void*)k_dense_engine_bulk
                   : wide ? (const void*)k_dense_engine<true, SK_ENG_KU>
                   : vec ? (const void*)k_dense_engine<true> : (const void*)k_dense_engine<false>;
  const size_t esmem = staged ? bulk::kSmem : 0;
  if (staged) smem_attr(ctx, k_dense_engine_bulk, int(bulk::kSmem));
  // panel-major scratch for the intermediate layers (three layers or more: the
  // first reads and the last writes the caller's row-major buffers anyway)
  p.blk[0] = p.blk[1] = nullptr;
  p.work = nullptr;
  // (only while the two scratch copies stay small against the device)
  const bool blocked = staged && p.L >= 3 && SK_ENG_BLOCKED != 0 &&
                       double((n + 255) / 256) * 256.0 * m * 8.0 < 0.2 * double(ctx->total_mem);
  const bool claim = staged || (wide && SK_ENG_CLAIM_REG != 0);
  if (claim) {
    arena_begin(ctx);
    if (SK_ENG_CLAIM) {
      p.work = reinterpret_cast<unsigned long long*>(aalloc<uint64_t>(ctx, p.L));
      SK_CUDA(cudaMemsetAsync(p.work, 0, size_t(p.L) * 8, ctx->stream));
    }
  }
  if (blocked) {
    const size_t padded = size_t((n + 255) / 256) * 256 * m;
    p.blk[0] = aalloc<float>(ctx, padded);
    p.blk[1] = aalloc<float>(ctx, padded);
  }
  const int per_sm = kernel_occupancy(ctx, fn, 256, esmem);  // cached per device
  const uint32_t tcols = wide ? 128u * SK_ENG_KU : 128u;
  const uint64_t warps = uint64_t((n + tcols - 1) / tcols) * m;
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((warps + 7) / 8, uint64_t(ctx->num_sms) * std::max(per_sm, 1))));
  void* args[] = {&p};
  timing_mark(ctx, SK_KT_DENSE_ENGINE);
  SK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, esmem, ctx->stream));
  g_launches.fetch_add(1);
  timing_mark(ctx);
  if (claim) arena_end(ctx);  // stream-ordered: later arena users queue behind the engine
}

#ifndef SK_ROWS_WIDE_MIN
#define SK_ROWS_WIDE_MIN 1024
#endif
#ifndef SK_ROWS_BULK
#define SK_ROWS_BULK 1
#endif
// K1b standalone applies when the activations do not fit the L2 comfortably
// (> 48 MB): there the in-order claim keeps one column panel hot.  Smaller
// problems stay on the register-staged wide task (cfg2, 16 MB of Y: d = 0.1
// 0.39 ms against 0.44 staged).
static bool rows_bulk_applies(const sk_csr* w, uint32_t n) {
  return SK_ROWS_BULK && size_t(w->cols) * n * 4 > (size_t(48) << 20);
}

// The staged wide task (K1b) as a standalone layer / mxm: a zeroed task counter
// from the arena, one resident wave.
template <typename Ops, int kEpi>
static void launch_rows_bulk(sk_ctx* ctx, const sk_csr* w, const float* d_bias, const float* y,
                             uint32_t n, float clip, float* out) {
  auto* kern = k_spmm_rows_bulk<Ops, kEpi>;
  smem_attr(ctx, kern, int(bulk::kSmem));
  const int per_sm = std::max(1, occupancy(ctx, kern, 256, bulk::kSmem));
  const uint64_t warps = uint64_t((n + 255) / 256) * w->rows;
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((warps + 7) / 8, uint64_t(ctx->num_sms) * per_sm)));
  arena_begin(ctx);
  auto* work = reinterpret_cast<unsigned long long*>(aalloc<uint64_t>(ctx, 1));
  SK_CUDA(cudaMemsetAsync(work, 0, 8, ctx->stream));
  SK_LAUNCH(kern, grid, 256, bulk::kSmem, ctx->stream, w->rp, w->ci, w->v, d_bias, y, w->rows, n,
            clip, out, ctx->d_err, work);
  arena_end(ctx);
}
void launch_layer_dense(sk_ctx* ctx, const sk_csr* w, const float* d_bias, const float* y,
                        uint32_t n, float clip, float* out) {
  if (w->rows == 0 || n == 0) return;
  if (tile_applies(ctx, w, n)) {
    launch_tile(ctx, w, d_bias, y, n, clip, out, true);
    return;
  }
  if (launch_narrow<OpArith, kEpiLayer>(ctx, w, d_bias, y, n, clip, out)) return;
  const bool vec = (n % 4 == 0);
  // light rows (<= 16 stored entries on average) and wide activations: four
  // 128-column chunks per task
  const bool light = vec && n >= 512 && w->nnz <= size_t(16) * w->rows;
  if (light)
    SK_LAUNCH((k_spmm_rows<OpArith, kEpiLayer, true, 4>), spmm_grid(ctx, w->rows, n, 4), 256, 0,
              ctx->stream, w->rp, w->ci, w->v, d_bias, y, w->rows, n, clip, out, ctx->d_err);
  else if (vec && n >= SK_ROWS_WIDE_MIN && rows_bulk_applies(w, n))
    launch_rows_bulk<OpArith, kEpiLayer>(ctx, w, d_bias, y, n, clip, out);
  else if (vec && n >= SK_ROWS_WIDE_MIN)
    SK_LAUNCH((k_spmm_rows_wide<OpArith, kEpiLayer>), spmm_grid(ctx, w->rows, n, 2), 256, 0,
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
  if (s == SK_ARITHMETIC && tile_applies(ctx, a, n)) {
    launch_tile(ctx, a, nullptr, b, n, 0.0f, out, false);
    return;
  }
  dispatch_semiring(s, [&](auto ops) {
    using Ops = decltype(ops);
    if (launch_narrow<Ops, kEpiNone>(ctx, a, nullptr, b, n, 0.0f, out)) return;
    if (n % 4 == 0 && n >= SK_ROWS_WIDE_MIN && a->nnz > size_t(16) * a->rows &&
        rows_bulk_applies(a, n))
      launch_rows_bulk<Ops, kEpiNone>(ctx, a, nullptr, b, n, 0.0f, out);
    else if (n % 4 == 0 && n >= SK_ROWS_WIDE_MIN && a->nnz > size_t(16) * a->rows)
      SK_LAUNCH((k_spmm_rows_wide<Ops, kEpiNone>), spmm_grid(ctx, a->rows, n, 2), 256, 0,
                ctx->stream, a->rp, a->ci, a->v, nullptr, b, a->rows, n, 0.0f, out, ctx->d_err);
    else if (n % 4 == 0)
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
