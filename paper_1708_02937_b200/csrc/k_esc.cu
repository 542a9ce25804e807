// Thin layers by expand-sort-compress (ESC).
//
// When a layer's input is small against its (row, window) item space the
// windowed engine pays its per-item work for almost no products (cfg3 layer 2:
// 136 K inputs, ~4.4 M products spread over 967 K windows).  Here the products
// are generated directly instead: every input entry (k, j, y) walks the
// out-edges of neuron k (W^T row k: the in-edges of the reference orientation,
// dnn.cpp:65-103, seen from the input side) and emits (key = i*n + j, w_ik*y).
// Products are generated in input order -- ascending k -- so a STABLE radix
// sort by key leaves every output's products in ascending k, and the run-wise
// fold acc = +0, acc += p (ascending k) is the reference's fold bit for bit
// (semiring.hpp:59-66); z = epilogue(acc + b) and the z == 0 prune follow.  The
// sorted keys are the output's CSR order (row i, then sample j).
//
// Only layers with every bias <= 0 come here: a position without products then
// gives epilogue(0 + b) == 0, so outputs exist only where products exist.
#include <cub/cub.cuh>

#include <cstring>

#include "sk_common.cuh"

namespace sk {

namespace {

// deg[e] = out-degree of the input entry's neuron (warp per input row)
__global__ void k_esc_degrees(const uint32_t* yrp, uint32_t rows, const uint32_t* trp,
                              uint32_t* deg, size_t nnz) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < rows;
       k += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t d = trp[k + 1] - trp[k];
    for (uint32_t e = yrp[k] + lane; e < yrp[k + 1]; e += 32) deg[e] = d;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) deg[nnz] = 0;  // scan sentinel -> total
}

// products of input row k: entry e writes its out-edges at off[e] .. off[e]+d
template <typename K>
__global__ void k_esc_expand(const uint32_t* yrp, const uint32_t* yci, const float* yv,
                             uint32_t rows, uint32_t n, const uint32_t* trp,
                             const uint32_t* tci, const float* tv, const uint32_t* off,
                             K* keys, float* vals) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < rows;
       k += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t tb = trp[k], d = trp[k + 1] - tb;
    if (d == 0) continue;
    for (uint32_t e = yrp[k]; e < yrp[k + 1]; ++e) {
      const uint32_t j = yci[e];
      const float y = yv[e];
      const uint32_t o = off[e];
      for (uint32_t t = lane; t < d; t += 32) {
        const uint32_t i = tci[tb + t];
        keys[o + t] = K(i) * K(n) + K(j);
        vals[o + t] = __fmul_rn(tv[tb + t], y);
      }
    }
  }
}

// run heads fold their run (ascending k) and apply the layer epilogue
template <typename K>
__global__ void k_esc_fold(const K* keys, const float* vals, uint32_t P, uint32_t n,
                           const float* bias, float clip, uint32_t* keep, float* z) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < P; t += gridDim.x * blockDim.x) {
    const K key = keys[t];
    uint32_t f = 0;
    if (t == 0 || keys[t - 1] != key) {
      float acc = 0.0f;
      for (uint32_t u = t; u < P && keys[u] == key; ++u) acc = __fadd_rn(acc, vals[u]);
      const float zz = layer_epilogue(acc, bias[uint32_t(key / K(n))], clip);
      f = zz != 0.0f ? 1u : 0u;
      z[t] = zz;
    }
    keep[t] = f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) keep[P] = 0;
}

template <typename K>
__global__ void k_esc_scatter(const K* keys, const float* z, const uint32_t* keep,
                              const uint32_t* pos, uint32_t P, uint32_t n, K* okey,
                              uint32_t* oci, float* ov) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < P; t += gridDim.x * blockDim.x)
    if (keep[t]) {
      const uint32_t s = pos[t];
      okey[s] = keys[t];
      oci[s] = uint32_t(keys[t] % K(n));
      ov[s] = z[t];
    }
}

// row_ptr[i] = first survivor with row >= i (sorted keys)
template <typename K>
__global__ void k_esc_row_ptr(const K* okey, uint32_t S, uint32_t rows, uint32_t n,
                              uint32_t* rp) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
       i += gridDim.x * blockDim.x) {
    const K lo_key = K(i) * K(n);
    uint32_t lo = 0, hi = S;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (okey[mid] < lo_key) lo = mid + 1;
      else hi = mid;
    }
    rp[i] = lo;
  }
}

// ---- small layers: one block does everything in shared memory ------------------
// (products <= kSmallCap: expand, bitonic sort, run fold, compaction, CSR)
constexpr int kSmallThreads = 1024, kSmallItems = 2;
constexpr uint32_t kSmallCap = uint32_t(kSmallThreads) * kSmallItems;  // products
constexpr uint32_t kSmallEntries = 512;                                 // input entries


unsigned grid_of(sk_ctx* ctx, uint64_t threads) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((threads + 255) / 256,
                                                            uint64_t(ctx->num_sms) * 16)));
}

int bits_for(uint64_t v) {  // smallest b with v <= 2^b
  int b = 0;
  while (b < 64 && (uint64_t(1) << b) < v) ++b;
  return b;
}

// The whole tiny layer in one CTA (<= kSmallEntries inputs, <= kSmallCap
// products): input rows by binary search (or, for K7's unsorted output read
// straight from its scratch, given per entry and the inputs sorted by (row,
// column) first), products expanded, a bitonic sort of
// (i n + j) << 11 | product index in shared memory (the product index breaks
// ties, so a run lists its products in input order = ascending k), run folds
// + epilogue, compaction, and the output CSR written directly (column, value
// and all m + 1 row pointers, each by a binary search of the survivors' rows);
// the host reads back only the count.  Replaces a row-id kernel, a block radix
// sort over every key bit and three finishing launches (cfg4 layer 2, 24
// inputs: ~30 -> ~6 us).
__global__ void __launch_bounds__(kSmallThreads)
    k_esc_tiny(const uint32_t* __restrict__ yrp, uint32_t rows, const uint32_t* __restrict__ yci,
               const float* __restrict__ yv, uint32_t nnz, uint32_t n,
               const uint32_t* __restrict__ trp, const uint32_t* __restrict__ tci,
               const float* __restrict__ tv, uint32_t m, const float* __restrict__ bias,
               float clip, uint32_t* __restrict__ oci,
               float* __restrict__ ov, uint32_t* __restrict__ count,
               const uint32_t* __restrict__ nnz_dev, uint32_t* __restrict__ handled,
               uint32_t* __restrict__ orow, const uint32_t* __restrict__ in_row) {
  __shared__ unsigned long long skey[kSmallCap];
  __shared__ float sval[kSmallCap];
  __shared__ uint32_t s_off[kSmallEntries + 1];
  __shared__ uint32_t s_tb[kSmallEntries];
  __shared__ uint32_t s_row[kSmallCap];  // input entries' rows, later the survivors' rows
  __shared__ uint32_t s_col[kSmallEntries];  // input entries' columns and values
  __shared__ float s_val[kSmallEntries];
  __shared__ uint32_t s_wsum[kSmallThreads / 32];
  constexpr uint32_t kIdx = 2049;
  static_assert(kIdx * 4 <= sizeof(skey), "the row-pointer samples live in skey");
  uint32_t* const s_idx = reinterpret_cast<uint32_t*>(skey);  // every 2^lst-th row pointer
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // block-wide exclusive sum of one value per thread
  auto block_excl = [&](uint32_t v, uint32_t& total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= uint32_t(o)) x += t;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t w = s_wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= uint32_t(o)) w += t;
      }
      s_wsum[lane] = w;
    }
    __syncthreads();
    total = s_wsum[31];
    const uint32_t ex = x - v + (wid ? s_wsum[wid - 1] : 0u);
    __syncthreads();
    return ex;
  };
  // bitonic sort of skey[0, P2), two keys per thread (indices tid, tid + 1024)
  // in registers: partners closer than 32 are in the same warp (shuffles, no
  // barrier); the farther ones go through shared memory, one barrier each
  auto sort_keys = [&](uint32_t P2) {
    unsigned long long v[2];
    v[0] = skey[tid];
    v[1] = tid + kSmallThreads < P2 ? skey[tid + kSmallThreads] : ~0ull;
    const bool two = P2 > kSmallThreads;
    for (uint32_t k = 2; k <= P2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        if (j >= 32) {
          __syncthreads();  // the previous round's reads are done
          skey[tid] = v[0];
          if (two) skey[tid + kSmallThreads] = v[1];
          __syncthreads();
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const uint32_t i = tid + h * kSmallThreads;
          unsigned long long o;
          if (j >= 32) {
            o = skey[i ^ j];
          } else {
            const uint32_t lo32 = __shfl_xor_sync(0xffffffffu, uint32_t(v[h]), j);
            const uint32_t hi32 = __shfl_xor_sync(0xffffffffu, uint32_t(v[h] >> 32), j);
            o = (unsigned long long)hi32 << 32 | lo32;
          }
          // the lower index of an ascending pair keeps the minimum
          const bool lower = (i & j) == 0, up = (i & k) == 0;
          const bool take_min = lower == up;
          v[h] = take_min ? (o < v[h] ? o : v[h]) : (o > v[h] ? o : v[h]);
        }
      }
    }
    __syncthreads();
    skey[tid] = v[0];
    if (two) skey[tid + kSmallThreads] = v[1];
    __syncthreads();
  };
  // deferred launch (the input's entry count is only on the device): a layer
  // beyond the tiny limits is left to the host (handled = 0, nothing written)
  if (nnz_dev) {
    nnz = *nnz_dev;
    if (nnz > kSmallEntries) {
      if (tid == 0) *handled = 0u, *count = 0u;
      return;
    }
  }
  // 1. each input entry's row: given by the producer (in_row), or from the
  //    row pointers sampled every 2^lst rows into shared memory (one coalesced
  //    load per thread), then per entry a binary search there and one of
  //    <= log2(2^lst) global steps inside its block -- not ~17 dependent L2 round
  //    trips, and not a walk over every row
  if (in_row) {
    // unsorted inputs (K7's scratch): sorted by (row, column) -- a run's
    // products then fold in ascending k, as the reference's mxm does
    uint32_t P2 = 1;
    while (P2 < nnz) P2 <<= 1;
    for (uint32_t q = tid; q < P2; q += kSmallThreads)
      skey[q] = q < nnz ? ((unsigned long long)in_row[q] * n + yci[q]) << 9 | q : ~0ull;
    __syncthreads();
    sort_keys(P2);
    if (tid < nnz) {
      const uint32_t e = uint32_t(skey[tid] & 511u);
      s_row[tid] = in_row[e];
      s_col[tid] = yci[e];
      s_val[tid] = yv[e];
    }
  } else {
    uint32_t lst = 6;
    while ((uint32_t(kIdx - 1) << lst) < rows) ++lst;
    const uint32_t nb = (rows + (1u << lst) - 1) >> lst;  // blocks (<= kIdx - 1)
    for (uint32_t b = tid; b <= nb; b += kSmallThreads) s_idx[b] = yrp[min(b << lst, rows)];
    __syncthreads();
    if (tid < nnz) {
      uint32_t lo = 0, hi = nb;  // last block with s_idx[b] <= tid
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_idx[mid] <= tid) lo = mid; else hi = mid;
      }
      uint32_t rlo = lo << lst, rhi = min(rows, (lo + 1) << lst);  // last row with yrp <= tid
      while (rhi - rlo > 1) {
        const uint32_t mid = (rlo + rhi) >> 1;
        if (yrp[mid] <= tid) rlo = mid; else rhi = mid;
      }
      s_row[tid] = rlo;
      s_col[tid] = yci[tid];
      s_val[tid] = yv[tid];
    }
  }
  __syncthreads();
  uint32_t deg = 0;
  if (tid < nnz) {
    const uint32_t k = s_row[tid];
    const uint32_t tb = trp[k];
    s_tb[tid] = tb;
    deg = trp[k + 1] - tb;
  }
  uint32_t P;
  const uint32_t eo = block_excl(deg, P);
  if (handled && P > kSmallCap) {  // block-uniform
    if (tid == 0) *handled = 0u, *count = 0u;
    return;
  }
  if (tid < nnz) s_off[tid] = eo;
  if (tid == 0) s_off[nnz] = P;
  __syncthreads();
  uint32_t P2 = 1;
  while (P2 < P) P2 <<= 1;
  // 2. expand: product q of entry e = (W^T row entry, input entry)
  for (uint32_t q = tid; q < P2; q += kSmallThreads) {
    if (q < P) {
      uint32_t lo = 0, hi = nnz;  // last entry with s_off[e] <= q
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_off[mid] <= q) lo = mid; else hi = mid;
      }
      const uint32_t t = s_tb[lo] + (q - s_off[lo]);
      skey[q] = ((unsigned long long)tci[t] * n + s_col[lo]) << 11 | q;
      sval[q] = __fmul_rn(tv[t], s_val[lo]);
    } else {
      skey[q] = ~0ull;  // padding sorts last
    }
  }
  __syncthreads();
  // 3. bitonic sort of the P2 product keys
  sort_keys(P2);
  // 4. run heads fold their products in order, epilogue; 5. compaction
  float z[kSmallItems];
  uint32_t keep[kSmallItems];
  uint32_t mine = 0;
#pragma unroll
  for (int u = 0; u < kSmallItems; ++u) {
    const uint32_t q = tid * kSmallItems + u;
    keep[u] = 0;
    z[u] = 0.0f;
    if (q < P) {
      const unsigned long long key = skey[q] >> 11;
      if (q == 0 || (skey[q - 1] >> 11) != key) {
        float acc = 0.0f;
        for (uint32_t r = q; r < P && (skey[r] >> 11) == key; ++r)
          acc = __fadd_rn(acc, sval[uint32_t(skey[r] & 2047u)]);
        z[u] = layer_epilogue(acc, bias[uint32_t(key / n)], clip);
        keep[u] = z[u] != 0.0f ? 1u : 0u;
      }
    }
    mine += keep[u];
  }
  uint32_t S;
  uint32_t pos = block_excl(mine, S);
#pragma unroll
  for (int u = 0; u < kSmallItems; ++u)
    if (keep[u]) {
      const unsigned long long key = skey[tid * kSmallItems + u] >> 11;
      const uint32_t i = uint32_t(key / n);
      oci[pos] = uint32_t(key - (unsigned long long)i * n);
      ov[pos] = z[u];
      s_row[pos] = i;
      ++pos;
    }
  __syncthreads();
  // 6. the survivors' rows (sorted) for the row-pointer kernel that follows
  for (uint32_t t = tid; t < S; t += kSmallThreads) orow[t] = s_row[t];
  if (tid == 0) {
    *count = S;
    if (handled) *handled = 1u;
  }
}

// rp[r] = survivors in rows < r (the survivors' rows sorted, count on the device)
__global__ void k_esc_fill_rp(const uint32_t* __restrict__ orow, const uint32_t* __restrict__ count,
                              uint32_t m, uint32_t* __restrict__ rp) {
  const uint32_t S = *count;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= m; r += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = S;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(orow + mid) < r) lo = mid + 1; else hi = mid;
    }
    rp[r] = lo;
  }
}

sk_csr* esc_tiny(sk_ctx* ctx, const sk_csr* y, const sk_csr* wt, const float* bias, float clip,
                 uint32_t maxdeg) {
  const uint32_t m = wt->cols, n = y->cols;
  const size_t capn = std::max<size_t>(1, size_t(y->nnz) * maxdeg);  // <= kSmallCap
  sk_csr* out = new_csr(ctx, m, n, capn);
  uint32_t* cnt = aalloc<uint32_t>(ctx, 1);
  uint32_t* orow = aalloc<uint32_t>(ctx, kSmallCap);
  SK_LAUNCH(k_esc_tiny, 1, kSmallThreads, 0, ctx->stream, y->rp, y->rows, y->ci, y->v,
            uint32_t(y->nnz), n, wt->rp, wt->ci, wt->v, m, bias, clip, out->ci, out->v,
            cnt, nullptr, nullptr, orow, nullptr);
  SK_LAUNCH(k_esc_fill_rp, grid_of(ctx, uint64_t(m) + 1), 256, 0, ctx->stream, orow, cnt, m,
            out->rp);
  out->nnz = Fetch(ctx).add(cnt, 1).run()[0];  // mailbox; the arrays keep their capacity
  return out;
}

// ---- sample-major ESC: one warp accumulates one sample ---------------------------
//
// The global ESC sorts ALL products by (i, j) (cfg3 layer 2: 4.4 M products, four
// 8-bit onesweep passes, ~0.2 ms).  Seen per sample j the products are few (cfg3
// layer 2: ~73 from ~2.3 active inputs), so one warp owns one sample: it walks the
// sample's active inputs k in ASCENDING order (a counting transpose of Y gives
// the entries; the warp ranks them) and adds each W^T row's products into a
// per-warp shared-memory hash table keyed by output row i.  The i of one W^T row
// are distinct, so within a step every slot sees one add, and across steps the
// adds arrive in ascending k: each slot folds acc = +0, acc += w_ik y_kj exactly
// as the reference's merge does (matrix.cpp:452-521 + dnn.cpp:65-103).  Then
// z = epilogue(acc + b_i) per occupied slot; survivors are appended as
// (i n + j, z) and sorted into CSR.  A sample with more than 32 active inputs
// or more distinct rows than the small table holds is queued for a one-warp
// block with a 16 K-slot table that sorts the entries first; beyond that the
// layer falls back to the global sort.
constexpr uint32_t kEmptySlot = 0xFFFFFFFFu;
constexpr int kSampWarps = 8;
constexpr uint32_t kSampSlots = 256, kSampBudget = 192;  // small kernel, per warp
constexpr uint32_t kBigSlots = 4096, kBigBudget = 3072;  // big kernel, one warp per block
constexpr uint32_t kBigEntries = 1024;                   // active inputs per sample, big kernel
constexpr size_t kBigSmem = size_t(kBigSlots) * 8 + size_t(kBigBudget) * 2 + size_t(kBigEntries) * 8;

__global__ void k_tv_count(const uint32_t* __restrict__ ci, size_t nnz, uint32_t* __restrict__ cnt) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += size_t(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[ci[e]], 1u);
}

// entries of input row k -> their sample's list (k and the value; list order free)
__global__ void k_tv_scatter(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             const float* __restrict__ v, uint32_t rows,
                             uint32_t* __restrict__ cursor, uint2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < rows;
       k += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t e = rp[k] + lane; e < rp[k + 1]; e += 32)
      out[atomicAdd(&cursor[ci[e]], 1u)] = make_uint2(k, __float_as_uint(v[e]));
}

struct SampArgs {
  const uint32_t* yt_rp;
  const uint2* yt;
  uint32_t n;
  const uint32_t* trp;
  const uint32_t* tci;
  const float* tv;
  const float* bias;
  float clip;
  unsigned long long* okey;
  float* oval;
  unsigned long long cap;
  unsigned long long* ctr;  // [0] survivors, [1] overflow flag, [2] queued samples
  uint32_t* queue;
};

// One product per lane into the warp's table (keys/acc of H slots; list holds
// the occupied slots from index `used`).  Returns the slots newly occupied.
template <uint32_t H>
__device__ __forceinline__ uint32_t tab_add(uint32_t* keys, float* acc, uint16_t* list,
                                            uint32_t used, bool live, uint32_t i, float p,
                                            int lane) {
  bool fresh = false;
  uint32_t s = (i * 2654435761u) & (H - 1);
  if (live) {
    for (;;) {
      const uint32_t prev = atomicCAS(&keys[s], kEmptySlot, i);
      if (prev == kEmptySlot) {
        fresh = true;
        break;
      }
      if (prev == i) break;
      s = (s + 1) & (H - 1);
    }
    acc[s] = __fadd_rn(acc[s], p);  // fresh slots hold +0
  }
  const unsigned b = __ballot_sync(0xffffffffu, fresh);
  if (fresh) list[used + __popc(b & ((1u << lane) - 1u))] = uint16_t(s);
  return __popc(b);
}

// W^T row entries [t0, te) of one input (activation y) into the table.
template <uint32_t H>
__device__ __forceinline__ uint32_t tab_add_range(const SampArgs& a, uint32_t* keys, float* acc,
                                                  uint16_t* list, uint32_t used, uint32_t t0,
                                                  uint32_t te, float y, int lane) {
  uint32_t added = 0;
  for (uint32_t base = t0; base < te; base += 32) {
    const uint32_t t = base + lane;
    const bool live = t < te;
    const uint32_t i = live ? a.tci[t] : 0u;
    const float w = live ? a.tv[t] : 0.0f;
    added += tab_add<H>(keys, acc, list, used + added, live, i, __fmul_rn(w, y), lane);
  }
  return added;
}

// Occupied slots: epilogue, survivors appended, slots reset for the next sample.
__device__ __forceinline__ void tab_flush(const SampArgs& a, uint32_t* keys, float* acc,
                                          const uint16_t* list, uint32_t used, uint32_t j,
                                          int lane, bool emit) {
  __syncwarp();
  for (uint32_t t = lane; t < used; t += 32) {
    const uint32_t s = list[t], i = keys[s];
    if (emit) {
      const float z = layer_epilogue(acc[s], a.bias[i], a.clip);
      if (z != 0.0f) {
        const unsigned long long pos = atomicAdd(&a.ctr[0], 1ull);
        if (pos < a.cap) {
          a.okey[pos] = (unsigned long long)i * a.n + j;
          a.oval[pos] = z;
        }
      }
    }
    keys[s] = kEmptySlot;
    acc[s] = 0.0f;
  }
  __syncwarp();
}

// One warp per sample with at most 32 active inputs: inputs ranked by k in
// registers, each input's first 32 W^T entries loaded one input ahead.
__global__ void __launch_bounds__(kSampWarps * 32) k_esc_sample(SampArgs a) {
  __shared__ uint32_t skeys[kSampWarps][kSampSlots];
  __shared__ float sacc[kSampWarps][kSampSlots];
  __shared__ uint16_t slist[kSampWarps][kSampBudget];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* const keys = skeys[wid];
  float* const acc = sacc[wid];
  uint16_t* const list = slist[wid];
  for (uint32_t s = lane; s < kSampSlots; s += 32) {
    keys[s] = kEmptySlot;
    acc[s] = 0.0f;
  }
  __syncwarp();
  const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
  uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t nb0 = 0, nb1 = 0;
  if (j < a.n) {
    nb0 = a.yt_rp[j];
    nb1 = a.yt_rp[j + 1];
  }
  for (; j < a.n; j += stride) {
    const uint32_t e0 = nb0, E = nb1 - nb0;
    if (j + stride < a.n) {  // next sample's bounds, one sample ahead
      nb0 = a.yt_rp[j + stride];
      nb1 = a.yt_rp[j + stride + 1];
    }
    if (E == 0) continue;
    if (E > 32) {  // warp-uniform
      if (lane == 0) a.queue[atomicAdd(&a.ctr[2], 1ull)] = j;
      continue;
    }
    const bool mine = uint32_t(lane) < E;
    uint2 ent = make_uint2(kEmptySlot, 0u);
    uint32_t tb = 0, te = 0;
    if (mine) {
      ent = a.yt[e0 + lane];
      tb = a.trp[ent.x];
      te = a.trp[ent.x + 1];
    }
    uint32_t rank = 0;  // position of this lane's input in ascending k (k distinct)
    for (uint32_t q = 0; q < E; ++q) rank += __shfl_sync(0xffffffffu, ent.x, q) < ent.x;
    int src = __ffs(__ballot_sync(0xffffffffu, mine && rank == 0)) - 1;
    uint32_t ctb = __shfl_sync(0xffffffffu, tb, src), cte = __shfl_sync(0xffffffffu, te, src);
    float cy = __uint_as_float(__shfl_sync(0xffffffffu, ent.y, src));
    bool cl = ctb + lane < cte;
    uint32_t ci = cl ? a.tci[ctb + lane] : 0u;
    float cw = cl ? a.tv[ctb + lane] : 0.0f;
    uint32_t used = 0;
    bool over = false;
    for (uint32_t q = 0; q < E; ++q) {
      uint32_t ntb = 0, nte = 0, ni = 0;
      float ny = 0.0f, nw = 0.0f;
      bool nl = false;
      if (q + 1 < E) {
        src = __ffs(__ballot_sync(0xffffffffu, mine && rank == q + 1)) - 1;
        ntb = __shfl_sync(0xffffffffu, tb, src);
        nte = __shfl_sync(0xffffffffu, te, src);
        ny = __uint_as_float(__shfl_sync(0xffffffffu, ent.y, src));
        nl = ntb + lane < nte;
        if (nl) {
          ni = a.tci[ntb + lane];
          nw = a.tv[ntb + lane];
        }
      }
      if (used + (cte - ctb) > kSampBudget) {
        over = true;
        break;
      }
      used += tab_add<kSampSlots>(keys, acc, list, used, cl, ci, __fmul_rn(cw, cy), lane);
      if (cte - ctb > 32)
        used += tab_add_range<kSampSlots>(a, keys, acc, list, used, ctb + 32, cte, cy, lane);
      __syncwarp();
      ctb = ntb;
      cte = nte;
      cy = ny;
      ci = ni;
      cw = nw;
      cl = nl;
    }
    if (over && lane == 0) a.queue[atomicAdd(&a.ctr[2], 1ull)] = j;
    tab_flush(a, keys, acc, list, used, j, lane, !over);
  }
}

// One warp per queued sample: inputs sorted by k in shared memory (bitonic),
// then the same ascending-k accumulation into a 4 K-slot table.
__global__ void __launch_bounds__(32) k_esc_sample_big(SampArgs a) {
  extern __shared__ __align__(16) uint32_t big_smem[];
  uint32_t* const keys = big_smem;
  float* const acc = reinterpret_cast<float*>(keys + kBigSlots);
  uint32_t* const ek = reinterpret_cast<uint32_t*>(acc + kBigSlots);
  float* const ev = reinterpret_cast<float*>(ek + kBigEntries);
  uint16_t* const list = reinterpret_cast<uint16_t*>(ev + kBigEntries);
  const int lane = threadIdx.x;
  const uint32_t nq = uint32_t(a.ctr[2]);
  if (blockIdx.x >= nq) return;
  for (uint32_t s = lane; s < kBigSlots; s += 32) {
    keys[s] = kEmptySlot;
    acc[s] = 0.0f;
  }
  __syncwarp();
  for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
    const uint32_t j = a.queue[q];
    const uint32_t e0 = a.yt_rp[j], E = a.yt_rp[j + 1] - e0;
    if (E > kBigEntries) {
      if (lane == 0) a.ctr[1] = 1;
      continue;
    }
    uint32_t n2 = 32;
    while (n2 < E) n2 <<= 1;
    for (uint32_t t = lane; t < n2; t += 32) {
      const uint2 e = t < E ? a.yt[e0 + t] : make_uint2(kEmptySlot, 0u);
      ek[t] = e.x;
      ev[t] = __uint_as_float(e.y);
    }
    __syncwarp();
    for (uint32_t size = 2; size <= n2; size <<= 1)
      for (uint32_t half = size >> 1; half; half >>= 1) {
        for (uint32_t t = lane; t < (n2 >> 1); t += 32) {
          const uint32_t x = 2 * t - (t & (half - 1)), z = x + half;
          const uint32_t kx = ek[x], kz = ek[z];
          if ((kx > kz) == ((x & size) == 0)) {
            const float vx = ev[x];
            ek[x] = kz;
            ek[z] = kx;
            ev[x] = ev[z];
            ev[z] = vx;
          }
        }
        __syncwarp();
      }
    uint32_t used = 0;
    bool over = false;
    for (uint32_t e = 0; e < E; ++e) {
      const uint32_t k = ek[e], tb = a.trp[k], te = a.trp[k + 1];
      if (used + (te - tb) > kBigBudget) {
        over = true;
        break;
      }
      used += tab_add_range<kBigSlots>(a, keys, acc, list, used, tb, te, ev[e], lane);
      __syncwarp();
    }
    if (over && lane == 0) a.ctr[1] = 1;
    tab_flush(a, keys, acc, list, used, j, lane, !over);
  }
}

__global__ void k_samp_csr(const unsigned long long* __restrict__ key, const float* __restrict__ val,
                           size_t cnt, uint32_t n, uint32_t* __restrict__ rows_cnt,
                           uint32_t* __restrict__ ci, float* __restrict__ v) {
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < cnt;
       q += size_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[q];
    const uint32_t i = uint32_t(k / n);
    ci[q] = uint32_t(k - (unsigned long long)i * n);
    v[q] = val[q];
    atomicAdd(&rows_cnt[i], 1u);
  }
}

// nullptr when a sample exceeds the big table (the caller falls back)
sk_csr* esc_sample(sk_ctx* ctx, const sk_csr* y, const sk_csr* wt, const float* bias,
                   float clip) {
  const uint32_t m = wt->cols, n = y->cols, rows = y->rows;
  // Y^T with values (counting transpose; per-sample order is fixed by the warp)
  uint32_t* yt_rp = aalloc<uint32_t>(ctx, size_t(n) + 1);
  uint32_t* cur = aalloc<uint32_t>(ctx, size_t(n) + 1);
  uint2* yt = aalloc<uint2>(ctx, std::max<size_t>(y->nnz, 1));
  uint32_t* queue = aalloc<uint32_t>(ctx, std::max<uint32_t>(n, 1));
  SK_CUDA(cudaMemsetAsync(cur, 0, (size_t(n) + 1) * 4, ctx->stream));
  SK_LAUNCH(k_tv_count, grid_of(ctx, y->nnz), 256, 0, ctx->stream, y->ci, y->nnz, cur);
  exclusive_scan_u32(ctx, cur, yt_rp, size_t(n) + 1);
  SK_CUDA(cudaMemcpyAsync(cur, yt_rp, size_t(n) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  SK_LAUNCH(k_tv_scatter, grid_of(ctx, uint64_t(rows) * 32), 256, 0, ctx->stream, y->rp, y->ci,
            y->v, rows, cur, yt);
  smem_attr(ctx, k_esc_sample_big, int(kBigSmem));
  const int occ = occupancy(ctx, k_esc_sample, kSampWarps * 32, 0);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(ctx->d_u64);
  unsigned long long cap = std::max<unsigned long long>(1u << 16, y->nnz);
  for (int attempt = 0; attempt < 2; ++attempt) {
    SampArgs a{yt_rp, yt, n, wt->rp, wt->ci, wt->v, bias, clip, nullptr, nullptr, cap, ctr, queue};
    a.okey = aalloc<unsigned long long>(ctx, cap);
    a.oval = aalloc<float>(ctx, cap);
    SK_CUDA(cudaMemsetAsync(ctr, 0, 24, ctx->stream));
    const unsigned grid = unsigned(std::min<uint64_t>((uint64_t(n) + kSampWarps - 1) / kSampWarps,
                                                      uint64_t(ctx->num_sms) * occ));
    SK_LAUNCH(k_esc_sample, grid, kSampWarps * 32, 0, ctx->stream, a);
    SK_LAUNCH(k_esc_sample_big, unsigned(ctx->num_sms) * 4, 32, kBigSmem, ctx->stream, a);
    unsigned long long h[2];  // survivors, overflow: through the mailbox
    std::memcpy(h, Fetch(ctx).add(ctr, 4).run(), sizeof(h));
    if (getenv("SK_ESC_DEBUG")) {
      unsigned long long qd = 0;
      SK_CUDA(cudaMemcpy(&qd, ctr + 2, 8, cudaMemcpyDeviceToHost));
      fprintf(stderr, "esc_sample: n=%u nnz=%llu queued=%llu survivors=%llu overflow=%llu\n", n,
              (unsigned long long)y->nnz, qd, h[0], h[1]);
    }
    if (h[1]) return nullptr;  // a sample beyond the big table
    const unsigned long long cnt = h[0];
    if (cnt > cap) {
      cap = cnt;
      continue;
    }
    unsigned long long* k2 = aalloc<unsigned long long>(ctx, std::max<unsigned long long>(cnt, 1));
    float* v2 = aalloc<float>(ctx, std::max<unsigned long long>(cnt, 1));
    if (cnt) {
      const int end_bit = bits_for(uint64_t(m) * n);
      size_t tmp = 0;
      SK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a.okey, k2, a.oval, v2, cnt, 0,
                                              end_bit, ctx->stream));
      void* t = aalloc<char>(ctx, tmp);
      SK_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, a.okey, k2, a.oval, v2, cnt, 0, end_bit,
                                              ctx->stream));
      g_launches.fetch_add(1);
    }
    sk_csr* o = new_csr(ctx, m, n, cnt);
    uint32_t* rc = aalloc<uint32_t>(ctx, size_t(m) + 1);
    SK_CUDA(cudaMemsetAsync(rc, 0, (size_t(m) + 1) * 4, ctx->stream));
    if (cnt)
      SK_LAUNCH(k_samp_csr, grid_of(ctx, cnt), 256, 0, ctx->stream, k2, v2, cnt, n, rc, o->ci,
                o->v);
    exclusive_scan_u32(ctx, rc, o->rp, size_t(m) + 1);
    return o;
  }
  fail(SK_ERR, "sample-major ESC: survivor count changed between attempts");
}

template <typename K>
sk_csr* esc_run(sk_ctx* ctx, const sk_csr* y, const sk_csr* wt, const float* bias, float clip,
                uint32_t maxdeg) {
  if (y->nnz <= kSmallEntries && double(y->nnz) * double(maxdeg) <= double(kSmallCap) &&
      y->rows >= 1 && double(wt->cols) * double(y->cols) < 9.0e15)  // (i n + j) << 11 in 64 bits
    return esc_tiny(ctx, y, wt, bias, clip, maxdeg);
  // sample-major (per-warp tables) when a sample holds few products on average;
  // a sample beyond the big table sends the layer to the global sort below
  const double per_sample = double(y->nnz) * double(wt->nnz) / double(std::max<uint32_t>(1, wt->rows)) /
                            double(std::max<uint32_t>(1, y->cols));
  if (per_sample <= 128.0 && ctx->tune.esc >= 0) {
    if (sk_csr* o = esc_sample(ctx, y, wt, bias, clip)) return o;
  }
  const uint32_t m = wt->cols, n = y->cols, rows = y->rows;
  const size_t nnz = y->nnz;
  // 1. per-entry product counts, scanned (sentinel entry -> total)
  uint32_t* deg = aalloc<uint32_t>(ctx, nnz + 1);
  uint32_t* off = aalloc<uint32_t>(ctx, nnz + 1);
  SK_LAUNCH(k_esc_degrees, grid_of(ctx, uint64_t(rows) * 32), 256, 0, ctx->stream, y->rp, rows,
            wt->rp, deg, nnz);
  size_t tmp = 0;
  SK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg, off, nnz + 1, ctx->stream));
  void* t0 = aalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceScan::ExclusiveSum(t0, tmp, deg, off, nnz + 1, ctx->stream));
  g_launches.fetch_add(1);
  const uint32_t P = Fetch(ctx).add(off + nnz, 1).run()[0];
  sk_csr* out = nullptr;
  if (P == 0) {
    out = new_csr(ctx, m, n, 0);
    SK_CUDA(cudaMemsetAsync(out->rp, 0, (size_t(m) + 1) * 4, ctx->stream));
    return out;
  }
  // 2. expand, 3. stable sort by (i, j)
  K* k0 = aalloc<K>(ctx, P);
  K* k1 = aalloc<K>(ctx, P);
  float* v0 = aalloc<float>(ctx, P);
  float* v1 = aalloc<float>(ctx, P);
  SK_LAUNCH(k_esc_expand<K>, grid_of(ctx, uint64_t(rows) * 32), 256, 0, ctx->stream, y->rp,
            y->ci, y->v, rows, n, wt->rp, wt->ci, wt->v, off, k0, v0);
  const int end_bit = bits_for(uint64_t(m) * n);
  tmp = 0;
  SK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, P, 0, end_bit,
                                          ctx->stream));
  void* t1 = aalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceRadixSort::SortPairs(t1, tmp, k0, k1, v0, v1, P, 0, end_bit, ctx->stream));
  g_launches.fetch_add(1);
  // 4. fold runs + epilogue, 5. compact survivors
  uint32_t* keep = aalloc<uint32_t>(ctx, size_t(P) + 1);
  uint32_t* pos = aalloc<uint32_t>(ctx, size_t(P) + 1);
  float* z = v0;  // free after the sort
  SK_LAUNCH(k_esc_fold<K>, grid_of(ctx, P), 256, 0, ctx->stream, k1, v1, P, n, bias, clip, keep,
            z);
  tmp = 0;
  SK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, keep, pos, size_t(P) + 1, ctx->stream));
  void* t2 = aalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceScan::ExclusiveSum(t2, tmp, keep, pos, size_t(P) + 1, ctx->stream));
  g_launches.fetch_add(1);
  const uint32_t S = Fetch(ctx).add(pos + P, 1).run()[0];
  out = new_csr(ctx, m, n, S);
  K* okey = k0;  // free after the sort
  if (S)
    SK_LAUNCH(k_esc_scatter<K>, grid_of(ctx, P), 256, 0, ctx->stream, k1, z, keep, pos, P, n,
              okey, out->ci, out->v);
  SK_LAUNCH(k_esc_row_ptr<K>, grid_of(ctx, uint64_t(m) + 1), 256, 0, ctx->stream, okey, S, m, n,
            out->rp);
  return out;
}

}  // namespace

__global__ void k_esc_max_row(const uint32_t* rp, uint32_t rows, unsigned int* out) {
  unsigned int mx = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    mx = max(mx, rp[i + 1] - rp[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// W^T of layer k (out-edges of every neuron) and its longest row, built on
// first use and cached with the model.
const sk_csr* model_layer_transpose(sk_ctx* ctx, sk_model* mm, uint32_t k) {
  if (mm->wT.size() != mm->layers) {
    mm->wT.assign(mm->layers, nullptr);
    mm->wT_maxdeg.assign(mm->layers, 0);
  }
  if (!mm->wT[k]) {
    sk_csr* t = csr_transpose(ctx, mm->w[k]);
    unsigned int* d = dalloc<unsigned int>(ctx, 1);
    SK_CUDA(cudaMemsetAsync(d, 0, 4, ctx->stream));
    SK_LAUNCH(k_esc_max_row, grid_of(ctx, t->rows), 256, 0, ctx->stream, t->rp, t->rows, d);
    unsigned int h = 0;
    SK_CUDA(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    dfree(ctx, d);
    mm->wT[k] = t;
    mm->wT_maxdeg[k] = h;
  }
  return mm->wT[k];
}

// ESC pays for the layer's products (estimated from the mean degree) where the
// windowed engine pays per (row, window) item: taken while the products stay
// within `ratio` per item, and while the exact product count fits the 32-bit
// offsets (input entries * longest W^T row).
bool esc_applicable(sk_ctx* ctx, const sk_model* md, uint32_t k, const sk_csr* y, double ratio) {
  if (!md->bias_nonpos[k] || y->nnz == 0) return false;
  const double m = double(std::max<uint32_t>(1, md->neurons));
  const double est = double(y->nnz) * double(md->w[k]->nnz) / m;
  const double items = m * double((uint64_t(y->cols) + 1023) / 1024);
  if (est > ratio * items || est > double(1u << 28)) return false;
  auto* mm = const_cast<sk_model*>(md);
  model_layer_transpose(ctx, mm, k);
  return double(y->nnz) * double(mm->wT_maxdeg[k]) < double(1u << 31);
}

// Layer k on the tiny ESC kernel launched before the input's entry count is
// known on the host (it is read from *d_nnz on the device), its input the
// entries (in_row, in_col, in_val) in any order (K7's scratch, before the
// gather): the output has the kernel's full capacity; d_cnt[0] receives its
// entry count and d_cnt[1] 1 when the kernel handled the layer (0: too many
// inputs or products -- nothing was written, the host takes the layer its
// usual way).  Every bias of layer k <= 0.
sk_csr* esc_tiny_deferred(sk_ctx* ctx, const sk_model* md, uint32_t k, uint32_t n,
                          const uint32_t* in_row, const uint32_t* in_col, const float* in_val,
                          const uint32_t* d_nnz, float clip, uint32_t* d_cnt) {
  auto* mm = const_cast<sk_model*>(md);
  const sk_csr* wt = model_layer_transpose(ctx, mm, k);
  const uint32_t m = wt->cols;
  sk_csr* out = new_csr(ctx, m, n, kSmallCap);
  uint32_t* orow = aalloc<uint32_t>(ctx, kSmallCap);
  SK_LAUNCH(k_esc_tiny, 1, kSmallThreads, 0, ctx->stream, nullptr, 0u, in_col, in_val, 0u, n,
            wt->rp, wt->ci, wt->v, m, md->bias + size_t(k) * md->neurons, clip, out->ci,
            out->v, d_cnt, d_nnz, d_cnt + 1, orow, in_row);
  // (a layer the kernel left to the host has count 0 here: rp is rewritten then)
  SK_LAUNCH(k_esc_fill_rp, grid_of(ctx, uint64_t(m) + 1), 256, 0, ctx->stream, orow, d_cnt, m,
            out->rp);
  return out;
}

bool esc_tiny_possible(const sk_model* md, uint32_t k, const sk_csr* y) {
  return md->bias_nonpos[k] && y->rows >= 1 &&
         double(md->neurons) * double(y->cols) < 9.0e15;  // (i n + j) << 11 in 64 bits
}

sk_csr* esc_layer(sk_ctx* ctx, const sk_model* md, const sk_csr* y, uint32_t k, float clip) {
  auto* mm = const_cast<sk_model*>(md);
  const sk_csr* wt = model_layer_transpose(ctx, mm, k);
  const float* bias = md->bias + size_t(k) * md->neurons;
  const uint32_t maxdeg = mm->wT_maxdeg[k];
  return uint64_t(md->neurons) * y->cols <= 0xFFFFFFFFull
             ? esc_run<uint32_t>(ctx, y, wt, bias, clip, maxdeg)
             : esc_run<uint64_t>(ctx, y, wt, bias, clip, maxdeg);
}

}  // namespace sk
