// K6: the order-free exact layer pushed from the input side (sample-major).
//
// When the host proves a layer exact (products_exact: every partial sum of
// W.Y is an exact fp32 value, so any accumulation order gives the ascending
// fold's result bit for bit -- proj/src/matrix.cpp:452-521), every product is
// the same constant v = w y (constant-valued weights, binary activations: the
// Graph-Challenge construction of BASELINE cfg3/cfg4), and every bias is <= 0
// (untouched positions give epilogue(0 + b) = 0), the layer reduces to counting:
//
//     z_ij = epilogue(c_ij v + b_i),  c_ij = |{k in in(i) : y_kj != 0}|,
//
// and an output survives iff c_ij v > -b_i.  Organised by SAMPLE, the count
// needs no gathered index loads at all: for sample j every active input neuron
// k adds 1 to the counter of each of its out-neurons (W^T row k, one coalesced
// 128-byte line per 32 out-edges) -- one shared-memory atomic per product.
//
//  * Y^T (sample-major lists of active neurons) comes from a counting
//    transpose of the neuron-major input: column counts, a scan, a scatter
//    (list order is free: the count is order-independent).
//  * A persistent CTA holds 8-bit counters for all m out-neurons (m/4 words) in
//    shared memory and takes samples one at a time; warps take the sample's
//    active neurons, lanes their out-edges.  An increment that brings a counter
//    to cmin (the smallest count any row's threshold admits) appends a
//    candidate; after the sample, candidates are evaluated against their own
//    row's threshold with the final count, survivors are appended (key i n + j,
//    value z), and the counters are cleared with vector stores.
//  * Survivors are sorted by key (CUB radix sort) into the output CSR.
#include <cub/cub.cuh>

#include "sk_common.cuh"

namespace sk {

namespace push {
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kCand = 1024;  // candidates per sample before the full sweep
constexpr int kU = 16;            // active neurons (slots) in flight per warp
}  // namespace push

struct PushArgs {
  const uint32_t* yt_rp;  // n + 1
  const uint32_t* yt_k;   // active neurons per sample
  const uint32_t* wt_rp;  // W^T row pointers (m_in + 1)
  const uint32_t* wt_ci;  // out-neurons
  const float* bias;      // m
  float clip, v;
  uint32_t m, n, cmin, words;
  unsigned long long* nout;  // survivors appended
  unsigned long long cap;
  unsigned long long* okey;
  uint32_t* oval;
};

// ---- Y^T: counting transpose of a neuron-major CSR (values not needed) --------------

__global__ void k_t_count(const uint32_t* __restrict__ ci, size_t nnz, uint32_t* __restrict__ cnt) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += size_t(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[ci[e]], 1u);
}

__global__ void k_t_scatter(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                            uint32_t rows, uint32_t* __restrict__ cursor,
                            uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < rows;
       k += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t e = rp[k] + lane; e < rp[k + 1]; e += 32) out[atomicAdd(&cursor[ci[e]], 1u)] = k;
}

// ---- the push kernel ----------------------------------------------------------------
//
// Samples are assigned statically (CTA c: c, c + G, ...), so the next sample is
// known: while the warps apply sample j's increments, every thread also loads
// one active neuron of sample j+1 and its W^T bounds, and stores them into the
// other half of a double-buffered slot table at the end -- the dependent chain
// (list entry -> W^T row pointers -> out-neurons -> atomic) costs one round
// trip per sample instead of three.
__global__ void __launch_bounds__(push::kThreads, 2) k_push_layer(PushArgs p) {
  using namespace push;
  extern __shared__ __align__(16) uint32_t cnt[];  // p.words (a multiple of 4)
  __shared__ uint2 slot[2][kThreads];              // (W^T row start, out-degree)
  __shared__ uint32_t s_nslot[2];
  __shared__ uint32_t cand[kCand];
  __shared__ uint32_t s_ncand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t t = tid * 4; t < p.words; t += kThreads * 4)
    *reinterpret_cast<uint4*>(cnt + t) = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) s_ncand = 0;
  // slots of a sample: thread t takes active neurons t, t + kThreads, ... (a
  // sample with more than kThreads active neurons runs in several rounds)
  auto fill = [&](uint32_t j, uint32_t round, int buf) {
    uint2 v = make_uint2(0u, 0u);
    uint32_t total = 0;
    if (j < p.n) {
      const uint32_t e0 = p.yt_rp[j], e1 = p.yt_rp[j + 1];
      const uint32_t e = e0 + round * kThreads + tid;
      total = e1 - e0;
      if (e < e1) {
        const uint32_t k = p.yt_k[e];
        const uint32_t b = p.wt_rp[k];
        v = make_uint2(b, p.wt_rp[k + 1] - b);
      }
    }
    slot[buf][tid] = v;
    if (tid == 0) s_nslot[buf] = total;
  };
  uint32_t j = blockIdx.x;
  fill(j, 0, 0);
  __syncthreads();
  int cur = 0;
  for (; j < p.n; j += gridDim.x) {
    const uint32_t total = s_nslot[cur];
    for (uint32_t round = 0; round * kThreads < total; ++round) {
      const uint32_t ns = min(uint32_t(kThreads), total - round * kThreads);
      // prefetch: the next round of this sample, or the next sample's first round
      const bool more = (round + 1) * kThreads < total;
      const uint32_t pj = more ? j : j + gridDim.x;
      const uint32_t pr = more ? round + 1 : 0;
      uint2 pv = make_uint2(0u, 0u);
      uint32_t ptotal = 0;
      if (pj < p.n) {
        const uint32_t e0 = p.yt_rp[pj], e1 = p.yt_rp[pj + 1];
        const uint32_t e = e0 + pr * kThreads + tid;
        ptotal = e1 - e0;
        if (e < e1) {
          const uint32_t k = p.yt_k[e];
          pv.x = p.wt_rp[k];
          pv.y = p.wt_rp[k + 1] - pv.x;
        }
      }
      // ---- increments: warp w takes slots w, w + kWarps, ... kU at a time
      for (uint32_t s0 = warp; s0 < ns; s0 += kWarps * kU) {
        uint32_t i0[kU], i1[kU];
        bool wide = false;  // some slot has more than 64 out-edges (rare)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t sl = s0 + u * kWarps;
          const uint2 bd = sl < ns ? slot[cur][sl] : make_uint2(0u, 0u);
          wide |= bd.y > 64;
          i0[u] = lane < bd.y ? p.wt_ci[bd.x + lane] : 0xFFFFFFFFu;
          i1[u] = lane + 32 < bd.y ? p.wt_ci[bd.x + 32 + lane] : 0xFFFFFFFFu;
        }
        auto inc = [&](uint32_t i) {
          if (i == 0xFFFFFFFFu) return;
          const uint32_t sh = (i & 3u) * 8u;
          const uint32_t old = atomicAdd(cnt + (i >> 2), 1u << sh);
          if (((old >> sh) & 0xFFu) + 1u == p.cmin) {
            const uint32_t q = atomicAdd(&s_ncand, 1u);
            if (q < kCand) cand[q] = i;
          }
        };
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          inc(i0[u]);
          inc(i1[u]);
        }
        if (wide) {  // warp-uniform
          for (int u = 0; u < kU; ++u) {
            const uint32_t sl = s0 + u * kWarps;
            const uint2 bd = sl < ns ? slot[cur][sl] : make_uint2(0u, 0u);
            for (uint32_t c = 64; c < bd.y; c += 32)
              inc(c + lane < bd.y ? p.wt_ci[bd.x + c + lane] : 0xFFFFFFFFu);
          }
        }
      }
      __syncthreads();
      if (!more) {
        // ---- candidates: the final count against the row's own threshold
        const uint32_t nc = s_ncand;
        auto emit = [&](uint32_t i, uint32_t c) {
          const float x = __fmul_rn(float(c), p.v);  // exact (products_exact)
          const float z = layer_epilogue(x, p.bias[i], p.clip);
          if (z != 0.0f) {
            const unsigned long long pos = atomicAdd(p.nout, 1ull);
            if (pos < p.cap) {
              p.okey[pos] = (unsigned long long)i * p.n + j;
              p.oval[pos] = __float_as_uint(z);
            }
          }
        };
        if (nc <= kCand) {
          for (uint32_t t = tid; t < nc; t += kThreads) {
            const uint32_t i = cand[t];
            emit(i, (cnt[i >> 2] >> ((i & 3u) * 8u)) & 0xFFu);
          }
        } else {  // more candidates than the list holds: sweep every counter
          for (uint32_t t = tid; t < p.m; t += kThreads) {
            const uint32_t c = (cnt[t >> 2] >> ((t & 3u) * 8u)) & 0xFFu;
            if (c >= p.cmin) emit(t, c);
          }
        }
        __syncthreads();
        for (uint32_t t = tid * 4; t < p.words; t += kThreads * 4)
          *reinterpret_cast<uint4*>(cnt + t) = make_uint4(0u, 0u, 0u, 0u);
        if (tid == 0) s_ncand = 0;
      }
      // publish the prefetched slots (the other buffer; nobody reads it now)
      slot[cur ^ 1][tid] = pv;
      if (tid == 0) s_nslot[cur ^ 1] = ptotal;
      __syncthreads();
      cur ^= 1;
    }
    if (total == 0) {  // an empty sample: still advance the prefetch chain
      const uint32_t pj = j + gridDim.x;
      fill(pj, 0, cur ^ 1);
      __syncthreads();
      cur ^= 1;
    }
  }
}

// ---- survivors -> CSR ---------------------------------------------------------------

__global__ void k_push_csr(const unsigned long long* __restrict__ key,
                           const uint32_t* __restrict__ val, size_t cnt, uint32_t n,
                           uint32_t* __restrict__ rows_cnt, uint32_t* __restrict__ ci,
                           float* __restrict__ v) {
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < cnt;
       q += size_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[q];
    const uint32_t i = uint32_t(k / n);
    ci[q] = uint32_t(k - (unsigned long long)i * n);
    v[q] = __uint_as_float(val[q]);
    atomicAdd(&rows_cnt[i], 1u);
  }
}

static unsigned grid_for_n(sk_ctx* ctx, size_t n) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 16)));
}

// Shared memory for the counters of m out-neurons (8-bit fields).
size_t push_smem(uint32_t m) { return size_t((m + 15) / 16) * 16; }

// Y (m_in x n, neuron-major, binary) -> output CSR (m x n) of one layer, or
// nullptr when the counters do not fit.  v = the constant product w y (> 0),
// cmin = the smallest count any row's threshold admits, wT = W^T (m_in rows).
sk_csr* push_layer(sk_ctx* ctx, const sk_csr* wT, const sk_csr* y, uint32_t m, const float* bias,
                   float clip, float v, uint32_t cmin) {
  const uint32_t n = y->cols, min_ = y->rows;
  const size_t smem = push_smem(m);
  if (smem > 160 * 1024) return nullptr;
  arena_begin(ctx);
  struct Scope {
    sk_ctx* c;
    ~Scope() { arena_end(c); }
  } scope{ctx};
  // Y^T by counting transpose
  uint32_t* yt_rp = aalloc<uint32_t>(ctx, size_t(n) + 1);
  uint32_t* cur = aalloc<uint32_t>(ctx, size_t(n) + 1);
  uint32_t* yt_k = aalloc<uint32_t>(ctx, y->nnz);
  SK_CUDA(cudaMemsetAsync(cur, 0, (size_t(n) + 1) * 4, ctx->stream));
  if (y->nnz) SK_LAUNCH(k_t_count, grid_for_n(ctx, y->nnz), 256, 0, ctx->stream, y->ci, y->nnz, cur);
  exclusive_scan_u32(ctx, cur, yt_rp, size_t(n) + 1);
  SK_CUDA(cudaMemcpyAsync(cur, yt_rp, size_t(n) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (y->nnz)
    SK_LAUNCH(k_t_scatter, grid_for_n(ctx, size_t(min_) * 32), 256, 0, ctx->stream, y->rp, y->ci,
              min_, cur, yt_k);
  // survivors: a first capacity, one retry with the exact count
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(ctx->d_u64);
  unsigned long long cap = std::max<unsigned long long>(1u << 16, y->nnz / 4);
  smem_attr(ctx, k_push_layer, int(smem));
  const int per_sm = occupancy(ctx, k_push_layer, push::kThreads, smem);
  const unsigned grid = unsigned(std::min<uint64_t>(n, uint64_t(ctx->num_sms) * std::max(1, per_sm)));
  for (int attempt = 0; attempt < 2; ++attempt) {
    unsigned long long* okey = aalloc<unsigned long long>(ctx, cap);
    uint32_t* oval = aalloc<uint32_t>(ctx, cap);
    SK_CUDA(cudaMemsetAsync(ctr, 0, 16, ctx->stream));
    PushArgs a;
    a.yt_rp = yt_rp;
    a.yt_k = yt_k;
    a.wt_rp = wT->rp;
    a.wt_ci = wT->ci;
    a.bias = bias;
    a.clip = clip;
    a.v = v;
    a.m = m;
    a.n = n;
    a.cmin = cmin;
    a.words = uint32_t(smem / 4);
    a.nout = ctr + 1;
    a.cap = cap;
    a.okey = okey;
    a.oval = oval;
    timing_mark(ctx, SK_KT_PUSH);
    SK_LAUNCH(k_push_layer, grid, push::kThreads, smem, ctx->stream, a);
    timing_mark(ctx);
    unsigned long long* h = reinterpret_cast<unsigned long long*>(ctx->h_u64);
    SK_CUDA(cudaMemcpyAsync(h, ctr + 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const unsigned long long cnt = h[0];
    if (cnt > cap) {
      cap = cnt;
      continue;
    }
    // sort the survivors by key (row-major output order)
    unsigned long long* k2 = aalloc<unsigned long long>(ctx, std::max<unsigned long long>(cnt, 1));
    uint32_t* v2 = aalloc<uint32_t>(ctx, std::max<unsigned long long>(cnt, 1));
    if (cnt) {
      int end_bit = 1;
      while (end_bit < 64 && (1ull << end_bit) < (unsigned long long)m * n) ++end_bit;
      size_t tmp = 0;
      SK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, okey, k2, oval, v2, cnt, 0, end_bit,
                                              ctx->stream));
      void* t = aalloc<char>(ctx, tmp);
      SK_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, okey, k2, oval, v2, cnt, 0, end_bit,
                                              ctx->stream));
      g_launches.fetch_add(1);
    }
    sk_csr* o = new_csr(ctx, m, n, cnt);
    uint32_t* rc = aalloc<uint32_t>(ctx, size_t(m) + 1);
    SK_CUDA(cudaMemsetAsync(rc, 0, (size_t(m) + 1) * 4, ctx->stream));
    if (cnt) SK_LAUNCH(k_push_csr, grid_for_n(ctx, cnt), 256, 0, ctx->stream, k2, v2, cnt, n, rc, o->ci, o->v);
    exclusive_scan_u32(ctx, rc, o->rp, size_t(m) + 1);
    return o;
  }
  fail(SK_ERR, "push layer: survivor count changed between attempts");
}

}  // namespace sk
