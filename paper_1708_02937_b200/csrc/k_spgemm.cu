// K3: windowed row-merge SpGEMM  C = A . B  (A m-by-l CSR, B l-by-n CSR), the
// engine behind mxm(CsrMatrix, CsrMatrix) (proj/src/matrix.cpp:452-521) and
// behind the sparse-activation forward pass (BASELINE cfg3-5), where A = W_ref
// (row i = in-edges of output neuron i) and B = Y_k neuron-major.
//
// Layout.  B carries a "window table" wp[k*nW + w] = offset of the first entry
// of row k whose column (sample) is >= w*S, for S = 2^sh samples per window;
// wp[l*nW] = nnz.  A window of row k is then the contiguous slice
// [wp[k*nW+w], wp[k*nW+w+1]).  The output of one layer is produced directly in
// this layout (its window table is the scan of per-(row,window) counts), so
// layers chain with no re-indexing.  Row pointers are wp[k*nW].
//
// Work item = (output row i, window w), one warp.  The warp owns a dense
// S-float accumulator in shared memory (initialised to a sentinel bit pattern
// that no FADD can produce, so "touched" is tracked without extra state) and
// per-128-sample dirty bytes.  The in-edges of row i are taken 32 at a time in
// ascending k; their window slices are flattened (warp scan + shuffle binary
// search) so all 32 lanes stay busy.  Within one step two lanes can hit the
// same sample only if they come from different in-edges; __match_any_sync
// detects that and the step is then applied lane by lane in lane order, i.e.
// ascending k.  Hence every output is a left fold in ascending k, exactly the
// reference's order -- bitwise, with no atomics on values.
//
// Epilogue (layer mode): z = acc + b_i; ReLU select; optional clip; keep z!=0.
// Untouched positions see z = epilogue(0 + b_i); a row whose value is nonzero
// there (b_i > 0 or NaN) is emitted densely, as the dense reference would.
// Generic mode keeps every touched position (the reference never prunes mxm
// results, matrix.cpp:449-451).
//
// Output placement: each item bump-allocates its span in a scratch buffer
// (one atomic per item with output), records (count, offset); a scan of the
// counts gives the output window table and a gather writes the final CSR
// order.  Capacity overflow is flagged on device and handled by the host.
#include <cub/cub.cuh>

#include <algorithm>

#include "sk_common.cuh"

namespace sk {

constexpr uint32_t kSent = 0xFFFFFFFFu;  // never produced by FADD (canonical NaN is 0x7fffffff)
constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

struct WinArgs {
  const uint32_t* arp;
  const uint32_t* aci;
  const float* av;
  const uint32_t* bci;
  const float* bv;
  const uint32_t* wp;  // B window table, l*nW+1
  uint32_t m, l, n, nW;
  int sh;
  const float* bias;
  float clip;
  uint32_t* item_cnt;
  unsigned long long* item_off;
  uint32_t* sc_c;
  float* sc_v;
  unsigned long long* bump;
  unsigned long long cap;
  int* overflow;
  int* err;
  int skip_if_empty;  // layer mode with all biases <= 0: empty input -> empty output
};

template <typename Ops, bool kLayer>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_spgemm_win(WinArgs p) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t S = 1u << p.sh;
  uint32_t* acc = sm + size_t(wid) * S;
  uint8_t* dirty = reinterpret_cast<uint8_t*>(sm + size_t(kWarpsPerBlock) * S) + wid * (S >> 7);
  const uint64_t items = uint64_t(p.m) * p.nW;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;

  if (kLayer && p.skip_if_empty && p.wp[size_t(p.l) * p.nW] == 0) {
    for (uint64_t it = gw * 32 + lane; it < items; it += nwarps * 32) p.item_cnt[it] = 0;
    return;
  }
  for (uint32_t t = lane; t < S; t += 32) acc[t] = kSent;
  for (uint32_t t = lane; t < (S >> 7); t += 32) dirty[t] = 0;
  __syncwarp();

  for (uint64_t it = gw; it < items; it += nwarps) {
    const uint32_t i = uint32_t(it / p.nW), w = uint32_t(it % p.nW);
    const uint32_t wbase = w << p.sh;
    const uint32_t wlen = min(S, p.n - wbase);
    const uint32_t eb = p.arp[i], ee = p.arp[i + 1];
    bool any = false;
    for (uint32_t e0 = eb; e0 < ee; e0 += 32) {
      const uint32_t e = e0 + lane;
      const bool valid = e < ee;
      uint32_t beg = 0, cnt = 0;
      float a = 0.0f;
      if (valid) {
        const uint32_t k = p.aci[e];
        a = p.av[e];
        const uint32_t* wk = p.wp + size_t(k) * p.nW + w;
        beg = wk[0];
        cnt = wk[1] - beg;
      }
      const uint32_t incl = warp_incl_scan(cnt, lane);
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (total == 0) continue;
      any = true;
      const uint32_t excl = incl - cnt;
      for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t idx = base + lane;
        const bool act = idx < total;
        int L = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, L + s - 1);
          if (v <= idx) L += s;
        }
        const uint32_t begL = __shfl_sync(0xffffffffu, beg, L);
        const uint32_t exclL = __shfl_sync(0xffffffffu, excl, L);
        const float aL = __shfl_sync(0xffffffffu, a, L);
        uint32_t s_loc = 0;
        float prod = 0.0f;
        if (act) {
          const uint32_t q = begL + (idx - exclL);
          s_loc = p.bci[q] - wbase;
          prod = Ops::mul(aL, p.bv[q], p.err);
        }
        const uint32_t key = act ? s_loc : (0x80000000u | uint32_t(lane));
        const uint32_t mm = __match_any_sync(0xffffffffu, key);
        const bool conflict = __any_sync(0xffffffffu, act && __popc(mm) > 1);
        if (!conflict) {
          if (act) {
            const uint32_t x = acc[s_loc];
            const float xf = (x == kSent) ? Ops::zero() : __uint_as_float(x);
            acc[s_loc] = __float_as_uint(Ops::add(xf, prod, p.err));
            dirty[s_loc >> 7] = 1;
          }
        } else {
          // Serialise in lane order (= ascending k within this step).
          for (int b = 0; b < 32; ++b) {
            const uint32_t sb = __shfl_sync(0xffffffffu, s_loc, b);
            const float pb = __shfl_sync(0xffffffffu, prod, b);
            const bool ab = __shfl_sync(0xffffffffu, act ? 1 : 0, b) != 0;
            if (lane == 0 && ab) {
              const uint32_t x = acc[sb];
              const float xf = (x == kSent) ? Ops::zero() : __uint_as_float(x);
              acc[sb] = __float_as_uint(Ops::add(xf, pb, p.err));
              dirty[sb >> 7] = 1;
            }
            __syncwarp();
          }
        }
        __syncwarp();
      }
    }

    // ---- epilogue --------------------------------------------------------------
    float b = 0.0f, zu = 0.0f;
    bool dense_row = false;
    if (kLayer) {
      b = p.bias[i];
      zu = layer_epilogue(0.0f, b, p.clip);
      dense_row = zu != 0.0f;
    }
    if (!any && !dense_row) {
      if (lane == 0) p.item_cnt[it] = 0;
      continue;
    }
    const uint32_t nch = (wlen + 127) >> 7;
    uint32_t mine = 0;
    for (uint32_t c = 0; c < nch; ++c) {
      if (!dirty[c] && !dense_row) continue;
      const uint32_t s0 = c * 128 + lane * 4;
      const uint4 x4 = *reinterpret_cast<const uint4*>(acc + s0);
      const uint32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t s = s0 + t;
        const bool touched = xs[t] != kSent;
        bool keep;
        if (kLayer) {
          const float z = touched ? layer_epilogue(__uint_as_float(xs[t]), b, p.clip) : zu;
          keep = (touched || dense_row) && z != 0.0f;
        } else {
          keep = touched;
        }
        mine += (s < wlen && keep) ? 1u : 0u;
      }
    }
    uint32_t tot = mine;
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    unsigned long long off = 0;
    if (lane == 0) {
      if (tot) {
        off = atomicAdd(p.bump, (unsigned long long)tot);
        if (off + tot > p.cap) atomicExch(p.overflow, 1);
      }
      p.item_cnt[it] = tot;
      p.item_off[it] = off;
    }
    off = __shfl_sync(0xffffffffu, off, 0);
    const bool can_write = tot && (off + tot <= p.cap);
    unsigned long long pos = off;
    for (uint32_t c = 0; c < nch; ++c) {
      if (!dirty[c] && !dense_row) continue;
      const uint32_t s0 = c * 128 + lane * 4;
      uint4* slot = reinterpret_cast<uint4*>(acc + s0);
      const uint4 x4 = *slot;
      const uint32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
      float zs[4];
      uint32_t keepm = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t s = s0 + t;
        const bool touched = xs[t] != kSent;
        bool keep;
        if (kLayer) {
          zs[t] = touched ? layer_epilogue(__uint_as_float(xs[t]), b, p.clip) : zu;
          keep = (touched || dense_row) && zs[t] != 0.0f;
        } else {
          zs[t] = __uint_as_float(xs[t]);
          keep = touched;
        }
        if (s < wlen && keep) keepm |= 1u << t;
      }
      const uint32_t kc = __popc(keepm);
      const uint32_t incl = warp_incl_scan(kc, lane);
      const uint32_t ctot = __shfl_sync(0xffffffffu, incl, 31);
      if (can_write) {
        unsigned long long q = pos + (incl - kc);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (keepm & (1u << t)) {
            p.sc_c[q] = wbase + s0 + t;
            p.sc_v[q] = zs[t];
            ++q;
          }
      }
      pos += ctot;
      *slot = make_uint4(kSent, kSent, kSent, kSent);
      __syncwarp();
      if (lane == 0) dirty[c] = 0;
      __syncwarp();
    }
  }
}

// Copy each item's span from scratch to its final CSR position.
__global__ void k_gather_items(const uint32_t* __restrict__ item_cnt,
                               const unsigned long long* __restrict__ item_off,
                               const uint32_t* __restrict__ wp_out, uint64_t items,
                               const uint32_t* __restrict__ sc_c, const float* __restrict__ sc_v,
                               uint32_t* __restrict__ oc, float* __restrict__ ov,
                               const int* overflow) {
  if (*overflow || wp_out[items] == 0) return;
  const int lane = threadIdx.x & 31;
  for (uint64_t it = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items;
       it += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t c = item_cnt[it];
    if (!c) continue;
    const unsigned long long src = item_off[it];
    const uint32_t dst = wp_out[it];
    for (uint32_t t = lane; t < c; t += 32) {
      oc[size_t(dst) + t] = sc_c[src + t];
      ov[size_t(dst) + t] = sc_v[src + t];
    }
  }
}

// Window table of a plain CSR: wp[k*nW+w] = rp[k] + lower_bound(row k, w*S).
__global__ void k_build_wp(const uint32_t* rp, const uint32_t* ci, uint32_t rows, uint32_t nW,
                           int sh, uint32_t* wp) {
  const uint64_t n = uint64_t(rows) * nW;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t <= n;
       t += uint64_t(gridDim.x) * blockDim.x) {
    if (t == n) {
      wp[n] = rows ? rp[rows] : 0;
      continue;
    }
    const uint32_t k = uint32_t(t / nW), w = uint32_t(t % nW);
    uint32_t lo = rp[k], hi = rp[k + 1];
    const uint32_t target = w << sh;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (ci[mid] < target) lo = mid + 1; else hi = mid;
    }
    wp[t] = lo;
  }
}

__global__ void k_rp_from_wp(const uint32_t* wp, uint32_t rows, uint32_t nW, uint32_t* rp) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
       i += gridDim.x * blockDim.x)
    rp[i] = wp[size_t(i) * nW];
}

// Upper bound on the products of A.B restricted by rows: sum_i sum_{k in A_i} nnz(B_k).
__global__ void k_count_products(const uint32_t* arp, const uint32_t* aci, uint32_t m,
                                 const uint32_t* brp, unsigned long long* total) {
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    for (uint32_t e = arp[i]; e < arp[i + 1]; ++e) c += brp[aci[e] + 1] - brp[aci[e]];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

// ---- host side -------------------------------------------------------------------

struct WinGeom {
  int sh;
  uint32_t S, nW;
};

static WinGeom geometry(uint32_t n) {
  // 2048-sample windows (8 KB per warp) by default; small batches use one window.
  int sh = 11;
  while (sh > 7 && (1u << (sh - 1)) >= n) --sh;
  WinGeom g;
  g.sh = sh;
  g.S = 1u << sh;
  g.nW = std::max<uint32_t>(1, (n + g.S - 1) >> sh);
  return g;
}

static size_t win_smem(const WinGeom& g) {
  return size_t(kWarpsPerBlock) * g.S * 4 + size_t(kWarpsPerBlock) * (g.S >> 7);
}

template <typename Ops, bool kLayer>
static void launch_win(sk_ctx* ctx, const WinArgs& a, const WinGeom& g) {
  const size_t smem = win_smem(g);
  static bool configured = false;  // per template instance
  if (!configured) {
    SK_CUDA(cudaFuncSetAttribute(k_spgemm_win<Ops, kLayer>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  int per_sm = 0;
  SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spgemm_win<Ops, kLayer>,
                                                        kWarpsPerBlock * 32, smem));
  const uint64_t items = uint64_t(a.m) * a.nW;
  const uint64_t want = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const unsigned grid =
      unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(ctx->num_sms) * std::max(per_sm, 1))));
  SK_LAUNCH((k_spgemm_win<Ops, kLayer>), grid, kWarpsPerBlock * 32, smem, ctx->stream, a);
}

static unsigned grid_warps(sk_ctx* ctx, uint64_t warps) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, uint64_t(ctx->num_sms) * 16)));
}

static uint32_t* build_wp(sk_ctx* ctx, const sk_csr* b, const WinGeom& g) {
  const uint64_t n = uint64_t(b->rows) * g.nW;
  uint32_t* wp = dalloc<uint32_t>(ctx, n + 1);
  SK_LAUNCH(k_build_wp, unsigned(std::min<uint64_t>((n + 256) / 256, uint64_t(ctx->num_sms) * 16)),
            256, 0, ctx->stream, b->rp, b->ci, b->rows, g.nW, g.sh, wp);
  return wp;
}

// One SpGEMM pass.  Returns false on scratch overflow (needed size in *need).
struct PassBuffers {
  uint32_t* item_cnt = nullptr;           // items+1
  unsigned long long* item_off = nullptr; // items
  uint32_t* sc_c = nullptr;
  float* sc_v = nullptr;
  unsigned long long cap = 0;
};

static void run_pass(sk_ctx* ctx, sk_semiring s, bool layer, const sk_csr* a,
                     const uint32_t* bci, const float* bv, const uint32_t* wp_b, uint32_t l,
                     uint32_t n, const WinGeom& g, const float* bias, float clip,
                     bool skip_if_empty, PassBuffers& pb, uint32_t* wp_out, uint32_t* oc,
                     float* ov, unsigned long long* bump, int* overflow) {
  WinArgs p;
  p.arp = a->rp;
  p.aci = a->ci;
  p.av = a->v;
  p.bci = bci;
  p.bv = bv;
  p.wp = wp_b;
  p.m = a->rows;
  p.l = l;
  p.n = n;
  p.nW = g.nW;
  p.sh = g.sh;
  p.bias = bias;
  p.clip = clip;
  p.item_cnt = pb.item_cnt;
  p.item_off = pb.item_off;
  p.sc_c = pb.sc_c;
  p.sc_v = pb.sc_v;
  p.bump = bump;
  p.cap = pb.cap;
  p.overflow = overflow;
  p.err = ctx->d_err;
  p.skip_if_empty = skip_if_empty ? 1 : 0;
  const uint64_t items = uint64_t(a->rows) * g.nW;
  SK_CUDA(cudaMemsetAsync(bump, 0, sizeof(unsigned long long), ctx->stream));
  timing_mark(ctx);
  if (layer) {
    launch_win<OpArith, true>(ctx, p, g);
  } else {
    dispatch_semiring(s, [&](auto ops) { launch_win<decltype(ops), false>(ctx, p, g); });
  }
  timing_mark(ctx);
  SK_CUDA(cudaMemsetAsync(pb.item_cnt + items, 0, 4, ctx->stream));
  exclusive_scan_u32(ctx, pb.item_cnt, wp_out, items + 1);
  SK_LAUNCH(k_gather_items, grid_warps(ctx, items), 256, 0, ctx->stream, pb.item_cnt,
            pb.item_off, wp_out, items, pb.sc_c, pb.sc_v, oc, ov, overflow);
}

sk_csr* mxm_csr_csr_impl(sk_ctx* ctx, const sk_csr* a, const sk_csr* b, sk_semiring s) {
  const uint32_t m = a->rows, n = b->cols;
  if (m == 0 || n == 0 || a->nnz == 0 || b->nnz == 0) {
    sk_csr* o = new_csr(ctx, m, n, 0);
    SK_CUDA(cudaMemsetAsync(o->rp, 0, (size_t(m) + 1) * 4, ctx->stream));
    return o;
  }
  const WinGeom g = geometry(n);
  uint32_t* wp_b = build_wp(ctx, b, g);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->d_u64);
  SK_CUDA(cudaMemsetAsync(d, 0, 16, ctx->stream));
  SK_LAUNCH(k_count_products, grid_warps(ctx, m), 256, 0, ctx->stream, a->rp, a->ci, m, b->rp, d);
  unsigned long long prods = 0;
  SK_CUDA(cudaMemcpyAsync(&prods, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  const unsigned long long cap = std::min<unsigned long long>(prods, uint64_t(m) * n);
  if (cap > 0xFFFFFFFFull) fail(SK_ERR_INVALID_ARGUMENT, "mxm result nnz exceeds the 32-bit index range");
  const uint64_t items = uint64_t(m) * g.nW;
  PassBuffers pb;
  pb.cap = cap;
  pb.item_cnt = dalloc<uint32_t>(ctx, items + 1);
  pb.item_off = reinterpret_cast<unsigned long long*>(dalloc<uint64_t>(ctx, items));
  pb.sc_c = dalloc<uint32_t>(ctx, cap);
  pb.sc_v = dalloc<float>(ctx, cap);
  uint32_t* wp_out = dalloc<uint32_t>(ctx, items + 1);
  uint32_t* oc = dalloc<uint32_t>(ctx, cap);
  float* ov = dalloc<float>(ctx, cap);
  int* overflow = reinterpret_cast<int*>(d + 1);
  run_pass(ctx, s, false, a, b->ci, b->v, wp_b, b->rows, n, g, nullptr, 0.0f, false, pb, wp_out,
           oc, ov, d, overflow);
  uint32_t nnz = 0;
  SK_CUDA(cudaMemcpyAsync(&nnz, wp_out + items, 4, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  sk_csr* o = new sk_csr;
  o->ctx = ctx;
  o->rows = m;
  o->cols = n;
  o->nnz = nnz;
  o->rp = dalloc<uint32_t>(ctx, size_t(m) + 1);
  o->ci = oc;
  o->v = ov;
  SK_LAUNCH(k_rp_from_wp, grid_warps(ctx, m + 1), 256, 0, ctx->stream, wp_out, m, g.nW, o->rp);
  dfree(ctx, wp_b);
  dfree(ctx, wp_out);
  dfree(ctx, pb.item_cnt);
  dfree(ctx, pb.item_off);
  dfree(ctx, pb.sc_c);
  dfree(ctx, pb.sc_v);
  return o;
}

// ---- the sparse-activation forward pass -----------------------------------------

sk_csr* sparse_forward_impl(sk_ctx* ctx, const sk_model* md, const sk_csr* y0, float clip,
                            uint64_t* nnz_trace) {
  const uint32_t m = md->neurons, n = y0->cols, L = md->layers;
  const WinGeom g = geometry(n);
  const uint64_t items = uint64_t(m) * g.nW;
  const uint64_t full = uint64_t(m) * n;

  size_t free_b = 0, total_b = 0;
  SK_CUDA(cudaMemGetInfo(&free_b, &total_b));
  // three entry buffers (two ping-pong activations + scratch), 8 B per entry
  const unsigned long long mem_cap = (unsigned long long)(free_b * 0.6 / 24.0);
  auto clamp_cap = [&](unsigned long long c) {
    c = std::min<unsigned long long>(c, full);
    c = std::min<unsigned long long>(c, mem_cap);
    c = std::min<unsigned long long>(c, 0xFFFFFFFFull);
    return std::max<unsigned long long>(c, 1);
  };
  unsigned long long cap = clamp_cap(std::max<unsigned long long>(4ull * y0->nnz, 1ull << 24));

  uint32_t* wp0 = build_wp(ctx, y0, g);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->d_u64);
  int* overflow = reinterpret_cast<int*>(d + 1);
  uint32_t* trace_d = dalloc<uint32_t>(ctx, size_t(L) + 1);
  SK_CUDA(cudaMemcpyAsync(trace_d, wp0 + items, 4, cudaMemcpyDeviceToDevice, ctx->stream));

  for (int attempt = 0; attempt < 2; ++attempt) {
    SK_CUDA(cudaMemsetAsync(overflow, 0, 4, ctx->stream));
    PassBuffers pb;
    pb.cap = cap;
    pb.item_cnt = dalloc<uint32_t>(ctx, items + 1);
    pb.item_off = reinterpret_cast<unsigned long long*>(dalloc<uint64_t>(ctx, items));
    pb.sc_c = dalloc<uint32_t>(ctx, cap);
    pb.sc_v = dalloc<float>(ctx, cap);
    uint32_t* wp_buf[2] = {dalloc<uint32_t>(ctx, items + 1), dalloc<uint32_t>(ctx, items + 1)};
    uint32_t* c_buf[2] = {dalloc<uint32_t>(ctx, cap), dalloc<uint32_t>(ctx, cap)};
    float* v_buf[2] = {dalloc<float>(ctx, cap), dalloc<float>(ctx, cap)};

    const uint32_t* in_c = y0->ci;
    const float* in_v = y0->v;
    const uint32_t* in_wp = wp0;
    int cur = 0;
    for (uint32_t k = 0; k < L; ++k) {
      run_pass(ctx, SK_ARITHMETIC, true, md->w[k], in_c, in_v, in_wp, m, n, g,
               md->bias + size_t(k) * m, clip, md->bias_nonpos[k] != 0, pb, wp_buf[cur],
               c_buf[cur], v_buf[cur], d, overflow);
      SK_CUDA(cudaMemcpyAsync(trace_d + k + 1, wp_buf[cur] + items, 4, cudaMemcpyDeviceToDevice,
                              ctx->stream));
      in_c = c_buf[cur];
      in_v = v_buf[cur];
      in_wp = wp_buf[cur];
      cur ^= 1;
    }
    int ov = 0;
    std::vector<uint32_t> trace(size_t(L) + 1);
    SK_CUDA(cudaMemcpyAsync(&ov, overflow, 4, cudaMemcpyDeviceToHost, ctx->stream));
    SK_CUDA(cudaMemcpyAsync(trace.data(), trace_d, trace.size() * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
    sync(ctx);
    const int last = cur ^ 1;
    if (!ov) {
      const uint32_t nnz = trace[L];
      sk_csr* o = new sk_csr;
      o->ctx = ctx;
      o->rows = m;
      o->cols = n;
      o->nnz = nnz;
      o->rp = dalloc<uint32_t>(ctx, size_t(m) + 1);
      o->ci = dalloc<uint32_t>(ctx, nnz);
      o->v = dalloc<float>(ctx, nnz);
      SK_LAUNCH(k_rp_from_wp, grid_warps(ctx, m + 1), 256, 0, ctx->stream, wp_buf[last], m, g.nW,
                o->rp);
      if (nnz) {
        SK_CUDA(cudaMemcpyAsync(o->ci, c_buf[last], size_t(nnz) * 4, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        SK_CUDA(cudaMemcpyAsync(o->v, v_buf[last], size_t(nnz) * 4, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      }
      if (nnz_trace)
        for (uint32_t k = 0; k <= L; ++k) nnz_trace[k] = trace[k];
      for (int q = 0; q < 2; ++q) {
        dfree(ctx, wp_buf[q]);
        dfree(ctx, c_buf[q]);
        dfree(ctx, v_buf[q]);
      }
      dfree(ctx, pb.item_cnt);
      dfree(ctx, pb.item_off);
      dfree(ctx, pb.sc_c);
      dfree(ctx, pb.sc_v);
      dfree(ctx, wp0);
      dfree(ctx, trace_d);
      return o;
    }
    for (int q = 0; q < 2; ++q) {
      dfree(ctx, wp_buf[q]);
      dfree(ctx, c_buf[q]);
      dfree(ctx, v_buf[q]);
    }
    dfree(ctx, pb.item_cnt);
    dfree(ctx, pb.item_off);
    dfree(ctx, pb.sc_c);
    dfree(ctx, pb.sc_v);
    // Retry once with the largest capacity memory allows.
    const unsigned long long bigger = clamp_cap(full);
    if (bigger <= cap) break;
    cap = bigger;
  }
  dfree(ctx, wp0);
  dfree(ctx, trace_d);
  fail(SK_ERR_OOM, "sparse forward: activation nnz exceeds the device capacity");
}

}  // namespace sk
