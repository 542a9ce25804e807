// K7: the order-free exact layer, one output row at a time, its in-edge slices
// streamed through registers with coalesced 16-byte loads.
//
// Same contract as k_exact_layer's specialised path (k_spgemm.cu): every product
// of the layer is the same exact fixed-point increment q, every bias <= 0, so
// an output z_is = epilogue(count_is * q * 2^gran, b_i) depends only on how
// many in-edges k of output row i have sample s in row k of Y -- the fold
// order cannot change a bit (products_exact), and the result is the reference's
// ascending fold (proj/src/matrix.cpp:452-521 + proj/src/dnn.cpp:86-103).
//
// Organisation (one warp = one persistent worker, one row at a time):
//  * A row's samples are covered in passes of SP = 4 * 2^FL samples.  The pass
//    accumulator is 2^FL words of four 8-bit fields (field f holds samples
//    [f 2^FL, (f+1) 2^FL) of the pass), each holding count * q + foff, so a
//    field's top bit turns on exactly when the count passes the smallest row
//    threshold: the update that turns it on marks a candidate.
//  * The slices [wpc[k][j], wpc[k][j+1]) of the row's in-edges k in Y's column
//    array, widened to 16-byte units, are laid end to end: lane c writes one
//    shared-memory record per unit of its in-edge's slice (unit index | mask of
//    the entries inside the slice), then lane l takes records l, l+32, ...:
//    consecutive lanes read consecutive units of mostly the same slice, so a
//    16-byte load instruction touches a few lines, not one line per lane as the
//    4-entry piece records of k_exact_layer did (~0.5 L1 tag requests per
//    product there).  Entries outside the slice take a zero increment (the
//    atomic still runs, on an arbitrary word, and changes nothing), so the
//    update loop has no per-entry branch; the next step's loads are issued
//    before the current step's atomics.
//  * Per pass: emit the windows (1024 samples, the output window table's unit)
//    holding candidates -- each candidate evaluated with the row's own
//    threshold and epilogue -- into scratch spans (item counts per (row,
//    window), scanned and gathered by the host code as for k_exact_layer), then
//    clear the accumulator: all of it, or when the pass is sparse only the words
//    its entries touched (cfg5: a full clear per pass would write m * n bytes of
//    shared memory, 15.7 GB per layer).
// Rows are handed out dynamically (the next row is claimed one row ahead); all
// passes of a row run back to back, so W streams through L2 once.
#include "sk_async.cuh"
#include "sk_common.cuh"
#include "k_exact_stream.cuh"

#include <algorithm>

namespace sk {

namespace {

constexpr int kSW = 1;  // warps per block (the accumulator base is then block-uniform)
constexpr int kU = 4;   // 16-byte units per lane and step (two steps in flight)

// accumulator (2^fl words) + candidate bitmap (4 * 2^fl bits) + unit records
__host__ __device__ constexpr uint32_t rec_cap(int fl) { return fl >= 12 ? 1024u : 512u; }
__host__ __device__ constexpr size_t warp_bytes(int fl) {
  return (size_t(4) << fl) + ((size_t(4) << fl) / 8) + size_t(4) * rec_cap(fl);
}

__device__ __forceinline__ uint32_t incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ uint32_t atoms_add(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}

// a << b with PTX semantics: shift amounts above 31 give 0
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int FL>
__global__ void __launch_bounds__(32 * kSW) k_exact_stream(StreamArgs p) {
  extern __shared__ __align__(16) uint8_t smraw[];
  constexpr uint32_t Wd = 1u << FL;  // accumulator words
  constexpr uint32_t SP = 4u << FL;  // samples per pass
  constexpr uint32_t NWP = SP >> 10; // output windows per pass
  constexpr uint32_t RC = rec_cap(FL);
  const int lane = threadIdx.x & 31;
  uint32_t* const acc =
      reinterpret_cast<uint32_t*>(smraw + (threadIdx.x >> 5) * warp_bytes(FL));
  uint32_t* const cand = acc + Wd;     // SP bits
  uint32_t* const rec = cand + SP / 32;  // RC unit records
  const uint32_t acc_s = async::smem_u32(acc);

  const uint32_t cw = p.clearw;
  for (uint32_t t = lane * 4; t < Wd; t += 128)
    *reinterpret_cast<uint4*>(acc + t) = make_uint4(cw, cw, cw, cw);
  for (uint32_t t = lane; t < SP / 32; t += 32) cand[t] = 0u;
  __syncwarp();

  const uint32_t nP = p.nP, q = p.q;
  const uint4* const bq = reinterpret_cast<const uint4*>(p.bci);

  // A record per 16-byte unit of the pass's slices, laid end to end: the unit's
  // index in the padded column array.  Lane c writes the records of in-edge c's
  // slice that fall into the batch [b0, b0 + RC) of the flattened units.
  auto write_recs = [&](uint32_t u0, uint32_t pre, uint32_t nu, uint32_t b0) {
    const uint32_t lo = max(pre, b0), hi = min(pre + nu, b0 + RC);
    uint32_t u = u0 + (lo - pre);
    for (uint32_t t = lo; t < hi; ++t, ++u) rec[t - b0] = u;
  };
  // Units [base, n) of the current batch, kU per lane and step (the next step's
  // loads are issued before this step's atomics).
  auto load = [&](uint32_t base, uint32_t n, bool (&ok)[kU], uint4 (&x)[kU]) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t t = base + 32 * u + lane;
      ok[u] = t < n;
      x[u] = ok[u] ? __ldg(bq + rec[t]) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  // Every entry of a loaded unit: its sample is inside this pass exactly when
  // it is one of the slice's entries (the rest are the row's own entries of
  // other passes or sentinels), and the increment's shift runs past 31 --
  // a zero increment -- for every other one.  cr collects top-bit transitions.
  auto apply = [&](const bool (&ok)[kU], const uint4 (&x)[kU], uint32_t pbase, uint32_t& cr) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;  // past the batch's end (last step only)
      const uint32_t v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t delta = shl_clamp(q, ((v[j] - pbase) >> (FL - 3)) & ~7u);
        const uint32_t old = atoms_add(acc_s + ((v[j] & (Wd - 1)) << 2), delta);
        cr |= (old + delta) & ~old & 0x80808080u;
      }
    }
  };
  // the candidates among a step's units (rare): every entry of the pass whose
  // field is past the smallest threshold is marked (re-marking is idempotent)
  auto mark = [&](const bool (&ok)[kU], const uint4 (&x)[kU], uint32_t pbase,
                  uint32_t& cflag) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;
      const uint32_t v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t sl = v[j] - pbase;
        if (sl >= SP) continue;
        if (((acc[v[j] & (Wd - 1)] >> (8 * (sl >> FL))) & 0xFFu) >= 0x80u) {
          atomicOr(cand + (sl >> 5), 1u << (sl & 31));
          cflag |= 1u << (sl >> 10);
        }
      }
    }
  };

  uint32_t nxt = 0;
  if (lane == 0) nxt = uint32_t(atomicAdd(p.work, 1ull));
  nxt = __shfl_sync(0xffffffffu, nxt, 0);
#pragma unroll 1
  while (nxt < p.m) {
    const uint32_t row = nxt;
    if (lane == 0) nxt = uint32_t(atomicAdd(p.work, 1ull));  // claimed one row ahead
    const uint32_t eb = __ldg(p.arp + row), ee = __ldg(p.arp + row + 1);
    const uint32_t nch = ee > eb ? (ee - eb + 31) / 32 : 1u;
    uint32_t k = 0;
    bool kok = false;
    uint32_t beg = 0, end = 0, nend = 0;
#pragma unroll 1
    for (uint32_t pass = 0; pass < nP; ++pass) {
      const uint32_t pbase = pass * SP;
      uint32_t cflag = 0, ntot = 0, T = 0;
#pragma unroll 1
      for (uint32_t ch = 0; ch < nch; ++ch) {
        // this lane's in-edge and its slice of the pass; the next pass's end is
        // prefetched (a pass starts where the previous one ended)
        if (pass == 0 || nch > 1) {
          const uint32_t e = eb + 32 * ch + lane;
          kok = e < ee;
          k = kok ? __ldg(p.aci + e) : 0u;
          beg = end = 0;
          if (kok) {
            beg = __ldg(p.wpc + size_t(k) * nP + pass);
            end = __ldg(p.wpc + size_t(k) * nP + pass + 1);
          }
        } else {
          beg = end;
          end = nend;
        }
        nend = kok && pass + 1 < nP ? __ldg(p.wpc + size_t(k) * nP + pass + 2) : 0u;
        ntot += __reduce_add_sync(0xffffffffu, end - beg);
        const uint32_t nu = end > beg ? ((end + 3) >> 2) - (beg >> 2) : 0u;
        const uint32_t incl = incl_scan(nu, lane);
        T = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t pre = incl - nu;
#pragma unroll 1
        for (uint32_t b0 = 0; b0 < T; b0 += RC) {
          __syncwarp();  // the previous batch's records are consumed
          write_recs(beg >> 2, pre, nu, b0);
          __syncwarp();
          const uint32_t n = min(RC, T - b0);
          bool ok[kU];
          uint4 x[kU];
          load(0, n, ok, x);
#pragma unroll 1
          for (uint32_t base = 0; base < n; base += 32 * kU) {
            bool okn[kU];
            uint4 xn[kU];
            const bool more = base + 32 * kU < n;
            if (more) load(base + 32 * kU, n, okn, xn);
            uint32_t cr = 0;
            apply(ok, x, pbase, cr);
            if (cr) mark(ok, x, pbase, cflag);
            if (more) {
#pragma unroll
              for (int u = 0; u < kU; ++u) {
                ok[u] = okn[u];
                x[u] = xn[u];
              }
            }
          }
        }
      }
      __syncwarp();

      // ---- emit the pass's windows --------------------------------------------------
      const uint32_t w0 = pass * NWP;
      const uint32_t nwp = min(NWP, p.nW - w0);
      uint32_t cmask = __reduce_or_sync(0xffffffffu, cflag);
      if (uint32_t(lane) < nwp && !((cmask >> lane) & 1u))
        p.item_cnt[uint64_t(row) * p.nW + w0 + lane] = 0u;
      if (cmask) {
        const float b = __ldg(p.bias + row);
        const float thr = __fmul_rn(-b, p.fx_scale);
#pragma unroll 1
        for (; cmask; cmask &= cmask - 1) {
          const uint32_t wsub = __ffs(cmask) - 1;
          const uint64_t it = uint64_t(row) * p.nW + w0 + wsub;
          const uint32_t slw = wsub * 1024 + lane * 32;  // this lane's 32 samples
          const uint32_t fs = 8 * (slw >> FL);
          const uint32_t* const aw = acc + (slw & (Wd - 1));
          const uint32_t t = cand[slw >> 5];
          uint32_t keep = 0;
          cand[slw >> 5] = 0u;
          for (uint32_t tt = t; tt; tt &= tt - 1) {
            const uint32_t bt = __ffs(tt) - 1;
            const int ai = int(((aw[bt] >> fs) & 0xFFu) - p.foff);
            if (__int2float_rn(ai) > thr) {
              const float x = __fmul_rn(__int2float_rn(ai), p.fx_unscale);
              if (layer_epilogue(x, b, p.clip) != 0.0f) keep |= 1u << bt;
            }
          }
          const uint32_t mine = __popc(keep);
          const uint32_t incl = incl_scan(mine, lane);
          const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
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
          if (tot && off + tot <= p.cap) {
            unsigned long long pos = off + (incl - mine);
            for (; keep; keep &= keep - 1) {
              const uint32_t bt = __ffs(keep) - 1;
              const int ai = int(((aw[bt] >> fs) & 0xFFu) - p.foff);
              const float x = __fmul_rn(__int2float_rn(ai), p.fx_unscale);
              p.sc_c[pos] = pbase + slw + bt;
              p.sc_v[pos] = layer_epilogue(x, b, p.clip);
              ++pos;
            }
          }
        }
      }
      __syncwarp();
      // ---- clear the accumulator ------------------------------------------------------
      if (ntot) {
        if (nch == 1 && T <= RC && ntot * 5 < Wd) {
          // sparse pass, its records all still in place: clear only the words its
          // units touched (every word of a loaded unit -- the neighbours' entries
          // too -- is either touched or already clear)
#pragma unroll 1
          for (uint32_t t = lane; t < T; t += 32) {
            const uint4 x = __ldg(bq + rec[t]);
            sts_u32(acc_s + ((x.x & (Wd - 1)) << 2), cw);
            sts_u32(acc_s + ((x.y & (Wd - 1)) << 2), cw);
            sts_u32(acc_s + ((x.z & (Wd - 1)) << 2), cw);
            sts_u32(acc_s + ((x.w & (Wd - 1)) << 2), cw);
          }
        } else {
          for (uint32_t t = lane * 4; t < Wd; t += 128)
            *reinterpret_cast<uint4*>(acc + t) = make_uint4(cw, cw, cw, cw);
        }
      }
      __syncwarp();
    }
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
  }
}


// The padded copy of an activation CSR that K7 streams, and its pass table.
// Row k starts at pk = 4k + (rp[k] & ~3) (16-byte aligned, and pk + len_k <=
// p_{k+1} without a scan); the gap after each row holds sentinels (samples no
// pass contains, low bits varied so their zero-increment atomics spread over
// the banks).  wpc[k*nP + j] = pk + (first entry of row k with sample >= j SP)
// - rp[k]; wpc[rows*nP] = p_rows.  Warp per row, the row's samples read once.
__global__ void k_pad_passes(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             uint32_t rows, uint32_t nP, int sh, uint32_t* __restrict__ pci,
                             uint32_t* __restrict__ wpc) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = gw; k < rows; k += nw) {
    const uint32_t rb = rp[k], re = rp[k + 1];
    const uint32_t pb = 4 * k + (rb & ~3u), pn = 4 * (k + 1) + (re & ~3u);
    uint32_t* const out = wpc + size_t(k) * nP;
    int carry = -1;  // pass of the entry before this chunk (-1: none)
    for (uint32_t e0 = rb; e0 < re; e0 += 128) {
      uint32_t sv[4];
      int we[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t e = e0 + 32 * u + lane;
        sv[u] = e < re ? __ldg(ci + e) : 0u;
        we[u] = e < re ? int(sv[u] >> sh) : int(nP);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t e = e0 + 32 * u + lane;
        if (e < re) pci[pb + (e - rb)] = sv[u];
        int prev = __shfl_up_sync(0xffffffffu, we[u], 1);
        if (lane == 0) prev = carry;
        if (e < re)
          for (int w = prev + 1; w <= we[u]; ++w) out[w] = pb + (e - rb);
        carry = __shfl_sync(0xffffffffu, we[u], 31);
      }
    }
    const int last = re > rb ? int(ci[re - 1] >> sh) : -1;
    for (int w = last + 1 + lane; w < int(nP); w += 32) out[w] = pb + (re - rb);
    // the gap up to the next row (and the slack after the last row)
    const uint32_t gend = k + 1 == rows ? pn + 8 : pn;
    for (uint32_t t = pb + (re - rb) + lane; t < gend; t += 32) pci[t] = 0xFFFFFFE0u | (t & 31u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wpc[size_t(rows) * nP] = 4 * rows + (rp[rows] & ~3u);
}

}  // namespace

size_t stream_warp_bytes(int fl) { return warp_bytes(fl); }

size_t stream_block_bytes(int fl) { return size_t(kSW) * stream_warp_bytes(fl); }

int stream_block_threads() { return 32 * kSW; }

const void* stream_kernel(int fl) {
  switch (fl) {
    case 10: return reinterpret_cast<const void*>(k_exact_stream<10>);
    case 11: return reinterpret_cast<const void*>(k_exact_stream<11>);
    case 12: return reinterpret_cast<const void*>(k_exact_stream<12>);
    case 13: return reinterpret_cast<const void*>(k_exact_stream<13>);
  }
  fail(SK_ERR_INVALID_ARGUMENT, "exact stream: field log2 must be 10..13");
}

size_t padded_size(uint32_t rows, size_t nnz) { return 4 * size_t(rows) + (nnz & ~size_t(3)) + 8; }

void launch_pad_passes(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* pci, uint32_t* wpc) {
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t(rows) + 7) / 8, uint64_t(ctx->num_sms) * 64)));
  SK_LAUNCH(k_pad_passes, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
}

void launch_exact_stream(sk_ctx* ctx, const StreamArgs& p, int fl, unsigned grid, size_t smem) {
  const int th = 32 * kSW;
  switch (fl) {
    case 10: SK_LAUNCH(k_exact_stream<10>, grid, th, smem, ctx->stream, p); return;
    case 11: SK_LAUNCH(k_exact_stream<11>, grid, th, smem, ctx->stream, p); return;
    case 12: SK_LAUNCH(k_exact_stream<12>, grid, th, smem, ctx->stream, p); return;
    case 13: SK_LAUNCH(k_exact_stream<13>, grid, th, smem, ctx->stream, p); return;
  }
  fail(SK_ERR_INVALID_ARGUMENT, "exact stream: field log2 must be 10..13");
}

}  // namespace sk
