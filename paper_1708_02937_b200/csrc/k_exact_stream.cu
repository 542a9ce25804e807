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
//  * Per pass: emit the survivors -- each candidate evaluated with the row's own
//    threshold and epilogue -- into a scratch span (one item per (row, pass):
//    count and offset, scanned and gathered by the host code as for
//    k_exact_layer; per-window items would write m * n / 1024 counts, 62 MB on
//    cfg5, almost all zero), then
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
constexpr uint32_t kNone = 0xFFFFFFFFu;
// pass-table values: entry position (bits 0-29) + two flags (stream_table_flags)
constexpr uint32_t kPos = 0x3FFFFFFFu, kHeadF = 0x80000000u, kTailF = 0x40000000u;

#ifndef SK_K7_RC6
#define SK_K7_RC6 384
#endif
// accumulator (2^fl words of 32 / fb fields) + candidate bitmap (a bit per
// sample of the pass) + 2 x unit records.  A batch of records is a whole number
// of steps (32 ku units): a batch ending inside a step would leave the step's
// other lanes idle.
__host__ __device__ constexpr uint32_t pass_samples(int fl, int fb) { return (32u / fb) << fl; }
__host__ __device__ constexpr uint32_t rec_cap(int fl, int fb, int ku) {
  return pass_samples(fl, fb) <= 4096 ? (ku == 6 ? 960u : 1024u)
                                      : (ku == 6 ? uint32_t(SK_K7_RC6) : 512u);
}
__host__ __device__ constexpr size_t warp_bytes(int fl, int fb, int ku) {
  return (size_t(4) << fl) + pass_samples(fl, fb) / 8 + size_t(8) * rec_cap(fl, fb, ku);
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

// FB: bits per field (8, or 4 when the offset threshold and the increment are
// small: twice the samples per accumulator byte; a field that wraps is detected
// -- its top bit goes from set to clear -- and the host reruns the layer with
// 8-bit fields)
// KU: 16-byte units per lane and step (4 for long passes, 6 for short ones)
template <int FL, int NS, int FB, int kU>
__global__ void __launch_bounds__(32 * kSW) k_exact_stream(StreamArgs p) {
  extern __shared__ __align__(16) uint8_t smraw[];
  constexpr uint32_t Wd = 1u << FL;                 // accumulator words
  constexpr uint32_t SP = pass_samples(FL, FB);     // samples per pass
  constexpr uint32_t NWP = SP >> 10;                // output windows per pass
  constexpr uint32_t RC = rec_cap(FL, FB, kU);
  constexpr int LB = FB == 8 ? 3 : 2;               // log2(FB)
  constexpr uint32_t TOP = FB == 8 ? 0x80808080u : 0x88888888u;  // field top bits
  constexpr uint32_t FMASK = (1u << FB) - 1u;
  constexpr uint32_t STEP = 32 * kU; // units per step
  const int lane = threadIdx.x & 31;
  uint32_t* const acc =
      reinterpret_cast<uint32_t*>(smraw + (threadIdx.x >> 5) * warp_bytes(FL, FB, kU));
  uint32_t* const cand = acc + Wd;          // SP bits
  uint32_t* const recs = cand + SP / 32;    // two buffers of RC unit records
  const uint32_t acc_s = async::smem_u32(acc);

  const uint32_t cw = p.clearw;
  for (uint32_t t = lane * 4; t < Wd; t += 128)
    *reinterpret_cast<uint4*>(acc + t) = make_uint4(cw, cw, cw, cw);
  for (uint32_t t = lane; t < SP / 32; t += 32) cand[t] = 0u;
  __syncwarp();

  const uint32_t nP = p.nP, q = p.q, m = p.m;
  const uint4* const bq = reinterpret_cast<const uint4*>(p.bci);

  // A record per 16-byte unit of a pass's slices, laid end to end: the unit's
  // index relative to bci (signed: the side units may lie below it).  Lane c
  // owns in-edges c, c + 32, ... (in-degree <= 32 NS, host-checked) and writes
  // the records of their slices that fall into the batch [b0, b0 + RC) of the
  // flattened units.  A slice whose first (last) unit is its row's first (last)
  // unit and holds another row's entries (the table value's head / tail flag)
  // reads the row's side unit there instead: the same unit with every entry
  // outside the row replaced by a sentinel (launch_pass_table).
  auto units = [](uint32_t b, uint32_t e) {
    b &= kPos;
    e &= kPos;
    return e > b ? ((e + 3) >> 2) - (b >> 2) : 0u;
  };
  const uint32_t side = p.side;
  auto write_recs = [&](uint32_t* rec, const uint32_t (&kk)[NS], const uint32_t (&bg)[NS],
                        const uint32_t (&en)[NS], uint32_t pre, uint32_t b0) {
#pragma unroll
    for (int q2 = 0; q2 < NS; ++q2) {
      const uint32_t nu = units(bg[q2], en[q2]);
      const uint32_t lo = max(pre, b0), hi = min(pre + nu, b0 + RC);
      uint32_t u = ((bg[q2] & kPos) >> 2) + (lo - pre);
      for (uint32_t t = lo; t < hi; ++t, ++u) rec[t - b0] = u;
      if (nu) {
        if ((bg[q2] & kHeadF) && pre >= b0 && pre < b0 + RC) rec[pre - b0] = side + 2 * kk[q2];
        const uint32_t last = pre + nu - 1;
        if ((en[q2] & kTailF) && last >= b0 && last < b0 + RC)
          rec[last - b0] = side + 2 * kk[q2] + 1;
      }
      pre += nu;
    }
  };
  // Units [base, n) of a batch, kU per lane (records base + lane, + 32, ...)
  auto load = [&](const uint32_t* rec, uint32_t base, uint32_t n, uint4 (&x)[kU]) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t t = base + 32 * u + lane;
      x[u] = t < n ? __ldg(bq + int32_t(rec[t])) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  // Every entry of a loaded unit: its sample is inside this pass exactly when
  // it is one of the slice's entries (the rest are the row's own entries of
  // other passes or sentinels), and the increment's shift runs past 31 --
  // a zero increment -- for every other one.  cr collects bits newly set, wr
  // bits cleared (masked to the fields' top bits by the caller: a top bit set is
  // a field passing the smallest threshold, a top bit cleared a field wrapping).
  auto apply = [&](uint32_t base, uint32_t n, const uint4 (&x)[kU], uint32_t pbase,
                   uint32_t& cr, uint32_t& wr) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (base + 32 * u + lane >= n) continue;
      const uint32_t v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t delta = shl_clamp(q, ((v[j] - pbase) >> (FL - LB)) & ~(FB - 1u));
        const uint32_t old = atoms_add(acc_s + ((v[j] & (Wd - 1)) << 2), delta);
        const uint32_t sum = old + delta;
        cr |= sum & ~old;
        if (FB == 4) wr |= old & ~sum;
      }
    }
  };
  // the candidates among a step's units (rare): every entry of the pass whose
  // field is past the smallest threshold is marked (re-marking is idempotent)
  auto mark = [&](uint32_t base, uint32_t n, const uint4 (&x)[kU], uint32_t pbase,
                  uint32_t& cflag) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (base + 32 * u + lane >= n) continue;
      const uint32_t v[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t sl = v[j] - pbase;
        if (sl >= SP) continue;
        if (((acc[v[j] & (Wd - 1)] >> (FB * (sl >> FL))) & FMASK) > (FMASK >> 1)) {
          atomicOr(cand + (sl >> 5), 1u << (sl & 31));
          cflag |= 1u << (sl >> 10);
        }
      }
    }
  };
  // the per-lane slice geometry of a unit (row, pass): prefix and total units
  auto geometry = [&](const uint32_t (&bg)[NS], const uint32_t (&en)[NS], uint32_t& pre,
                      uint32_t& T) {
    uint32_t nu = 0;
#pragma unroll
    for (int q2 = 0; q2 < NS; ++q2) nu += units(bg[q2], en[q2]);
    const uint32_t incl = incl_scan(nu, lane);
    T = __shfl_sync(0xffffffffu, incl, 31);
    pre = incl - nu;
  };
  // this lane's in-edges of a row (kNone: none) and their first pass bounds
  auto row_edges = [&](uint32_t eb, uint32_t ee, uint32_t (&kk)[NS]) {
#pragma unroll
    for (int q2 = 0; q2 < NS; ++q2) {
      const uint32_t e = eb + 32 * q2 + lane;
      kk[q2] = e < ee ? __ldg(p.aci + e) : kNone;
    }
  };
  auto first_bounds = [&](const uint32_t (&kk)[NS], uint32_t (&bg)[NS], uint32_t (&en)[NS],
                          uint32_t (&ea)[NS]) {
#pragma unroll
    for (int q2 = 0; q2 < NS; ++q2) {
      bg[q2] = en[q2] = ea[q2] = 0;
      if (kk[q2] != kNone) {
        const uint32_t* wk = p.wpc + size_t(kk[q2]) * nP;
        bg[q2] = __ldg(wk);
        en[q2] = __ldg(wk + 1);
        if (nP > 1) ea[q2] = __ldg(wk + 2);
      }
    }
  };

  // ---- the step pipeline: (row, pass) units in order, each a sequence of steps
  // of <= STEP units; the next step's loads (the next unit's records first when
  // the unit ends) are issued before the current step is applied, and the row
  // after the current one is claimed and its in-edges and first pass bounds
  // fetched in stages over the current row's passes.
  uint32_t c_row = 0;
  if (lane == 0) c_row = uint32_t(atomicAdd(p.work, 1ull));
  c_row = __shfl_sync(0xffffffffu, c_row, 0);
  if (c_row >= m) return;
  // this lane's in-edges, their slices of the current pass, the ends of the next
  uint32_t k[NS], c_beg[NS], c_end[NS], eA[NS];
  row_edges(__ldg(p.arp + c_row), __ldg(p.arp + c_row + 1), k);
  first_bounds(k, c_beg, c_end, eA);
  uint32_t c_pass = 0, cb = 0, c_pre, c_T;
  geometry(c_beg, c_end, c_pre, c_T);
  write_recs(recs, k, c_beg, c_end, c_pre, 0);
  __syncwarp();
  uint4 xc[kU];
  load(recs, 0, min(RC, c_T), xc);
  uint32_t s_b0 = 0, s_base = 0;  // the current step within the current unit
  uint32_t cflag = 0;             // windows of the current unit holding candidates (this lane)
  // next-row prefetch state (stages 0..4 over the current row's passes)
  uint32_t st = 0, n_row = kNone, n_eb = 0, n_ee = 0;
  uint32_t n_k[NS], n_b[NS], n_e[NS], n_e2[NS];
#pragma unroll
  for (int q2 = 0; q2 < NS; ++q2) n_k[q2] = kNone, n_b[q2] = n_e[q2] = n_e2[q2] = 0;
  auto stage = [&] {
    if (st == 0) {
      if (lane == 0) n_row = uint32_t(atomicAdd(p.work, 1ull));
    } else if (st == 1) {
      n_row = __shfl_sync(0xffffffffu, n_row, 0);
      if (n_row < m) {
        n_eb = __ldg(p.arp + n_row);
        n_ee = __ldg(p.arp + n_row + 1);
      }
    } else if (st == 2) {
      if (n_row < m) {
        row_edges(n_eb, n_ee, n_k);
      } else {
#pragma unroll
        for (int q2 = 0; q2 < NS; ++q2) n_k[q2] = kNone;
      }
    } else if (st == 3) {
      first_bounds(n_k, n_b, n_e, n_e2);
    }
    if (st < 4) ++st;
  };

#pragma unroll 1
  for (;;) {
    const uint32_t c_pbase = c_pass * SP;
    const uint32_t s_n = min(RC, c_T - min(c_T, s_b0));  // units in the current batch
    // ---- the next step --------------------------------------------------------------
    uint32_t n_b0 = s_b0, n_base = s_base + STEP;
    if (n_base >= s_n) {
      n_base = 0;
      n_b0 = s_b0 + RC;
    }
    const bool same_unit = n_b0 < c_T;
    bool more = true;
    uint32_t x_row = 0, x_pass = 0, x_pre = 0, x_T = 0;
    uint32_t x_beg[NS], x_end[NS], x_eA[NS], x_k[NS];
    uint4 xn[kU];
    if (same_unit) {
      uint32_t* const rec = recs + cb * RC;
      if (n_b0 != s_b0) {  // the unit's next batch of records (this step's units are loaded)
        __syncwarp();
        write_recs(rec, k, c_beg, c_end, c_pre, n_b0);
        __syncwarp();
      }
      load(rec, n_base, min(RC, c_T - n_b0), xn);
    } else {
      if (c_pass + 1 < nP) {
        x_row = c_row;
        x_pass = c_pass + 1;
#pragma unroll
        for (int q2 = 0; q2 < NS; ++q2) {
          x_k[q2] = k[q2];
          x_beg[q2] = c_end[q2];
          x_end[q2] = eA[q2];
          x_eA[q2] = k[q2] != kNone && x_pass + 1 < nP
                         ? __ldg(p.wpc + size_t(k[q2]) * nP + x_pass + 2) : 0u;
        }
      } else {
        while (st < 4) stage();
        x_row = n_row;
        x_pass = 0;
#pragma unroll
        for (int q2 = 0; q2 < NS; ++q2) {
          x_k[q2] = n_k[q2];
          x_beg[q2] = n_b[q2];
          x_end[q2] = n_e[q2];
          x_eA[q2] = n_e2[q2];
        }
        more = n_row < m;
      }
      if (more) {
        geometry(x_beg, x_end, x_pre, x_T);
        write_recs(recs + (cb ^ 1) * RC, x_k, x_beg, x_end, x_pre, 0);
        __syncwarp();
        load(recs + (cb ^ 1) * RC, 0, min(RC, x_T), xn);
      }
      stage();
    }

    // ---- apply the current step -------------------------------------------------------
    {
      uint32_t cr = 0, wr = 0;
      apply(s_base, s_n, xc, c_pbase, cr, wr);
      if (cr & TOP) mark(s_base, s_n, xc, c_pbase, cflag);
      if (FB == 4 && (wr & TOP)) atomicExch(p.wrap, 1);
    }
    if (same_unit) {
      s_b0 = n_b0;
      s_base = n_base;
#pragma unroll
      for (int u = 0; u < kU; ++u) xc[u] = xn[u];
      continue;
    }
    __syncwarp();
    uint32_t* const rec = recs + cb * RC;

    // ---- emit the pass: one item per (row, pass) ------------------------------------
    // Candidates of the windows that hold any are evaluated with the row's own
    // threshold and epilogue (keep masks replace the candidate words); one
    // reservation per pass; survivors are written window by window, lane by
    // lane: sample order.
    const uint64_t it = uint64_t(c_row) * nP + c_pass;
    uint32_t cmask = __reduce_or_sync(0xffffffffu, cflag);
    if (!cmask) {
      if (lane == 0) p.item_cnt[it] = 0u;
    } else {
      const float b = __ldg(p.bias + c_row);
      const float thr = __fmul_rn(-b, p.fx_scale);
      uint32_t tot = 0;
#pragma unroll 1
      for (uint32_t cm = cmask; cm; cm &= cm - 1) {
        const uint32_t slw = (__ffs(cm) - 1) * 1024 + lane * 32;  // this lane's 32 samples
        const uint32_t fs = FB * (slw >> FL);
        const uint32_t* const aw = acc + (slw & (Wd - 1));
        uint32_t keep = 0;
        for (uint32_t tt = cand[slw >> 5]; tt; tt &= tt - 1) {
          const uint32_t bt = __ffs(tt) - 1;
          const int ai = int(((aw[bt] >> fs) & FMASK) - p.foff);
          if (__int2float_rn(ai) > thr) {
            const float x = __fmul_rn(__int2float_rn(ai), p.fx_unscale);
            if (layer_epilogue(x, b, p.clip) != 0.0f) keep |= 1u << bt;
          }
        }
        cand[slw >> 5] = keep;
        tot += __reduce_add_sync(0xffffffffu, __popc(keep));
      }
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
      const bool can = tot && off + tot <= p.cap;
#pragma unroll 1
      for (uint32_t cm = cmask; cm; cm &= cm - 1) {
        const uint32_t slw = (__ffs(cm) - 1) * 1024 + lane * 32;
        const uint32_t fs = FB * (slw >> FL);
        const uint32_t* const aw = acc + (slw & (Wd - 1));
        uint32_t keep = cand[slw >> 5];
        cand[slw >> 5] = 0u;
        const uint32_t mine = __popc(keep);
        const uint32_t incl = incl_scan(mine, lane);
        unsigned long long pos = off + (incl - mine);
        off += __shfl_sync(0xffffffffu, incl, 31);
        if (can) {
          for (; keep; keep &= keep - 1) {
            const uint32_t bt = __ffs(keep) - 1;
            const int ai = int(((aw[bt] >> fs) & FMASK) - p.foff);
            const float x = __fmul_rn(__int2float_rn(ai), p.fx_unscale);
            p.sc_c[pos] = c_pbase + slw + bt;
            p.sc_v[pos] = layer_epilogue(x, b, p.clip);
            if (p.sc_r && pos < 512) p.sc_r[pos] = c_row;
            ++pos;
          }
        }
      }
    }
    __syncwarp();
    cflag = 0;
    // ---- clear the accumulator ----------------------------------------------------
    if (c_T) {
      if (c_T <= RC && c_T * 20 < Wd) {
        // sparse pass, its records in place: clear only the words its units
        // touched (every word of a loaded unit -- the row's other entries and
        // sentinels too -- is either touched or already clear)
#pragma unroll 1
        for (uint32_t t = lane; t < c_T; t += 32) {
          const uint4 x = __ldg(bq + int32_t(rec[t]));
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

    // ---- rotate to the next unit ------------------------------------------------------
    if (!more) break;
    if (x_pass == 0) st = 0;  // a new row: start claiming the one after it
    c_row = x_row;
    c_pass = x_pass;
#pragma unroll
    for (int q2 = 0; q2 < NS; ++q2) {
      k[q2] = x_k[q2];
      c_beg[q2] = x_beg[q2];
      c_end[q2] = x_end[q2];
      eA[q2] = x_eA[q2];
    }
    c_pre = x_pre;
    c_T = x_T;
    cb ^= 1u;
    s_b0 = s_base = 0;
#pragma unroll
    for (int u = 0; u < kU; ++u) xc[u] = xn[u];
  }
}

// The padded copy of an activation CSR that K7 streams, and its pass table.
// Row k starts at pk = 4k + (rp[k] & ~3) (16-byte aligned, and pk + len_k <=
// p_{k+1} without a scan); the gap after each row holds sentinels (samples no
// pass contains, low bits varied so their zero-increment atomics spread over
// the banks).  wpc[k*nP + j] = pk + (first entry of row k with sample >= j SP)
// - rp[k]; wpc[rows*nP] = p_rows.  Warp per row, the row's samples read once.
// kC entries per lane and chunk (32 kC per warp): 8 for long rows, 2 for short
// ones (cfg5's ~60 entries: a 256-entry chunk was ~360 instructions per row)
template <int kC>
__global__ void k_pad_passes(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             uint32_t rows, uint32_t nP, int sh, uint32_t* __restrict__ pci,
                             uint32_t* __restrict__ wpc) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  // software pipeline over the warp's rows: bounds two rows ahead, the first
  // 256 entries one row ahead, so a short row (cfg5: ~60 entries) does not wait
  // a full memory round trip per row
  auto bounds = [&](uint32_t k, uint32_t& b, uint32_t& e) {
    b = e = 0;
    if (k < rows) {
      b = __ldg(rp + k);
      e = __ldg(rp + k + 1);
    }
  };
  auto chunk = [&](uint32_t e0, uint32_t re, uint32_t (&sv)[kC]) {
#pragma unroll
    for (int u = 0; u < kC; ++u) {
      const uint32_t e = e0 + 32 * u + lane;
      sv[u] = e < re ? __ldg(ci + e) : 0xFFFFFFFFu;
    }
  };
  uint32_t rb, re, nb, ne;
  bounds(gw, rb, re);
  bounds(gw + nw, nb, ne);
  uint32_t sv[kC];
  chunk(rb, re, sv);
  const bool count = nP <= 64;
  for (uint32_t k = gw; k < rows; k += nw) {
    uint32_t nnb, nne, svn[kC];
    bounds(k + 2 * nw, nnb, nne);
    chunk(nb, ne, svn);
    const uint32_t pb = 4 * k + (rb & ~3u), pn = 4 * (k + 1) + (re & ~3u);
    uint32_t* const dst = pci + pb - rb;  // entry e of the row goes to dst[e]
    // pass table from the copied entries themselves: lane j (and j + 32) counts
    // the row's entries below j SP (<= 64 passes; more take a binary search per
    // pass -- dependent loads, the slow way on rows as short as cfg5's)
    uint32_t below0 = 0, below1 = 0;
    for (uint32_t e0 = rb; e0 < re; e0 += 32 * kC) {
      if (e0 != rb) chunk(e0, re, sv);
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const uint32_t e = e0 + 32 * u + lane;
        if (e < re) dst[e] = sv[u];
      }
      if (count) {
        for (uint32_t j = 1; j < nP; ++j) {
          uint32_t c = 0;
#pragma unroll
          for (int u = 0; u < kC; ++u) c += sv[u] < (j << sh) ? 1u : 0u;
          c = __reduce_add_sync(0xffffffffu, c);
          if (uint32_t(lane) == (j & 31)) (j < 32 ? below0 : below1) += c;
        }
      }
    }
    uint32_t* const out = wpc + size_t(k) * nP;
    if (count) {
      if (uint32_t(lane) < nP) out[lane] = pb + below0;
      if (uint32_t(lane) + 32 < nP) out[lane + 32] = pb + below1;
    } else {
      for (uint32_t j = lane; j < nP; j += 32) {
        const uint32_t key = j << sh;
        uint32_t lo = rb, hi = re;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (__ldg(ci + mid) < key) lo = mid + 1; else hi = mid;
        }
        out[j] = pb + (lo - rb);
      }
    }
    // the gap up to the next row (and the slack after the last row)
    const uint32_t gend = k + 1 == rows ? pn + 8 : pn;
    for (uint32_t t = pb + (re - rb) + lane; t < gend; t += 32) pci[t] = 0xFFFFFFE0u | (t & 31u);
    rb = nb;
    re = ne;
    nb = nnb;
    ne = nne;
#pragma unroll
    for (int u = 0; u < kC; ++u) sv[u] = svn[u];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wpc[size_t(rows) * nP] = 4 * rows + (rp[rows] & ~3u);
}

// The padded copy with every pass slice in BANK ORDER (<= 8 passes).  K7 counts
// order-free, so the entries of a slice may come in any order; its lanes take
// consecutive 16-byte units of a slice, and the accumulator word of sample s is
// s mod 2^FL -- bank s mod 32.  With a slice sorted by (s + 13 k) mod 32 (k the
// row: the rotation decorrelates the slices that share a 32-unit step), the
// j-th entries of neighbouring units fall into different banks: an ATOMS.ADD
// then meets the 2-3 slices of its step, not 32 random banks
// (tools/micro/atoms_vs_red.cu: 3.6 cycles per instruction at random words,
// 1.7 conflict-free).  Warp per row: a shared-memory histogram over
// (pass, bank), its exclusive scan (also the pass table), then a counting-sort
// scatter; the order inside a bank is whatever the atomics give.
template <int kC>
__global__ void __launch_bounds__(256) k_pad_banked(const uint32_t* __restrict__ rp,
                                                    const uint32_t* __restrict__ ci,
                                                    uint32_t rows, uint32_t nP, int sh,
                                                    uint32_t* __restrict__ pci,
                                                    uint32_t* __restrict__ wpc) {
  __shared__ uint32_t hist_all[8][256];
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* const hist = hist_all[threadIdx.x >> 5];
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  auto bounds = [&](uint32_t k, uint32_t& b, uint32_t& e) {
    b = e = 0;
    if (k < rows) {
      b = __ldg(rp + k);
      e = __ldg(rp + k + 1);
    }
  };
  auto chunk = [&](uint32_t e0, uint32_t re, uint32_t (&sv)[kC]) {
#pragma unroll
    for (int u = 0; u < kC; ++u) {
      const uint32_t e = e0 + 32 * u + lane;
      sv[u] = e < re ? __ldg(ci + e) : 0xFFFFFFFFu;
    }
  };
  uint32_t rb, re, nb, ne;
  bounds(gw, rb, re);
  bounds(gw + nw, nb, ne);
  uint32_t sv[kC];
  chunk(rb, re, sv);
  for (uint32_t k = gw; k < rows; k += nw) {
    uint32_t nnb, nne, svn[kC];
    bounds(k + 2 * nw, nnb, nne);
    chunk(nb, ne, svn);  // the next row's first chunk, in flight over this row's sort
    const uint32_t pb = 4 * k + (rb & ~3u), pn = 4 * (k + 1) + (re & ~3u);
    const uint32_t rot = 13u * k;
    auto key = [&](uint32_t s) { return ((s >> sh) << 5) | ((s + rot) & 31u); };
    *reinterpret_cast<uint4*>(hist + 8 * lane) = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(hist + 8 * lane + 4) = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    const bool one = re - rb <= 32 * kC;  // the whole row is in registers
    for (uint32_t e0 = rb; e0 < re; e0 += 32 * kC) {
      if (e0 != rb) chunk(e0, re, sv);
#pragma unroll
      for (int u = 0; u < kC; ++u)
        if (e0 + 32 * u + lane < re) atomicAdd(hist + key(sv[u]), 1u);
    }
    __syncwarp();
    // exclusive scan of the 256 counters: 8 consecutive per lane (4 lanes per pass)
    uint32_t c[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = hist[8 * lane + j];
      tot += c[j];
    }
    uint32_t run = incl_scan(tot, int(lane)) - tot;
    if ((lane & 3u) == 0 && (lane >> 2) < nP) wpc[size_t(k) * nP + (lane >> 2)] = pb + run;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hist[8 * lane + j] = run;
      run += c[j];
    }
    __syncwarp();
    uint32_t* const dst = pci + pb;
    for (uint32_t e0 = rb; e0 < re; e0 += 32 * kC) {
      if (!one) chunk(e0, re, sv);
#pragma unroll
      for (int u = 0; u < kC; ++u)
        if (e0 + 32 * u + lane < re) dst[atomicAdd(hist + key(sv[u]), 1u)] = sv[u];
    }
    __syncwarp();
    const uint32_t gend = k + 1 == rows ? pn + 8 : pn;
    for (uint32_t t = pb + (re - rb) + lane; t < gend; t += 32) pci[t] = 0xFFFFFFE0u | (t & 31u);
    rb = nb;
    re = ne;
    nb = nnb;
    ne = nne;
#pragma unroll
    for (int u = 0; u < kC; ++u) sv[u] = svn[u];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wpc[size_t(rows) * nP] = 4 * rows + (rp[rows] & ~3u);
}

// The padded copy for short rows (mean <= 96 entries, <= 64 passes): a warp
// takes 32 consecutive rows (their row pointers in one coalesced load), then
// kB rows at a time with all their first 64 entries loaded before any is
// stored -- the per-row latency chain of a warp-per-row walk (cfg5's 262144
// rows of ~60 entries: 100 us) becomes kB rows per memory round trip.  The pass
// table from ballots over the loaded entries; longer rows continue in 32-entry
// chunks.  Same output as k_pad_passes.
__global__ void k_pad_rows(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                           uint32_t rows, uint32_t nP, int sh, uint32_t* __restrict__ pci,
                           uint32_t* __restrict__ wpc) {
  constexpr int kB = 4;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k0 = gw * 32; k0 < rows; k0 += nw * 32) {
    const uint32_t nr = min(32u, rows - k0);
    const uint32_t rpv = __ldg(rp + k0 + min(lane, nr));
    const uint32_t rend = __ldg(rp + k0 + nr);
    for (uint32_t r0 = 0; r0 < nr; r0 += kB) {
      uint32_t rb[kB], re[kB], v[kB][2];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const uint32_t r = r0 + i;
        rb[i] = __shfl_sync(0xffffffffu, rpv, r & 31);
        const uint32_t nx = __shfl_sync(0xffffffffu, rpv, (r + 1) & 31);
        re[i] = r + 1 < nr ? nx : rend;
        if (r >= nr) re[i] = rb[i];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const uint32_t e = rb[i] + 32 * c + lane;
          v[i][c] = e < re[i] ? __ldg(ci + e) : 0xFFFFFFFFu;
        }
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const uint32_t r = r0 + i;
        if (r >= nr) break;
        const uint32_t k = k0 + r, len = re[i] - rb[i];
        const uint32_t pb = 4 * k + (rb[i] & ~3u);
        uint32_t* const dst = pci + pb;
        uint32_t mine0 = 0, mine1 = 0;  // entries below pass lane / lane + 32
        auto count = [&](uint32_t x) {
          for (uint32_t j = 1; j < nP; ++j) {
            const uint32_t c = __popc(__ballot_sync(0xffffffffu, x < (j << sh)));
            if (lane == (j & 31)) (j < 32 ? mine0 : mine1) += c;
          }
        };
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (32 * c + lane < len) dst[32 * c + lane] = v[i][c];
          count(v[i][c]);
        }
        for (uint32_t e0 = 64; e0 < len; e0 += 32) {  // long rows: the rest in chunks
          const uint32_t x = e0 + lane < len ? __ldg(ci + rb[i] + e0 + lane) : 0xFFFFFFFFu;
          if (e0 + lane < len) dst[e0 + lane] = x;
          count(x);
        }
        uint32_t* const out = wpc + size_t(k) * nP;
        if (lane < nP) out[lane] = pb + mine0;
        if (lane + 32 < nP) out[lane + 32] = pb + mine1;
        // the gap up to the next row (1..7 words; the last row: 8 more)
        const uint32_t gap = 4 - (re[i] & 3u) + (rb[i] & 3u) + (k + 1 == rows ? 8u : 0u);
        if (lane < gap) {
          const uint32_t t = pb + len + lane;
          pci[t] = 0xFFFFFFE0u | (t & 31u);
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wpc[size_t(rows) * nP] = 4 * rows + (rp[rows] & ~3u);
}

// The pass table of an activation CSR that K7 reads in place (Y's own column
// array, 16-byte units), and each row's two side units.  Thread per row; the
// row's pass boundaries by binary searches, up to kS of them interleaved (their
// dependent loads overlap): no pass over the entries themselves (the padded
// copy wrote every entry: 100 us on cfg5's 262144 short rows).
//   wpc[k*nP + j] = (first entry of row k with sample >= j SP)
//                   | kHeadF when a slice starting there has its first unit in
//                     the row's first unit and the row starts inside a unit
//                   | kTailF when a slice ending there has its last unit in the
//                     row's last unit and the row ends inside a unit
//   (j = 0: rb, both flags when rb is not a multiple of 4 -- the value also
//   ends row k - 1's last slice); wpc[rows*nP] = nnz (+ kTailF).
//   side[2k] / side[2k+1]: the row's first / last unit with every entry outside
//   the row replaced by a sentinel (a sample no pass contains, low bits varied).
__global__ void k_pass_table(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             uint32_t rows, uint32_t nP, int sh, uint32_t* __restrict__ wpc,
                             uint4* __restrict__ side) {
  constexpr int kS = 8;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < rows; k += stride) {
    const uint32_t rb = __ldg(rp + k), re = __ldg(rp + k + 1);
    auto side_unit = [&](uint32_t u) {
      uint32_t v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t e = 4 * u + j;
        v[j] = e >= rb && e < re ? __ldg(ci + e) : 0xFFFFFFE0u | ((4 * k + j) & 31u);
      }
      return make_uint4(v[0], v[1], v[2], v[3]);
    };
    const uint4 h = side_unit(rb >> 2), t = side_unit(re > rb ? (re - 1) >> 2 : rb >> 2);
    side[2 * size_t(k)] = h;
    side[2 * size_t(k) + 1] = t;
    const bool hmis = (rb & 3u) != 0, tmis = (re & 3u) != 0;
    uint32_t* const out = wpc + size_t(k) * nP;
    out[0] = rb | (hmis ? kHeadF | kTailF : 0u);
    for (uint32_t j0 = 1; j0 < nP; j0 += kS) {
      uint32_t lo[kS], hi[kS];
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        lo[s] = rb;
        hi[s] = j0 + s < nP ? re : rb;
      }
      for (bool any = true; any;) {
        any = false;
#pragma unroll
        for (int s = 0; s < kS; ++s)
          if (lo[s] < hi[s]) {
            const uint32_t mid = (lo[s] + hi[s]) >> 1;
            if (__ldg(ci + mid) < ((j0 + s) << sh)) lo[s] = mid + 1; else hi[s] = mid;
            any = true;
          }
      }
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if (j0 + s < nP) {
          const uint32_t v = lo[s];
          const bool hf = hmis && (v >> 2) == (rb >> 2);
          const bool tf = tmis && v > rb && ((v - 1) >> 2) == ((re - 1) >> 2);
          out[j0 + s] = v | (hf ? kHeadF : 0u) | (tf ? kTailF : 0u);
        }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t e = rp[rows];
    wpc[size_t(rows) * nP] = e | ((e & 3u) ? kTailF : 0u);
  }
}

}  // namespace

size_t stream_block_bytes(int fl, int fb, int ku) { return size_t(kSW) * warp_bytes(fl, fb, ku); }

int stream_block_threads() { return 32 * kSW; }

template <int NS, int FB, int KU>
static const void* stream_kernel_ns(int fl) {
  switch (fl) {
    case 8: return reinterpret_cast<const void*>(k_exact_stream<8, NS, FB, KU>);
    case 9: return reinterpret_cast<const void*>(k_exact_stream<9, NS, FB, KU>);
    case 10: return reinterpret_cast<const void*>(k_exact_stream<10, NS, FB, KU>);
    case 11: return reinterpret_cast<const void*>(k_exact_stream<11, NS, FB, KU>);
  }
  fail(SK_ERR_INVALID_ARGUMENT, "exact stream: field log2 must be 8..11");
}

template <int NS, int FB>
static const void* stream_kernel_ku(int fl, int ku) {
  return ku == 6 ? stream_kernel_ns<NS, FB, 6>(fl) : stream_kernel_ns<NS, FB, 4>(fl);
}

const void* stream_kernel(int fl, int ns, int fb, int ku) {
  if (ns < 1 || ns > 3 || (fb != 4 && fb != 8))
    fail(SK_ERR_INVALID_ARGUMENT, "exact stream: in-edge slots 1..3, fields of 4 or 8 bits");
  // in-degree <= 32 takes the two-slot kernel (its second slot stays empty)
  if (ns <= 2) return fb == 8 ? stream_kernel_ku<2, 8>(fl, ku) : stream_kernel_ku<2, 4>(fl, ku);
  return fb == 8 ? stream_kernel_ku<3, 8>(fl, ku) : stream_kernel_ku<3, 4>(fl, ku);
}

size_t padded_size(uint32_t rows, size_t nnz) { return 4 * size_t(rows) + (nnz & ~size_t(3)) + 8; }

void launch_pad_banked(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* pci, uint32_t* wpc, bool short_rows) {
  if (nP > 8) fail(SK_ERR_INVALID_ARGUMENT, "bank-ordered padded copy: at most 8 passes");
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t(rows) + 7) / 8, uint64_t(ctx->num_sms) * 8)));
  if (short_rows)
    SK_LAUNCH(k_pad_banked<2>, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
  else
    SK_LAUNCH(k_pad_banked<8>, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
}

void launch_pad_passes(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* pci, uint32_t* wpc, bool short_rows) {
  // one resident wave (8 blocks of 8 warps per SM), each warp walking rows with
  // the next row's bounds prefetched
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t(rows) + 7) / 8, uint64_t(ctx->num_sms) * 8)));
  if (short_rows && nP <= 64) {
    const unsigned rb = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t(rows) + 255) / 256, uint64_t(ctx->num_sms) * 8)));
    SK_LAUNCH(k_pad_rows, rb, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
  } else if (short_rows)
    SK_LAUNCH(k_pad_passes<2>, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
  else
    SK_LAUNCH(k_pad_passes<8>, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, pci, wpc);
}

void launch_pass_table(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* wpc, void* side) {
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t(rows) + 255) / 256, uint64_t(ctx->num_sms) * 8)));
  SK_LAUNCH(k_pass_table, blocks, 256, 0, ctx->stream, rp, ci, rows, nP, sh, wpc,
            static_cast<uint4*>(side));
}

void launch_exact_stream(sk_ctx* ctx, const StreamArgs& p, int fl, int ns, int fb, int ku,
                         unsigned grid, size_t smem) {
  const void* kern = stream_kernel(fl, ns, fb, ku);
  void* args[] = {const_cast<StreamArgs*>(&p)};
  SK_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(32 * kSW), args, smem, ctx->stream));
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace sk
