// Construction, conversion, element-wise and generator kernels.
//
//  csr_from_triples  (proj/src/matrix.cpp:145-189): device range check ->
//      radix sort on (row<<32|col) (stable) -> adjacent-duplicate check ->
//      exact-zero elision -> row_ptr by lower_bound.  Errors carry the
//      reference's messages; the first offending triple is found with atomicMin
//      so the reported one is the one the reference's sequential loop reports.
//  CsrMatrix validating ctor (matrix.cpp:89-119): per-row device check.
//  to_dense / from_dense (matrix.cpp:191-227): warp per row; from_dense is
//      the ballot/popc ordered compaction ("select != 0").
//  ewise_add / ewise_mul (matrix.cpp:245-392): union semantics.
//  Generators: counter-addressed SplitMix64, bitwise equal to oracle/sk_oracle.c.
#include <cub/cub.cuh>

#include <cstring>

#include "sk_common.cuh"

namespace sk {

// ---- helpers ------------------------------------------------------------------

__global__ void k_range_check(const uint32_t* r, const uint32_t* c, size_t n,
                              uint32_t rows, uint32_t cols,
                              unsigned long long* first_bad) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    if (r[i] >= rows || c[i] >= cols) atomicMin(first_bad, (unsigned long long)i);
}

__global__ void k_make_keys(const uint32_t* r, const uint32_t* c, size_t n,
                            uint64_t* keys, uint32_t* idx) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    keys[i] = (uint64_t(r[i]) << 32) | c[i];
    idx[i] = uint32_t(i);
  }
}

__global__ void k_dup_check(const uint64_t* keys, size_t n,
                            unsigned long long* first_dup) {
  for (size_t i = 1 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    if (keys[i] == keys[i - 1]) atomicMin(first_dup, (unsigned long long)i);
}

__global__ void k_keep_flags(const uint32_t* idx, const float* v, size_t n,
                             uint32_t* flags) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    flags[i] = (v ? v[idx[i]] : 1.0f) != 0.0f ? 1u : 0u;
}

__global__ void k_scatter_kept(const uint64_t* keys, const uint32_t* idx,
                               const float* v, const uint32_t* flags,
                               const uint32_t* pos, size_t n, uint32_t* out_row,
                               uint32_t* out_col, float* out_v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    if (!flags[i]) continue;
    const uint32_t p = pos[i];
    out_row[p] = uint32_t(keys[i] >> 32);
    out_col[p] = uint32_t(keys[i]);
    out_v[p] = v[idx[i]];
  }
}

// rp[i] = lower_bound(rows_sorted, i) for i in [0, nrows]
__global__ void k_row_ptr_from_sorted(const uint32_t* rows_sorted, size_t nnz,
                                      uint32_t nrows, uint32_t* rp) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i <= nrows;
       i += size_t(gridDim.x) * blockDim.x) {
    size_t lo = 0, hi = nnz;
    while (lo < hi) {
      size_t mid = (lo + hi) >> 1;
      if (rows_sorted[mid] < i) lo = mid + 1; else hi = mid;
    }
    rp[i] = uint32_t(lo);
  }
}

static unsigned grid_for(sk_ctx* ctx, size_t n, unsigned block = 256) {
  return std::max(1u, std::min<unsigned>(ceil_div(n, block), ctx->num_sms * 16));
}

static uint64_t read_u64(sk_ctx* ctx, const void* d) {
  // through the context's pinned mirror (a pageable copy is a staged, blocking one)
  SK_CUDA(cudaMemcpyAsync(ctx->h_u64 + 2, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return ctx->h_u64[2];
}

static void set_u64(sk_ctx* ctx, void* d, uint64_t v) {
  SK_CUDA(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, ctx->stream));
}

static int end_bit_for(uint32_t rows) {
  int b = 0;
  while (b < 32 && (uint64_t(1) << b) < uint64_t(rows)) ++b;
  return 32 + b;
}

// Sorted (row,col)-keyed triples -> CSR with exact-zero elision.
static sk_csr* csr_from_sorted(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                               const uint64_t* keys, const uint32_t* idx,
                               const float* v, size_t n, bool drop_zeros) {
  uint32_t* flags = dalloc<uint32_t>(ctx, n + 1);
  uint32_t* pos = dalloc<uint32_t>(ctx, n + 1);
  SK_CUDA(cudaMemsetAsync(flags + n, 0, 4, ctx->stream));
  if (n) SK_LAUNCH(k_keep_flags, grid_for(ctx, n), 256, 0, ctx->stream, idx,
                   drop_zeros ? v : nullptr, n, flags);
  exclusive_scan_u32(ctx, flags, pos, n + 1);
  uint32_t nnz32 = 0;
  SK_CUDA(cudaMemcpyAsync(&nnz32, pos + n, 4, cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  const size_t nnz = nnz32;
  sk_csr* a = new_csr(ctx, rows, cols, nnz);
  uint32_t* srow = dalloc<uint32_t>(ctx, nnz);
  if (n) SK_LAUNCH(k_scatter_kept, grid_for(ctx, n), 256, 0, ctx->stream, keys, idx, v,
                   flags, pos, n, srow, a->ci, a->v);
  SK_LAUNCH(k_row_ptr_from_sorted, grid_for(ctx, size_t(rows) + 1), 256, 0, ctx->stream,
            srow, nnz, rows, a->rp);
  dfree(ctx, srow);
  dfree(ctx, flags);
  dfree(ctx, pos);
  return a;
}

static void sort_pairs(sk_ctx* ctx, uint64_t* kin, uint64_t* kout, uint32_t* vin,
                       uint32_t* vout, size_t n, int end_bit) {
  size_t tmp = 0;
  SK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit,
                                          ctx->stream));
  void* t = dalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, n, 0, end_bit,
                                          ctx->stream));
  g_launches.fetch_add(1);
  dfree(ctx, t);
}

sk_csr* csr_from_device_triples(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                const uint32_t* d_r, const uint32_t* d_c,
                                const float* d_v, size_t n, const uint32_t* h_r,
                                const uint32_t* h_c, uint64_t* dup_index) {
  unsigned long long* first_bad = reinterpret_cast<unsigned long long*>(ctx->d_u64);
  // 1. range (matrix.cpp:147-153)
  set_u64(ctx, first_bad, ~0ull);
  if (n) SK_LAUNCH(k_range_check, grid_for(ctx, n), 256, 0, ctx->stream, d_r, d_c, n,
                   rows, cols, first_bad);
  uint64_t bad = read_u64(ctx, first_bad);
  if (bad != ~0ull) {
    uint32_t br = 0, bc = 0;
    if (h_r) {
      br = h_r[bad];
      bc = h_c[bad];
    } else {
      SK_CUDA(cudaMemcpy(&br, d_r + bad, 4, cudaMemcpyDeviceToHost));
      SK_CUDA(cudaMemcpy(&bc, d_c + bad, 4, cudaMemcpyDeviceToHost));
    }
    fail(SK_ERR_INVALID_ARGUMENT, "triple (" + std::to_string(br) + ", " + std::to_string(bc) +
                                      ") outside " + dim_string(rows, cols));
  }
  // 2. sort by (row, col) (matrix.cpp:154-157)
  uint64_t* k0 = dalloc<uint64_t>(ctx, n);
  uint64_t* k1 = dalloc<uint64_t>(ctx, n);
  uint32_t* i0 = dalloc<uint32_t>(ctx, n);
  uint32_t* i1 = dalloc<uint32_t>(ctx, n);
  if (n) {
    SK_LAUNCH(k_make_keys, grid_for(ctx, n), 256, 0, ctx->stream, d_r, d_c, n, k0, i0);
    sort_pairs(ctx, k0, k1, i0, i1, n, end_bit_for(rows));
  }
  // 3. duplicates (matrix.cpp:158-165)
  set_u64(ctx, first_bad, ~0ull);
  if (n > 1) SK_LAUNCH(k_dup_check, grid_for(ctx, n), 256, 0, ctx->stream, k1, n, first_bad);
  bad = read_u64(ctx, first_bad);
  if (bad != ~0ull) {
    const uint64_t key = read_u64(ctx, k1 + bad);
    uint32_t orig = 0;  // input position of the later duplicate (the sort is stable)
    SK_CUDA(cudaMemcpyAsync(&orig, i1 + bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    for (void* p : {(void*)k0, (void*)k1, (void*)i0, (void*)i1}) dfree(ctx, p);
    if (dup_index) {  // caller reports it (the Matrix Market reader: by line)
      *dup_index = orig;
      return nullptr;
    }
    fail(SK_ERR_INVALID_ARGUMENT, "duplicate coordinate (" + std::to_string(key >> 32) + ", " +
                                      std::to_string(uint32_t(key)) + ")");
  }
  // 4. nnz limit (matrix.cpp:166-168)
  if (n > 0xFFFFFFFFull) {
    for (void* p : {(void*)k0, (void*)k1, (void*)i0, (void*)i1}) dfree(ctx, p);
    fail(SK_ERR_INVALID_ARGUMENT, "nnz exceeds the 32-bit index range");
  }
  // 5. zero elision + row_ptr (matrix.cpp:170-188)
  sk_csr* a = csr_from_sorted(ctx, rows, cols, k1, i1, d_v, n, true);
  for (void* p : {(void*)k0, (void*)k1, (void*)i0, (void*)i1}) dfree(ctx, p);
  return a;
}

// ---- transpose (used by the generators and the column-major views) -------------

__global__ void k_expand_keys_t(const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                                uint64_t* keys, uint32_t* idx) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * blockDim.x) >> 5) {
    for (uint32_t e = rp[r] + lane; e < rp[r + 1]; e += 32) {
      keys[e] = (uint64_t(ci[e]) << 32) | r;
      idx[e] = e;
    }
  }
}

sk_csr* csr_transpose(sk_ctx* ctx, const sk_csr* a) {
  const size_t n = a->nnz;
  uint64_t* k0 = dalloc<uint64_t>(ctx, n);
  uint64_t* k1 = dalloc<uint64_t>(ctx, n);
  uint32_t* i0 = dalloc<uint32_t>(ctx, n);
  uint32_t* i1 = dalloc<uint32_t>(ctx, n);
  SK_LAUNCH(k_expand_keys_t, grid_for(ctx, size_t(a->rows) * 32), 256, 0, ctx->stream,
            a->rp, a->ci, a->rows, k0, i0);
  if (n) sort_pairs(ctx, k0, k1, i0, i1, n, end_bit_for(a->cols));
  sk_csr* t = csr_from_sorted(ctx, a->cols, a->rows, k1, i1, a->v, n, false);
  for (void* p : {(void*)k0, (void*)k1, (void*)i0, (void*)i1}) dfree(ctx, p);
  return t;
}

// ---- validating constructor (matrix.cpp:89-119) ---------------------------------

__global__ void k_validate_rows(const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                                uint32_t cols, size_t nnz, unsigned long long* bad_row) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += gridDim.x * blockDim.x) {
    const uint32_t b = rp[i], e = rp[i + 1];
    bool bad = b > e || e > nnz;
    for (uint32_t k = b; !bad && k < e; ++k) {
      if (ci[k] >= cols) bad = true;
      else if (k > b && ci[k - 1] >= ci[k]) bad = true;
    }
    if (bad) atomicMin(bad_row, (unsigned long long)i);
  }
}

}  // namespace sk

using namespace sk;

extern "C" sk_status sk_csr_from_triples(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                         const uint32_t* row, const uint32_t* col,
                                         const float* val, size_t n, sk_csr** out) {
  return guarded([&] {
    if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
    SK_CUDA(cudaSetDevice(ctx->device));
    uint32_t* dr = dalloc<uint32_t>(ctx, n);
    uint32_t* dc = dalloc<uint32_t>(ctx, n);
    float* dv = dalloc<float>(ctx, n);
    if (n) {
      SK_CUDA(cudaMemcpyAsync(dr, row, n * 4, cudaMemcpyHostToDevice, ctx->stream));
      SK_CUDA(cudaMemcpyAsync(dc, col, n * 4, cudaMemcpyHostToDevice, ctx->stream));
      SK_CUDA(cudaMemcpyAsync(dv, val, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    }
    try {
      *out = csr_from_device_triples(ctx, rows, cols, dr, dc, dv, n, row, col);
    } catch (...) {
      dfree(ctx, dr);
      dfree(ctx, dc);
      dfree(ctx, dv);
      throw;
    }
    dfree(ctx, dr);
    dfree(ctx, dc);
    dfree(ctx, dv);
  });
}

namespace sk {
__global__ void k_fill_f32(float* p, size_t n, float x) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    p[i] = x;
}
}  // namespace sk

// Shared by sk_csr_from_parts (values from the host) and sk_csr_from_pattern
// (v == nullptr: every stored value is `fill`, written on the device).
static sk_status csr_from_host(sk_ctx* ctx, uint32_t rows, uint32_t cols, const uint32_t* rp,
                               const uint32_t* ci, const float* v, float fill, int validate,
                               sk_csr** out) {
  return guarded([&] {
    if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
    SK_CUDA(cudaSetDevice(ctx->device));
    if (validate && rp[0] != 0) fail(SK_ERR_INVALID_ARGUMENT, "row_ptr[0] must be 0");
    const size_t nnz = rp[rows];
    sk_csr* a = new_csr(ctx, rows, cols, nnz);
    SK_CUDA(cudaMemcpyAsync(a->rp, rp, (size_t(rows) + 1) * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
    if (nnz) {
      SK_CUDA(cudaMemcpyAsync(a->ci, ci, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
      if (v)
        SK_CUDA(cudaMemcpyAsync(a->v, v, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
      else
        SK_LAUNCH(k_fill_f32, grid_for(ctx, nnz), 256, 0, ctx->stream, a->v, nnz, fill);
    }
    if (!v) {
      a->stats = const_value_stats(fill, nnz);
      a->stats_valid = true;
    }
    if (validate && rows) {
      unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx->d_u64);
      set_u64(ctx, bad, ~0ull);
      SK_LAUNCH(k_validate_rows, grid_for(ctx, rows), 256, 0, ctx->stream, a->rp, a->ci, rows,
                cols, nnz, bad);
      const uint64_t r = read_u64(ctx, bad);
      if (r != ~0ull) {
        csr_release(a);
        // Reproduce the reference's message for the first offending row.
        const uint32_t i = uint32_t(r);
        if (rp[i] > rp[i + 1] || rp[i + 1] > nnz)
          fail(SK_ERR_INVALID_ARGUMENT, "row_ptr must be non-decreasing");
        for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
          if (ci[k] >= cols)
            fail(SK_ERR_INVALID_ARGUMENT, "column index " + std::to_string(ci[k]) +
                                              " out of range in row " + std::to_string(i));
          if (k > rp[i] && ci[k - 1] >= ci[k])
            fail(SK_ERR_INVALID_ARGUMENT,
                 "column indices must be strictly increasing within row " + std::to_string(i));
        }
        fail(SK_ERR_INVALID_ARGUMENT, "invalid CSR row " + std::to_string(i));
      }
    }
    sync(ctx);  // host arrays are borrowed only for the call
    *out = a;
  });
}

extern "C" sk_status sk_csr_from_parts(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                       const uint32_t* rp, const uint32_t* ci,
                                       const float* v, int validate, sk_csr** out) {
  if (!v && rp && rp[rows] != 0) {
    set_last_error("null values array");
    return SK_ERR_INVALID_ARGUMENT;
  }
  return csr_from_host(ctx, rows, cols, rp, ci, v, 0.0f, validate, out);
}

// The pattern upload on a caller stream (e.g. a copy stream), so that it
// overlaps work already queued on the context's stream; the handle carries an
// event every consumer waits on.  No validation (the caller's pattern is
// trusted, as with validate = 0).
extern "C" sk_status sk_csr_from_pattern_async(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                               const uint32_t* rp, const uint32_t* ci,
                                               float value, void* stream, sk_csr** out) {
  return guarded([&] {
    if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
    SK_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t nnz = rp[rows];
    auto* a = new sk_csr;
    a->ctx = ctx;
    a->rows = rows;
    a->cols = cols;
    a->nnz = nnz;
    void* p = nullptr;
    SK_CUDA(cudaMallocAsync(&p, (size_t(rows) + 1) * 4, s));
    a->rp = static_cast<uint32_t*>(p);
    SK_CUDA(cudaMallocAsync(&p, (nnz + kCiPad) * 4, s));
    a->ci = static_cast<uint32_t*>(p);
    SK_CUDA(cudaMallocAsync(&p, std::max<size_t>(nnz, 1) * 4, s));
    a->v = static_cast<float*>(p);
    SK_CUDA(cudaMemcpyAsync(a->rp, rp, (size_t(rows) + 1) * 4, cudaMemcpyHostToDevice, s));
    if (nnz) {
      SK_CUDA(cudaMemcpyAsync(a->ci, ci, nnz * 4, cudaMemcpyHostToDevice, s));
      SK_LAUNCH(k_fill_f32, grid_for(ctx, nnz), 256, 0, s, a->v, nnz, value);
    }
    a->stats = const_value_stats(value, nnz);
    a->stats_valid = true;
    SK_CUDA(cudaEventCreateWithFlags(&a->ready, cudaEventDisableTiming));
    SK_CUDA(cudaEventRecord(a->ready, s));
    *out = a;
  });
}

namespace sk {
// 16-bit column indices widened to the handle's 32-bit array (8 per thread-step)
__global__ void k_widen_u16(const uint16_t* __restrict__ in, size_t n, uint32_t* __restrict__ out) {
  const size_t n8 = n / 8;
  const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t nth = size_t(gridDim.x) * blockDim.x;
  for (size_t i = tid; i < n8; i += nth) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(in) + i);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint4* o = reinterpret_cast<uint4*>(out) + 2 * i;
    o[0] = make_uint4(w[0] & 0xFFFFu, w[0] >> 16, w[1] & 0xFFFFu, w[1] >> 16);
    o[1] = make_uint4(w[2] & 0xFFFFu, w[2] >> 16, w[3] & 0xFFFFu, w[3] >> 16);
  }
  for (size_t i = n8 * 8 + tid; i < n; i += nth) out[i] = in[i];
}
}  // namespace sk

extern "C" sk_status sk_csr_from_pattern16_async(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                                 const uint32_t* rp, const uint16_t* ci,
                                                 float value, void* stream, sk_csr** out) {
  return guarded([&] {
    if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
    if (cols > 65536u)
      fail(SK_ERR_INVALID_ARGUMENT, "16-bit column indices need cols <= 65536");
    SK_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t nnz = rp[rows];
    auto* a = new sk_csr;
    a->ctx = ctx;
    a->rows = rows;
    a->cols = cols;
    a->nnz = nnz;
    void* p = nullptr;
    SK_CUDA(cudaMallocAsync(&p, (size_t(rows) + 1) * 4, s));
    a->rp = static_cast<uint32_t*>(p);
    SK_CUDA(cudaMallocAsync(&p, (nnz + kCiPad) * 4, s));
    a->ci = static_cast<uint32_t*>(p);
    SK_CUDA(cudaMallocAsync(&p, std::max<size_t>(nnz, 1) * 4, s));
    a->v = static_cast<float*>(p);
    SK_CUDA(cudaMemcpyAsync(a->rp, rp, (size_t(rows) + 1) * 4, cudaMemcpyHostToDevice, s));
    if (nnz) {
      void* t = nullptr;  // the 16-bit staging copy (16-byte aligned: cudaMallocAsync)
      SK_CUDA(cudaMallocAsync(&t, nnz * 2, s));
      SK_CUDA(cudaMemcpyAsync(t, ci, nnz * 2, cudaMemcpyHostToDevice, s));
      SK_LAUNCH(k_widen_u16, grid_for(ctx, (nnz + 7) / 8), 256, 0, s,
                static_cast<const uint16_t*>(t), nnz, a->ci);
      SK_CUDA(cudaFreeAsync(t, s));
      SK_LAUNCH(k_fill_f32, grid_for(ctx, nnz), 256, 0, s, a->v, nnz, value);
    }
    a->stats = const_value_stats(value, nnz);
    a->stats_valid = true;
    SK_CUDA(cudaEventCreateWithFlags(&a->ready, cudaEventDisableTiming));
    SK_CUDA(cudaEventRecord(a->ready, s));
    *out = a;
  });
}

extern "C" sk_status sk_csr_from_pattern(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                         const uint32_t* rp, const uint32_t* ci, float value,
                                         int validate, sk_csr** out) {
  return csr_from_host(ctx, rows, cols, rp, ci, nullptr, value, validate, out);
}

// ==== to_dense / from_dense / nnz ====================================================

namespace sk {

__global__ void k_scatter_rows(const uint32_t* rp, const uint32_t* ci, const float* v,
                               uint32_t rows, uint32_t cols, float* out) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t e = rp[r] + lane; e < rp[r + 1]; e += 32)
      out[size_t(r) * cols + ci[e]] = v[e];
}

__global__ void k_count_nonzero_rows(const float* d, uint32_t rows, uint32_t cols,
                                     unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * blockDim.x) >> 5) {
    uint32_t c = 0;
    const float* row = d + size_t(r) * cols;
    for (uint32_t j = lane; j < cols; j += 32) c += row[j] != 0.0f;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[r] = c;
  }
}

__global__ void k_compact_rows(const float* d, uint32_t rows, uint32_t cols,
                               const unsigned long long* off, uint32_t* rp, uint32_t* ci,
                               float* v) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * blockDim.x) >> 5) {
    uint64_t o = off[r];
    if (lane == 0) rp[r] = uint32_t(o);
    if (r == rows - 1 && lane == 0) rp[rows] = uint32_t(off[rows]);
    const float* row = d + size_t(r) * cols;
    for (uint32_t j0 = 0; j0 < cols; j0 += 32) {
      const uint32_t j = j0 + lane;
      const float x = j < cols ? row[j] : 0.0f;
      const bool keep = x != 0.0f;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const uint32_t p = uint32_t(o) + __popc(m & ((1u << lane) - 1));
        ci[p] = j;
        v[p] = x;
      }
      o += __popc(m);
    }
  }
}

}  // namespace sk

extern "C" sk_status sk_to_dense(sk_ctx* ctx, const sk_csr* a, float ambient, sk_dense** out) {
  return guarded([&] {
    csr_ready(ctx, a);
    SK_CUDA(cudaSetDevice(ctx->device));
    sk_dense* d = new_dense(ctx, a->rows, a->cols);
    fill(ctx, d->d, d->elems(), ambient);
    if (a->rows)
      SK_LAUNCH(k_scatter_rows, grid_for(ctx, size_t(a->rows) * 32), 256, 0, ctx->stream,
                a->rp, a->ci, a->v, a->rows, a->cols, d->d);
    *out = d;
  });
}

namespace sk {

// Zero-filled dense copy of a CSR matrix into caller-owned device memory.
void csr_scatter_dense(sk_ctx* ctx, const sk_csr* a, float* out) {
  SK_CUDA(cudaMemsetAsync(out, 0, size_t(a->rows) * a->cols * 4, ctx->stream));
  if (a->rows && a->nnz)
    SK_LAUNCH(k_scatter_rows, grid_for(ctx, size_t(a->rows) * 32), 256, 0, ctx->stream, a->rp,
              a->ci, a->v, a->rows, a->cols, out);
}

sk_csr* from_dense_impl(sk_ctx* ctx, const float* d, uint32_t rows, uint32_t cols) {
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(
      dalloc<uint64_t>(ctx, size_t(rows) + 1));
  unsigned long long* off = reinterpret_cast<unsigned long long*>(
      dalloc<uint64_t>(ctx, size_t(rows) + 1));
  SK_CUDA(cudaMemsetAsync(cnt + rows, 0, 8, ctx->stream));
  if (rows)
    SK_LAUNCH(k_count_nonzero_rows, grid_for(ctx, size_t(rows) * 32), 256, 0, ctx->stream, d,
              rows, cols, cnt);
  exclusive_scan_u64(ctx, reinterpret_cast<uint64_t*>(cnt), reinterpret_cast<uint64_t*>(off),
                     size_t(rows) + 1);
  const uint64_t nnz = read_u64(ctx, off + rows);
  if (nnz > 0xFFFFFFFFull) {
    dfree(ctx, cnt);
    dfree(ctx, off);
    fail(SK_ERR_INVALID_ARGUMENT, "nnz exceeds the 32-bit index range");
  }
  sk_csr* a = new_csr(ctx, rows, cols, nnz);
  if (rows)
    SK_LAUNCH(k_compact_rows, grid_for(ctx, size_t(rows) * 32), 256, 0, ctx->stream, d, rows,
              cols, off, a->rp, a->ci, a->v);
  else
    SK_CUDA(cudaMemsetAsync(a->rp, 0, 4, ctx->stream));
  dfree(ctx, cnt);
  dfree(ctx, off);
  return a;
}
}  // namespace sk

extern "C" sk_status sk_from_dense(sk_ctx* ctx, const sk_dense* d, sk_csr** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    *out = from_dense_impl(ctx, d->d, d->rows, d->cols);
  });
}

namespace sk {
__global__ void k_count_nz(const float* d, size_t n, unsigned long long* total) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    c += d[i] != 0.0f;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}
}  // namespace sk

extern "C" sk_status sk_dense_nnz(sk_ctx* ctx, const sk_dense* d, size_t* out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    unsigned long long* t = reinterpret_cast<unsigned long long*>(ctx->d_u64);
    set_u64(ctx, t, 0);
    if (d->elems())
      SK_LAUNCH(k_count_nz, grid_for(ctx, d->elems()), 256, 0, ctx->stream, d->d, d->elems(), t);
    *out = read_u64(ctx, t);
  });
}

// ==== element-wise ===================================================================

namespace sk {

template <typename Ops, bool kMul>
__device__ __forceinline__ float combine(float a, float b, int* err) {
  return kMul ? Ops::mul(a, b, err) : Ops::add(a, b, err);
}

template <typename Ops, bool kMul>
__global__ void k_ewise_dense(const float* a, const float* b, size_t n, float* out, int* err) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = combine<Ops, kMul>(a[i], b[i], err);
}

// sparse (op) dense: every position first gets the "absent" combination...
template <typename Ops, bool kMul>
__global__ void k_ewise_mixed_base(const float* dn, size_t n, bool sparse_left, float* out,
                                   int* err) {
  const float z = Ops::zero();
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = sparse_left ? combine<Ops, kMul>(z, dn[i], err) : combine<Ops, kMul>(dn[i], z, err);
}
// ...then stored positions overwrite it (matrix.cpp:294-312).
template <typename Ops, bool kMul>
__global__ void k_ewise_mixed_stored(const uint32_t* rp, const uint32_t* ci, const float* v,
                                     uint32_t rows, uint32_t cols, const float* dn,
                                     bool sparse_left, float* out, int* err) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t e = rp[r] + lane; e < rp[r + 1]; e += 32) {
      const size_t p = size_t(r) * cols + ci[e];
      out[p] = sparse_left ? combine<Ops, kMul>(v[e], dn[p], err)
                           : combine<Ops, kMul>(dn[p], v[e], err);
    }
}

// Union merge of two CSR rows (matrix.cpp:253-290): pass 0 counts, pass 1 writes.
template <typename Ops, bool kMul>
__global__ void k_merge_rows(const uint32_t* arp, const uint32_t* aci, const float* av,
                             const uint32_t* brp, const uint32_t* bci, const float* bv,
                             uint32_t rows, uint32_t* cnt, const uint32_t* orp,
                             uint32_t* oci, float* ov, int* err) {
  const float z = Ops::zero();
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += gridDim.x * blockDim.x) {
    uint32_t p = arp[r], pe = arp[r + 1], q = brp[r], qe = brp[r + 1];
    uint32_t o = orp ? orp[r] : 0, c = 0;
    while (p < pe || q < qe) {
      uint32_t col;
      float val = 0.0f;
      if (q == qe || (p < pe && aci[p] < bci[q])) {
        col = aci[p];
        if (orp) val = combine<Ops, kMul>(av[p], z, err);
        ++p;
      } else if (p == pe || bci[q] < aci[p]) {
        col = bci[q];
        if (orp) val = combine<Ops, kMul>(z, bv[q], err);
        ++q;
      } else {
        col = aci[p];
        if (orp) val = combine<Ops, kMul>(av[p], bv[q], err);
        ++p;
        ++q;
      }
      if (orp) {
        oci[o + c] = col;
        ov[o + c] = val;
      }
      ++c;
    }
    if (!orp) cnt[r] = c;
  }
}

}  // namespace sk

static void require_same_shape(const char* op, uint32_t ar, uint32_t ac, uint32_t br,
                               uint32_t bc) {
  // matrix.cpp:32-38
  if (ar != br || ac != bc)
    fail(SK_ERR_DIMENSION, std::string(op) + ": operands " + dim_string(ar, ac) + " and " +
                               dim_string(br, bc) + " differ in shape");
}

extern "C" sk_status sk_ewise_dense(sk_ctx* ctx, int mul, const sk_dense* a,
                                    const sk_dense* b, sk_semiring s, sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    require_same_shape(mul ? "ewise_mul" : "ewise_add", a->rows, a->cols, b->rows, b->cols);
    sk_dense* o = new_dense(ctx, a->rows, a->cols);
    const size_t n = a->elems();
    dispatch_semiring(s, [&](auto ops) {
      using Ops = decltype(ops);
      if (n == 0) return;
      if (mul)
        SK_LAUNCH((k_ewise_dense<Ops, true>), grid_for(ctx, n), 256, 0, ctx->stream, a->d, b->d,
                  n, o->d, ctx->d_err);
      else
        SK_LAUNCH((k_ewise_dense<Ops, false>), grid_for(ctx, n), 256, 0, ctx->stream, a->d,
                  b->d, n, o->d, ctx->d_err);
    });
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, mul ? "ewise_mul" : "ewise_add");
      } catch (...) {
        sk_dense_free(o);
        throw;
      }
    }
    *out = o;
  });
}

extern "C" sk_status sk_ewise_mixed(sk_ctx* ctx, int mul, const sk_csr* sp, const sk_dense* dn,
                                    int sparse_left, sk_semiring s, sk_dense** out) {
  return guarded([&] {
    csr_ready(ctx, sp);
    SK_CUDA(cudaSetDevice(ctx->device));
    const char* op = mul ? "ewise_mul" : "ewise_add";
    if (sparse_left)
      require_same_shape(op, sp->rows, sp->cols, dn->rows, dn->cols);
    else
      require_same_shape(op, dn->rows, dn->cols, sp->rows, sp->cols);
    sk_dense* o = new_dense(ctx, dn->rows, dn->cols);
    const size_t n = dn->elems();
    dispatch_semiring(s, [&](auto ops) {
      using Ops = decltype(ops);
      if (n == 0) return;
      if (mul) {
        SK_LAUNCH((k_ewise_mixed_base<Ops, true>), grid_for(ctx, n), 256, 0, ctx->stream, dn->d,
                  n, sparse_left != 0, o->d, ctx->d_err);
        SK_LAUNCH((k_ewise_mixed_stored<Ops, true>), grid_for(ctx, size_t(sp->rows) * 32), 256,
                  0, ctx->stream, sp->rp, sp->ci, sp->v, sp->rows, sp->cols, dn->d,
                  sparse_left != 0, o->d, ctx->d_err);
      } else {
        SK_LAUNCH((k_ewise_mixed_base<Ops, false>), grid_for(ctx, n), 256, 0, ctx->stream,
                  dn->d, n, sparse_left != 0, o->d, ctx->d_err);
        SK_LAUNCH((k_ewise_mixed_stored<Ops, false>), grid_for(ctx, size_t(sp->rows) * 32), 256,
                  0, ctx->stream, sp->rp, sp->ci, sp->v, sp->rows, sp->cols, dn->d,
                  sparse_left != 0, o->d, ctx->d_err);
      }
    });
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, op);
      } catch (...) {
        sk_dense_free(o);
        throw;
      }
    }
    *out = o;
  });
}

extern "C" sk_status sk_ewise_csr(sk_ctx* ctx, int mul, const sk_csr* a, const sk_csr* b,
                                  sk_semiring s, sk_csr** out) {
  return guarded([&] {
    csr_ready(ctx, a);
    csr_ready(ctx, b);
    SK_CUDA(cudaSetDevice(ctx->device));
    require_same_shape(mul ? "ewise_mul" : "ewise_add", a->rows, a->cols, b->rows, b->cols);
    const uint32_t rows = a->rows;
    uint32_t* cnt = dalloc<uint32_t>(ctx, size_t(rows) + 1);
    uint32_t* rp = dalloc<uint32_t>(ctx, size_t(rows) + 1);
    SK_CUDA(cudaMemsetAsync(cnt + rows, 0, 4, ctx->stream));
    sk_csr* o = nullptr;
    dispatch_semiring(s, [&](auto ops) {
      using Ops = decltype(ops);
      auto kern = mul ? k_merge_rows<Ops, true> : k_merge_rows<Ops, false>;
      if (rows)
        SK_LAUNCH(kern, grid_for(ctx, rows), 256, 0, ctx->stream, a->rp, a->ci, a->v, b->rp,
                  b->ci, b->v, rows, cnt, nullptr, nullptr, nullptr, ctx->d_err);
      exclusive_scan_u32(ctx, cnt, rp, size_t(rows) + 1);
      uint32_t nnz = 0;
      SK_CUDA(cudaMemcpyAsync(&nnz, rp + rows, 4, cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      o = new_csr(ctx, rows, a->cols, nnz);
      SK_CUDA(cudaMemcpyAsync(o->rp, rp, (size_t(rows) + 1) * 4, cudaMemcpyDeviceToDevice,
                              ctx->stream));
      if (rows)
        SK_LAUNCH(kern, grid_for(ctx, rows), 256, 0, ctx->stream, a->rp, a->ci, a->v, b->rp,
                  b->ci, b->v, rows, nullptr, o->rp, o->ci, o->v, ctx->d_err);
    });
    dfree(ctx, cnt);
    dfree(ctx, rp);
    if (s == SK_GF2) {
      try {
        check_device_error(ctx, mul ? "ewise_mul" : "ewise_add");
      } catch (...) {
        csr_release(o);
        throw;
      }
    }
    *out = o;
  });
}

// ==== category set =====================================================================

namespace sk {
__global__ void k_flag_cols_csr(const uint32_t* ci, const float* v, size_t nnz,
                                uint8_t* flags) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < nnz;
       e += size_t(gridDim.x) * blockDim.x)
    if (v[e] != 0.0f) flags[ci[e]] = 1;  // benign race: every writer stores 1
}
__global__ void k_flag_cols_dense(const float* d, uint32_t rows, uint32_t cols,
                                  uint8_t* flags) {
  const size_t n = size_t(rows) * cols;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    if (d[i] != 0.0f) flags[i % cols] = 1;
}

__global__ void k_post_list(const int* nsel, const uint32_t* list, volatile uint32_t* box,
                            uint32_t cap, uint32_t seq) {
  const uint32_t n = uint32_t(*nsel);
  if (threadIdx.x == 0) box[kMboxHdr] = n;
  if (n <= cap)
    for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) box[kMboxHdr + 1 + j] = list[j];
  __threadfence_system();  // every thread's stores before the flag
  __syncthreads();
  if (threadIdx.x == 0) box[0] = seq;
}

void categories_from_flags(sk_ctx* ctx, uint8_t* flags, uint32_t n, uint32_t* idx,
                           size_t cap, size_t* count) {
  uint32_t* out = dalloc<uint32_t>(ctx, n);
  int* nsel = reinterpret_cast<int*>(ctx->d_u64);
  size_t tmp = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  SK_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, nsel, n, ctx->stream));
  void* t = dalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceSelect::Flagged(t, tmp, it, flags, out, nsel, n, ctx->stream));
  g_launches.fetch_add(1);
  // count + (when it fits) the list itself through the mailbox: no device->host
  // copies, no stream synchronise (both stall beside a bulk upload on another stream)
  const uint32_t seq = ++ctx->mbox_seq;
  SK_LAUNCH(k_post_list, 1, 256, 0, ctx->stream, nsel, out, ctx->mbox_dev, kMboxWords - 1, seq);
  mbox_wait(ctx, seq);
  const uint32_t h = ctx->mbox[kMboxHdr];
  *count = size_t(h);
  if (idx && h) {
    const size_t take = std::min<size_t>(cap, h);
    if (h <= kMboxWords - 1) {
      std::memcpy(idx, ctx->mbox + kMboxHdr + 1, take * 4);
    } else {
      SK_CUDA(cudaMemcpyAsync(idx, out, take * 4, cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
    }
  }
  dfree(ctx, t);
  dfree(ctx, out);
}
}  // namespace sk

extern "C" sk_status sk_categories_csr(sk_ctx* ctx, const sk_csr* y, uint32_t* idx, size_t cap,
                                       size_t* count) {
  return guarded([&] {
    csr_ready(ctx, y);
    SK_CUDA(cudaSetDevice(ctx->device));
    if (y->nnz == 0) {  // no stored entry, no category: nothing to launch or read back
      *count = 0;
      return;
    }
    uint8_t* flags = dalloc<uint8_t>(ctx, y->cols);
    SK_CUDA(cudaMemsetAsync(flags, 0, y->cols, ctx->stream));
    if (y->nnz)
      SK_LAUNCH(k_flag_cols_csr, grid_for(ctx, y->nnz), 256, 0, ctx->stream, y->ci, y->v, y->nnz,
                flags);
    categories_from_flags(ctx, flags, y->cols, idx, cap, count);
    dfree(ctx, flags);
  });
}

extern "C" sk_status sk_categories_dense(sk_ctx* ctx, const sk_dense* y, uint32_t* idx,
                                         size_t cap, size_t* count) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    uint8_t* flags = dalloc<uint8_t>(ctx, y->cols);
    SK_CUDA(cudaMemsetAsync(flags, 0, y->cols, ctx->stream));
    if (y->elems())
      SK_LAUNCH(k_flag_cols_dense, grid_for(ctx, y->elems()), 256, 0, ctx->stream, y->d, y->rows,
                y->cols, flags);
    categories_from_flags(ctx, flags, y->cols, idx, cap, count);
    dfree(ctx, flags);
  });
}

// ==== generators (bitwise equal to oracle/sk_oracle.c) ===============================

namespace sk {

__device__ __forceinline__ uint32_t bounded(uint64_t bits, uint32_t range) {
  return uint32_t(__umul64hi(bits, uint64_t(range)));
}

// Row i (global index i + row_offset) draws distinct sorted columns in place.
__global__ void k_gen_fixed_rows(uint32_t rows, uint32_t cols, uint32_t k, uint64_t seed,
                                 uint64_t row_offset, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += gridDim.x * blockDim.x) {
    const uint64_t rs = splitmix_at(seed, uint64_t(i) + row_offset);
    uint32_t* row = out + size_t(i) * k;
    uint32_t have = 0;
    for (uint64_t t = 0; have < k; ++t) {
      const uint32_t c = bounded(splitmix_at(rs, t), cols);
      uint32_t lo = 0, hi = have;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (row[mid] < c) lo = mid + 1; else hi = mid;
      }
      if (lo < have && row[lo] == c) continue;
      for (uint32_t q = have; q > lo; --q) row[q] = row[q - 1];
      row[lo] = c;
      ++have;
    }
  }
}

__device__ __forceinline__ float uniform_pm1(uint64_t seed, uint64_t idx) {
  const float v = float(__dadd_rn(-1.0, __dmul_rn(2.0, to_unit(splitmix_at(seed, idx)))));
  return v == 0.0f ? 1.0f : v;
}

__global__ void k_gen_values(float* v, size_t n, uint64_t seed, float value, int uniform) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < n;
       e += size_t(gridDim.x) * blockDim.x)
    v[e] = uniform ? uniform_pm1(seed, e) : value;
}

__global__ void k_iota_rp(uint32_t* rp, uint32_t rows, uint32_t k) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
       i += gridDim.x * blockDim.x)
    rp[i] = i * k;
}

// cfg2: W_ref row j, column i present iff U(at(sel, i*m+j)) < density.
__global__ void k_gen_density(uint32_t m, double density, uint64_t sel, uint64_t val,
                              const uint32_t* rp, uint32_t* cnt, uint32_t* ci, float* v) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    const uint32_t o = rp ? rp[j] : 0;
    for (uint32_t i = 0; i < m; ++i) {
      const uint64_t idx = uint64_t(i) * m + j;
      if (to_unit(splitmix_at(sel, idx)) < density) {
        if (rp) {
          ci[o + c] = i;
          v[o + c] = uniform_pm1(val, idx);
        }
        ++c;
      }
    }
    if (!rp) cnt[j] = c;
  }
}

__global__ void k_widen_u32(const uint32_t* in, uint64_t* out, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[i];
}
__global__ void k_narrow_u64(const uint64_t* in, uint32_t* out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(in[i]);
}

// The reference's own gen_weight (proj/src/matgen.cpp:50-87): entry (i, j) of the
// m x m CSR owns counter i*m+j of the select and value streams; present iff
// to_unit(select) < 1/inverse_sparsity, value float(-1 + 4 to_unit(value)),
// exact zeros elided.  Warp per row, lanes over columns, ballot compaction keeps
// the columns ascending.  Pass 1 (rp == nullptr) counts, pass 2 writes.
__global__ void k_gen_weight_ref(uint32_t m, double p, uint64_t sel, uint64_t val,
                                 const uint32_t* rp, uint32_t* cnt, uint32_t* ci, float* v) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += (gridDim.x * blockDim.x) >> 5) {
    uint32_t o = rp ? rp[i] : 0u;
    uint32_t c = 0;
    for (uint32_t j0 = 0; j0 < m; j0 += 32) {
      const uint32_t j = j0 + lane;
      bool keep = false;
      float x = 0.0f;
      if (j < m) {
        const uint64_t idx = uint64_t(i) * m + j;
        if (to_unit(splitmix_at(sel, idx)) < p) {
          x = float(__dadd_rn(-1.0, __dmul_rn(4.0, to_unit(splitmix_at(val, idx)))));
          keep = x != 0.0f;
        }
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, keep);
      if (rp && keep) {
        const uint32_t pos = o + __popc(bm & ((1u << lane) - 1u));
        ci[pos] = j;
        v[pos] = x;
      }
      o += __popc(bm);
      c += __popc(bm);
    }
    if (!rp && lane == 0) cnt[i] = c;
  }
}

__global__ void k_gen_input_dense(float* y, size_t n, uint64_t stream) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    y[i] = float(to_unit(splitmix_at(stream, i)));
}

sk_csr* gen_fixed_csr(sk_ctx* ctx, uint32_t rows, uint32_t cols, uint32_t k, uint64_t sel_seed,
                      uint64_t row_offset, uint64_t val_seed, float value, int uniform) {
  if (k > cols) fail(SK_ERR_INVALID_ARGUMENT, "k exceeds the number of columns");
  sk_csr* a = new_csr(ctx, rows, cols, size_t(rows) * k);
  SK_LAUNCH(k_gen_fixed_rows, grid_for(ctx, rows, 128), 128, 0, ctx->stream, rows, cols, k,
            sel_seed, row_offset, a->ci);
  SK_LAUNCH(k_gen_values, grid_for(ctx, a->nnz), 256, 0, ctx->stream, a->v, a->nnz, val_seed,
            value, uniform);
  SK_LAUNCH(k_iota_rp, grid_for(ctx, size_t(rows) + 1), 256, 0, ctx->stream, a->rp, rows, k);
  return a;
}

}  // namespace sk

extern "C" sk_status sk_gen_layer_fixed(sk_ctx* ctx, uint32_t m, uint32_t k, uint64_t layer_seed,
                                        float value, sk_csr** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    const int uniform = value != value;
    sk_csr* w = gen_fixed_csr(ctx, m, m, k, splitmix_at(layer_seed, 0), 0,
                              splitmix_at(layer_seed, 1), value, uniform);
    sk_csr* t = csr_transpose(ctx, w);
    csr_release(w);
    *out = t;
  });
}

extern "C" sk_status sk_gen_layer_density(sk_ctx* ctx, uint32_t m, double density,
                                          uint64_t layer_seed, sk_csr** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    const uint64_t sel = splitmix_at(layer_seed, 0), val = splitmix_at(layer_seed, 1);
    uint32_t* cnt = dalloc<uint32_t>(ctx, size_t(m) + 1);
    uint32_t* rp = dalloc<uint32_t>(ctx, size_t(m) + 1);
    SK_CUDA(cudaMemsetAsync(cnt + m, 0, 4, ctx->stream));
    SK_LAUNCH(k_gen_density, grid_for(ctx, m, 128), 128, 0, ctx->stream, m, density, sel, val,
              nullptr, cnt, nullptr, nullptr);
    exclusive_scan_u32(ctx, cnt, rp, size_t(m) + 1);
    uint32_t nnz = 0;
    SK_CUDA(cudaMemcpyAsync(&nnz, rp + m, 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    sk_csr* a = new_csr(ctx, m, m, nnz);
    SK_CUDA(cudaMemcpyAsync(a->rp, rp, (size_t(m) + 1) * 4, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    SK_LAUNCH(k_gen_density, grid_for(ctx, m, 128), 128, 0, ctx->stream, m, density, sel, val,
              a->rp, nullptr, a->ci, a->v);
    dfree(ctx, cnt);
    dfree(ctx, rp);
    *out = a;
  });
}

extern "C" sk_status sk_gen_weight(sk_ctx* ctx, uint32_t m, double inverse_sparsity,
                                   uint64_t seed, sk_csr** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    // GenSpec::validate (matgen.cpp:25-31)
    if (m < 1) fail(SK_ERR_INVALID_ARGUMENT, "GenSpec: m must be >= 1");
    if (!(inverse_sparsity >= 1.0))
      fail(SK_ERR_INVALID_ARGUMENT, "GenSpec: inverse_sparsity must be >= 1");
    const double p = 1.0 / inverse_sparsity;
    const uint64_t sel = splitmix_at(seed, 0), val = splitmix_at(seed, 1);  // kWeightSelect/Value
    uint32_t* cnt = dalloc<uint32_t>(ctx, size_t(m) + 1);
    unsigned long long* rp64 =
        reinterpret_cast<unsigned long long*>(dalloc<uint64_t>(ctx, size_t(m) + 1));
    uint64_t* cnt64 = dalloc<uint64_t>(ctx, size_t(m) + 1);
    SK_LAUNCH(k_gen_weight_ref, grid_for(ctx, size_t(m) * 32), 256, 0, ctx->stream, m, p, sel,
              val, nullptr, cnt, nullptr, nullptr);
    SK_LAUNCH(k_widen_u32, grid_for(ctx, m), 256, 0, ctx->stream, cnt, cnt64, m);
    SK_CUDA(cudaMemsetAsync(cnt64 + m, 0, 8, ctx->stream));
    exclusive_scan_u64(ctx, cnt64, reinterpret_cast<uint64_t*>(rp64), size_t(m) + 1);
    const uint64_t nnz = read_u64(ctx, rp64 + m);
    if (nnz > 0xFFFFFFFFull) {
      dfree(ctx, cnt);
      dfree(ctx, rp64);
      dfree(ctx, cnt64);
      fail(SK_ERR_INVALID_ARGUMENT, "generated nnz exceeds the 32-bit index range");
    }
    sk_csr* a = new_csr(ctx, m, m, nnz);
    SK_LAUNCH(k_narrow_u64, grid_for(ctx, size_t(m) + 1), 256, 0, ctx->stream,
              reinterpret_cast<const uint64_t*>(rp64), a->rp, size_t(m) + 1);
    SK_LAUNCH(k_gen_weight_ref, grid_for(ctx, size_t(m) * 32), 256, 0, ctx->stream, m, p, sel,
              val, a->rp, nullptr, a->ci, a->v);
    dfree(ctx, cnt);
    dfree(ctx, rp64);
    dfree(ctx, cnt64);
    *out = a;
  });
}

extern "C" sk_status sk_gen_input_dense(sk_ctx* ctx, uint32_t m, uint32_t n, uint64_t seed,
                                        sk_dense** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    sk_dense* d = new_dense(ctx, m, n);
    if (d->elems())
      SK_LAUNCH(k_gen_input_dense, grid_for(ctx, d->elems()), 256, 0, ctx->stream, d->d,
                d->elems(), splitmix_at(seed, 2));
    *out = d;
  });
}

extern "C" sk_status sk_gen_input_binary(sk_ctx* ctx, uint32_t m, uint32_t n, uint32_t k,
                                         uint64_t seed, uint64_t sample_offset, sk_csr** out) {
  return guarded([&] {
    SK_CUDA(cudaSetDevice(ctx->device));
    sk_csr* b = gen_fixed_csr(ctx, n, m, k, splitmix_at(seed, 4), sample_offset, 0, 1.0f, 0);
    sk_csr* t = csr_transpose(ctx, b);
    csr_release(b);
    t->stats = const_value_stats(1.0f, t->nnz);  // binary: known at construction
    t->stats_valid = true;
    *out = t;
  });
}

// ---- column-sharded exchange over peer memory ----------------------------------------
// Each rank's block of output rows (a CSR of rows [row_off, row_off + rows) of
// Y_{k+1}) is written by ONE kernel straight into every rank's next-layer input
// buffers (CUDA IPC pointers to the peers' memory: stores over NVLink), at its
// entry offset nnz_off, with the row pointers shifted by nnz_off; the last rank
// also writes the closing row pointer.  The buffers are plain cudaMalloc
// allocations exported with cudaIpcGetMemHandle.

namespace sk {
namespace {

struct PublishDst {
  uint32_t* rp[8];
  uint32_t* ci[8];
  float* v[8];
};

__global__ void k_csr_publish(const uint32_t* rp, const uint32_t* ci, const float* v, uint32_t rows,
                              size_t nnz, PublishDst dst, uint32_t nd, uint32_t row_off,
                              uint32_t nnz_off, int write_last) {
  const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  const size_t nth = size_t(gridDim.x) * blockDim.x;
  for (uint32_t d = 0; d < nd; ++d) {
    uint32_t* const oci = dst.ci[d] + nnz_off;
    float* const ov = dst.v[d] + nnz_off;
    for (size_t e = tid; e < nnz; e += nth) {
      oci[e] = ci[e];
      ov[e] = v[e];
    }
    uint32_t* const orp = dst.rp[d] + row_off;
    for (size_t i = tid; i < rows; i += nth) orp[i] = rp[i] + nnz_off;
    if (write_last && tid == 0) orp[rows] = rp[rows] + nnz_off;
  }
}

}  // namespace
}  // namespace sk

static void ipc_ctx(sk_ctx* ctx) {
  if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
  SK_CUDA(cudaSetDevice(ctx->device));
}

extern "C" sk_status sk_ipc_alloc(sk_ctx* ctx, size_t bytes, void** dptr, unsigned char* handle) {
  return guarded([&] {
    ipc_ctx(ctx);
    void* p = nullptr;
    SK_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      fail(SK_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    std::memcpy(handle, &h, sizeof(h));
    *dptr = p;
  });
}

extern "C" sk_status sk_ipc_open(sk_ctx* ctx, const unsigned char* handle, void** dptr) {
  return guarded([&] {
    ipc_ctx(ctx);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    SK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = p;
  });
}

extern "C" sk_status sk_ipc_close(void* dptr) {
  return guarded([&] {
    if (dptr) SK_CUDA(cudaIpcCloseMemHandle(dptr));
  });
}

extern "C" sk_status sk_ipc_free(void* dptr) {
  return guarded([&] {
    if (dptr) SK_CUDA(cudaFree(dptr));
  });
}

namespace sk {
void csr_publish_impl(sk_ctx* ctx, const sk_csr* blk, uint32_t ndst, uint32_t* const* dst_rp,
                      uint32_t* const* dst_ci, float* const* dst_v, uint32_t row_off,
                      uint64_t nnz_off, int write_last) {
  csr_ready(ctx, blk);
  if (ndst > 8) fail(SK_ERR_INVALID_ARGUMENT, "at most 8 destinations (one NVLink box)");
  if (nnz_off + blk->nnz > 0xFFFFFFFFull)
    fail(SK_ERR_INVALID_ARGUMENT, "exchange exceeds the 32-bit index range");
  PublishDst d{};
  for (uint32_t r = 0; r < ndst; ++r) {
    d.rp[r] = dst_rp[r];
    d.ci[r] = dst_ci[r];
    d.v[r] = dst_v[r];
  }
  const uint64_t work = std::max<uint64_t>(blk->nnz, blk->rows);
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((work + 255) / 256, uint64_t(ctx->num_sms) * 8)));
  SK_LAUNCH(k_csr_publish, grid, 256, 0, ctx->stream, blk->rp, blk->ci, blk->v, blk->rows,
            blk->nnz, d, ndst, row_off, uint32_t(nnz_off), write_last);
}
}  // namespace sk

extern "C" sk_status sk_csr_publish(sk_ctx* ctx, const sk_csr* blk, uint32_t ndst,
                                    uint32_t* const* dst_rp, uint32_t* const* dst_ci,
                                    float* const* dst_v, uint32_t row_off, uint64_t nnz_off,
                                    int write_last) {
  return guarded([&] {
    ipc_ctx(ctx);
    csr_publish_impl(ctx, blk, ndst, dst_rp, dst_ci, dst_v, row_off, nnz_off, write_last);
  });
}
