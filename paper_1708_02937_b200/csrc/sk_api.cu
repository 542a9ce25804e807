// C-ABI entry points of libsk_b200 (include/sk_api.h): contexts, handles,
// transfers, model construction and argument/shape checking.  Shape checks
// and their messages follow the reference (proj/src/matrix.cpp:28-46,
// proj/src/dnn.cpp:23-61,86-98); the compute lives in k_*.cu.
#include <cub/cub.cuh>

#include <cstring>
#include <initializer_list>
#include <map>
#include <mutex>
#include <tuple>

#include "sk_async.cuh"
#include "sk_common.cuh"

namespace sk {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;

void set_last_error(const std::string& msg) { t_last_error = msg; }

void dfree(sk_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

void arena_begin(sk_ctx* ctx) {
  if (ctx->arena_depth++ > 0) return;
  ctx->arena_top = 0;
  if (ctx->arena_high > ctx->arena_cap) {  // grow once to the last call's high-water mark
    if (ctx->arena) cudaFreeAsync(ctx->arena, ctx->stream);
    ctx->arena = nullptr;
    ctx->arena_cap = 0;
    const size_t cap = ctx->arena_high + ctx->arena_high / 8;
    void* p = nullptr;
    if (cudaMallocAsync(&p, cap, ctx->stream) == cudaSuccess) {
      ctx->arena = static_cast<uint8_t*>(p);
      ctx->arena_cap = cap;
    } else {
      cudaGetLastError();  // fall back to per-allocation memory this call
    }
  }
}

void* arena_alloc_bytes(sk_ctx* ctx, size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (ctx->arena_depth == 0) return dalloc<uint8_t>(ctx, bytes);  // not inside a call
  const size_t top = ctx->arena_top;
  ctx->arena_top += bytes;
  ctx->arena_high = std::max(ctx->arena_high, ctx->arena_top);
  if (top + bytes <= ctx->arena_cap) return ctx->arena + top;
  void* p = dalloc<uint8_t>(ctx, bytes);  // spill; the next call's arena covers it
  ctx->arena_spill.push_back(p);
  return p;
}

void arena_end(sk_ctx* ctx) {
  if (--ctx->arena_depth > 0) return;
  for (void* p : ctx->arena_spill) dfree(ctx, p);
  ctx->arena_spill.clear();
}

sk_dense* new_dense(sk_ctx* ctx, uint32_t rows, uint32_t cols) {
  auto* d = new sk_dense;
  d->ctx = ctx;
  d->rows = rows;
  d->cols = cols;
  d->d = dalloc<float>(ctx, d->elems());
  return d;
}

sk_csr* new_csr(sk_ctx* ctx, uint32_t rows, uint32_t cols, size_t nnz) {
  auto* a = new sk_csr;
  a->ctx = ctx;
  a->rows = rows;
  a->cols = cols;
  a->nnz = nnz;
  a->rp = dalloc<uint32_t>(ctx, size_t(rows) + 1);
  a->ci = dalloc<uint32_t>(ctx, nnz + kCiPad);
  a->v = dalloc<float>(ctx, nnz);
  return a;
}

void csr_release(sk_csr* a) {
  if (!a) return;
  if (a->refs.fetch_sub(1) == 1) {
    if (a->ready) {
      csr_ready(a->ctx, a);  // the copies finish before the stream-ordered frees
      cudaEventDestroy(a->ready);
    }
    dfree(a->ctx, a->rp);
    dfree(a->ctx, a->ci);
    dfree(a->ctx, a->v);
    if (a->tile_vals) dfree(a->ctx, a->tile_vals);
    if (a->pack.buf) dfree(a->ctx, a->pack.buf);
    if (a->tile_mask) dfree(a->ctx, a->tile_mask);
    delete a;
  }
}

void sync(sk_ctx* ctx) { SK_CUDA(cudaStreamSynchronize(ctx->stream)); }

__global__ void k_post_words(PostSrc s, volatile uint32_t* box, uint32_t seq) {
  const uint32_t lane = threadIdx.x;
  uint32_t o = kMboxHdr;
  for (int i = 0; i < s.cnt; ++i) {
    for (uint32_t j = lane; j < s.n[i]; j += 32) box[o + j] = s.p[i][j];
    o += s.n[i];
  }
  __threadfence_system();  // each lane's payload stores before the flag
  __syncwarp();
  if (lane == 0) box[0] = seq;
}

Fetch& Fetch::add(const void* dev, uint32_t words) {
  if (s.cnt >= 8) fail(SK_ERR_INVALID_ARGUMENT, "fetch: too many sources");
  s.p[s.cnt] = static_cast<const uint32_t*>(dev);
  s.n[s.cnt] = words;
  ++s.cnt;
  return *this;
}

void mbox_wait(sk_ctx* ctx, uint32_t seq) {
  volatile uint32_t* flag = ctx->mbox;
  for (unsigned spins = 1;; ++spins) {
    if (*flag == seq) return;
    if ((spins & 0x3FF) == 0) {  // a faulted or drained stream must not spin forever
      const cudaError_t q = cudaStreamQuery(ctx->stream);
      if (q == cudaSuccess) {
        if (*flag == seq) return;
        fail(SK_ERR_CUDA, "mailbox: the stream drained without posting");
      }
      if (q != cudaErrorNotReady) SK_CUDA(q);
    }
    __builtin_ia32_pause();
  }
}

const uint32_t* Fetch::run() {
  uint32_t total = 0;
  for (int i = 0; i < s.cnt; ++i) total += s.n[i];
  if (total > kMboxWords) fail(SK_ERR_INVALID_ARGUMENT, "fetch: payload exceeds the mailbox");
  const uint32_t seq = ++ctx->mbox_seq;
  SK_LAUNCH(k_post_words, 1, 32, 0, ctx->stream, s, ctx->mbox_dev, seq);
  mbox_wait(ctx, seq);
  return ctx->mbox + kMboxHdr;
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_attr;                        // smem bytes set
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;           // blocks per SM
}  // namespace

void kernel_smem_attr(sk_ctx* ctx, const void* kernel, int bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& have = g_attr[{kernel, ctx->device}];
  if (have >= bytes) return;
  SK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

namespace async {
bool make_tmap_2d_f32(CUtensorMap* map, const float* base, uint64_t rows, uint64_t cols,
                      uint64_t pitch_elems, uint32_t box_rows, uint32_t box_cols) {
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch_elems * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace async

int kernel_occupancy(sk_ctx* ctx, const void* kernel, int threads, size_t smem) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  const auto key = std::make_tuple(kernel, ctx->device, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per_sm = 0;
  SK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  g_occ[key] = per_sm;
  return per_sm;
}

void timing_mark(sk_ctx* ctx, int tag) {
  if (!ctx->timing) return;
  if (ctx->ev_used == ctx->ev.size()) {
    cudaEvent_t e;
    SK_CUDA(cudaEventCreate(&e));
    ctx->ev.push_back(e);
  }
  if (ctx->ev_used % 2 == 0) {
    if (ctx->ev_tag.size() <= ctx->ev_used / 2) ctx->ev_tag.resize(ctx->ev_used / 2 + 1);
    ctx->ev_tag[ctx->ev_used / 2] = tag;
  }
  SK_CUDA(cudaEventRecord(ctx->ev[ctx->ev_used++], ctx->stream));
}

void check_device_error(sk_ctx* ctx, const char* op) {
  int err = 0;
  SK_CUDA(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream));
  sync(ctx);
  if (err != 0) {
    SK_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
    if (err == kErrGf2Domain)
      fail(SK_ERR_DOMAIN, std::string(op) + ": GF(2) scalar must be 0 or 1");
    fail(SK_ERR, std::string(op) + ": device error " + std::to_string(err));
  }
}

void exclusive_scan_u32(sk_ctx* ctx, const uint32_t* in, uint32_t* out, size_t n) {
  size_t tmp = 0;
  SK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, ctx->stream));
  void* t = dalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, ctx->stream));
  g_launches.fetch_add(1);
  dfree(ctx, t);
}

void exclusive_scan_u64(sk_ctx* ctx, const uint64_t* in, uint64_t* out, size_t n) {
  size_t tmp = 0;
  SK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, ctx->stream));
  void* t = dalloc<char>(ctx, tmp);
  SK_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, ctx->stream));
  g_launches.fetch_add(1);
  dfree(ctx, t);
}

float semiring_zero_host(sk_semiring s) {
  switch (s) {
    case SK_MAX_PLUS: return -INFINITY;
    case SK_MIN_MAX: return INFINITY;
    default: return 0.0f;
  }
}

static void require_ctx(sk_ctx* ctx) {
  if (!ctx) fail(SK_ERR_INVALID_ARGUMENT, "null context");
  SK_CUDA(cudaSetDevice(ctx->device));
}

// ---- small kernels used by the API layer ---------------------------------------

__global__ void k_fill(float* p, size_t n, float v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_identity(float* p, uint32_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < size_t(n);
       i += size_t(gridDim.x) * blockDim.x)
    p[i * n + i] = 1.0f;
}

void fill(sk_ctx* ctx, float* p, size_t n, float v) {
  if (n == 0) return;
  unsigned grid = std::min<unsigned>(ceil_div(n, 256), ctx->num_sms * 8);
  SK_LAUNCH(k_fill, grid, 256, 0, ctx->stream, p, n, v);
}

}  // namespace sk

using namespace sk;

// ==== library / context ==========================================================

extern "C" const char* sk_last_error(void) { return sk::t_last_error.c_str(); }
extern "C" const char* sk_version(void) { return "sk_b200 0.1 (sm_100a)"; }
extern "C" uint64_t sk_kernel_launch_count(void) { return g_launches.load(); }

extern "C" sk_status sk_ctx_create(int device, sk_ctx** out) {
  return guarded([&] {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      fail(SK_ERR_CUDA, std::string("no CUDA device available: ") +
                            (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    if (device < 0 || device >= count)
      fail(SK_ERR_INVALID_ARGUMENT, "device " + std::to_string(device) + " out of range");
    SK_CUDA(cudaSetDevice(device));
    auto* c = new sk_ctx;
    c->device = device;
    SK_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    SK_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    {
      size_t fr = 0, tot = 0;
      SK_CUDA(cudaMemGetInfo(&fr, &tot));
      c->total_mem = tot;
    }
    cudaMemPool_t pool;
    SK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thresh = UINT64_MAX;
    SK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    SK_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
    SK_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
    SK_CUDA(cudaMalloc(&c->d_u64, 64 * sizeof(uint64_t)));
    SK_CUDA(cudaMemset(c->d_u64, 0, 64 * sizeof(uint64_t)));
    SK_CUDA(cudaMallocHost(&c->h_u64, 64 * sizeof(uint64_t)));
    SK_CUDA(cudaHostAlloc(&c->mbox, (kMboxHdr + kMboxWords) * sizeof(uint32_t),
                          cudaHostAllocMapped));
    std::memset(c->mbox, 0, (kMboxHdr + kMboxWords) * sizeof(uint32_t));
    SK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->mbox_dev), c->mbox, 0));
    *out = c;
  });
}

extern "C" sk_status sk_ctx_destroy(sk_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_u64);
    cudaFreeHost(ctx->h_u64);
    cudaFreeHost(ctx->mbox);
    for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->watch)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->pin_ev)
      if (e) cudaEventDestroy(e);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    if (ctx->stamps) cudaFree(ctx->stamps);
    if (ctx->arena) cudaFreeAsync(ctx->arena, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

extern "C" sk_status sk_ctx_set_stream(sk_ctx* ctx, void* s) {
  return guarded([&] {
    require_ctx(ctx);
    const cudaStream_t next = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    if (next != ctx->stream) SK_CUDA(cudaStreamSynchronize(ctx->stream));  // arena reuse order
    ctx->stream = next;
  });
}

extern "C" void* sk_ctx_stream(const sk_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

extern "C" sk_status sk_ctx_set_density_switch(sk_ctx* ctx, double dense_above,
                                               double sparse_below) {
  return guarded([&] {
    require_ctx(ctx);
    if (!(sparse_below >= 0.0) || (dense_above > 0 && sparse_below > dense_above))
      fail(SK_ERR_INVALID_ARGUMENT, "density switch needs 0 <= sparse_below <= dense_above");
    ctx->dense_above = dense_above > 0 ? dense_above : 0.0;
    ctx->sparse_below = sparse_below;
  });
}

extern "C" sk_status sk_ctx_set_tuning(sk_ctx* ctx, const sk_tuning* t) {
  return guarded([&] {
    require_ctx(ctx);
    if (!t) fail(SK_ERR_INVALID_ARGUMENT, "null tuning");
    auto in = [](int v, std::initializer_list<int> ok) {
      for (int o : ok)
        if (v == o) return true;
      return false;
    };
    if (!in(t->exact, {-1, 0, 1}) || !in(t->esc, {-1, 0, 1}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact / esc must be -1, 0 or 1");
    if (!in(t->exact_kernel, {0, 1, 2, 3, 4, 5}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact_kernel must be 0..5");
    if (!in(t->exact_group, {0, 1, 2, 4, 8, 16, 32, 64}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact_group must be 0, 1, 2, 4, 8, 16, 32 or 64");
    if (!in(t->exact_records, {0, 64, 192}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact_records must be 0, 64 or 192");
    auto wl = [](int v) { return v == 0 || (v >= 8 && v <= 12); };
    if (!wl(t->window_log2) || !wl(t->exact_window_log2))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: window log2 must be 0 or 8..12");
    if (!in(t->exact_fields, {0, 4, 8}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact_fields must be 0, 4 or 8");
    if (!in(t->exact_layout, {0, 1, 2, 3}))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: exact_layout must be 0, 1, 2 or 3");
    if (!(t->esc_ratio == t->esc_ratio))
      fail(SK_ERR_INVALID_ARGUMENT, "tuning: esc_ratio is NaN");
    ctx->tune = *t;
  });
}

extern "C" sk_status sk_ctx_get_tuning(const sk_ctx* ctx, sk_tuning* t) {
  return guarded([&] {
    if (!ctx || !t) fail(SK_ERR_INVALID_ARGUMENT, "null context or tuning");
    *t = ctx->tune;
  });
}

extern "C" sk_status sk_ctx_last_exact(const sk_ctx* ctx, sk_exact_info* info) {
  return guarded([&] {
    if (!ctx || !info) fail(SK_ERR_INVALID_ARGUMENT, "null context or info");
    *info = ctx->last_exact;
  });
}

extern "C" sk_status sk_ctx_set_timing(sk_ctx* ctx, int enable) {
  return guarded([&] {
    require_ctx(ctx);
    ctx->timing = enable != 0;
    ctx->ev_used = 0;
    if (enable && !ctx->stamps) {
      ctx->stamps_cap = 1 << 16;
      SK_CUDA(cudaMalloc(&ctx->stamps, size_t(ctx->stamps_cap) * sizeof(long long)));
    }
    if (!enable && ctx->stamps) {
      sync(ctx);
      cudaFree(ctx->stamps);
      ctx->stamps = nullptr;
      ctx->stamps_cap = 0;
    }
  });
}

namespace sk {
constexpr int kPinSlots = 4;
constexpr size_t kPinSlotBytes = size_t(64) << 10;

void upload_staged(sk_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (bytes > kPinSlotBytes) {  // pageable: staged by the driver before the call returns
    SK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return;
  }
  if (!ctx->pin) {
    SK_CUDA(cudaMallocHost(&ctx->pin, kPinSlots * kPinSlotBytes));
    for (cudaEvent_t& e : ctx->pin_ev) SK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int slot = ctx->pin_next;
  ctx->pin_next = (slot + 1) % kPinSlots;
  SK_CUDA(cudaEventSynchronize(ctx->pin_ev[slot]));  // the slot's previous copy is done
  char* p = ctx->pin + size_t(slot) * kPinSlotBytes;
  std::memcpy(p, src, bytes);
  SK_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
  SK_CUDA(cudaEventRecord(ctx->pin_ev[slot], ctx->stream));
}
}  // namespace sk

extern "C" sk_status sk_ctx_timer_start(sk_ctx* ctx) {
  return guarded([&] {
    require_ctx(ctx);
    SK_CUDA(cudaSetDevice(ctx->device));
    for (cudaEvent_t& e : ctx->watch)
      if (!e) SK_CUDA(cudaEventCreate(&e));
    SK_CUDA(cudaEventRecord(ctx->watch[0], ctx->stream));
  });
}

extern "C" sk_status sk_ctx_timer_stop(sk_ctx* ctx, float* ms) {
  return guarded([&] {
    require_ctx(ctx);
    if (!ms) fail(SK_ERR_INVALID_ARGUMENT, "sk_ctx_timer_stop: null output");
    if (!ctx->watch[0]) fail(SK_ERR_INVALID_ARGUMENT, "sk_ctx_timer_stop: timer never started");
    SK_CUDA(cudaSetDevice(ctx->device));
    SK_CUDA(cudaEventRecord(ctx->watch[1], ctx->stream));
    SK_CUDA(cudaEventSynchronize(ctx->watch[1]));
    SK_CUDA(cudaEventElapsedTime(ms, ctx->watch[0], ctx->watch[1]));
  });
}

extern "C" sk_status sk_ctx_layer_stamps(sk_ctx* ctx, long long* ns, size_t n) {
  return guarded([&] {
    require_ctx(ctx);
    if (!ctx->stamps) fail(SK_ERR_INVALID_ARGUMENT, "timing is not enabled");
    if (n > ctx->stamps_cap) n = ctx->stamps_cap;
    SK_CUDA(cudaMemcpyAsync(ns, ctx->stamps, n * sizeof(long long), cudaMemcpyDeviceToHost,
                            ctx->stream));
    sync(ctx);
  });
}

extern "C" sk_status sk_ctx_layer_paths(sk_ctx* ctx, unsigned char* paths, size_t n) {
  return guarded([&] {
    require_ctx(ctx);
    if (n && !paths) fail(SK_ERR_INVALID_ARGUMENT, "null paths buffer");
    for (size_t q = 0; q < n; ++q)
      paths[q] = q < ctx->last_paths.size() ? ctx->last_paths[q] : (unsigned char)SK_PATH_EMPTY;
  });
}

extern "C" sk_status sk_ctx_kernel_times(sk_ctx* ctx, float* ms, size_t cap, size_t* count) {
  return guarded([&] {
    require_ctx(ctx);
    sync(ctx);
    const size_t pairs = ctx->ev_used / 2;
    *count = pairs;
    for (size_t i = 0; i < pairs && i < cap; ++i)
      SK_CUDA(cudaEventElapsedTime(&ms[i], ctx->ev[2 * i], ctx->ev[2 * i + 1]));
    ctx->ev_used = 0;
  });
}

extern "C" sk_status sk_ctx_kernel_times_tagged(sk_ctx* ctx, float* ms, int* tags, size_t cap,
                                                size_t* count) {
  return guarded([&] {
    require_ctx(ctx);
    sync(ctx);
    const size_t pairs = ctx->ev_used / 2;
    *count = pairs;
    for (size_t i = 0; i < pairs && i < cap; ++i) {
      SK_CUDA(cudaEventElapsedTime(&ms[i], ctx->ev[2 * i], ctx->ev[2 * i + 1]));
      tags[i] = ctx->ev_tag[i];
    }
    ctx->ev_used = 0;
  });
}

extern "C" sk_status sk_ctx_synchronize(sk_ctx* ctx) {
  return guarded([&] {
    require_ctx(ctx);
    sync(ctx);
  });
}

extern "C" sk_status sk_host_register(void* p, size_t bytes) {
  return guarded([&] { SK_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault)); });
}

extern "C" sk_status sk_host_unregister(void* p) {
  return guarded([&] { SK_CUDA(cudaHostUnregister(p)); });
}

// ==== dense =======================================================================

extern "C" sk_status sk_dense_create(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                     float fillv, sk_dense** out) {
  return guarded([&] {
    require_ctx(ctx);
    sk_dense* d = new_dense(ctx, rows, cols);
    fill(ctx, d->d, d->elems(), fillv);
    *out = d;
  });
}

extern "C" sk_status sk_dense_upload(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                     const float* host, sk_dense** out) {
  return guarded([&] {
    require_ctx(ctx);
    sk_dense* d = new_dense(ctx, rows, cols);
    if (d->elems())
      SK_CUDA(cudaMemcpyAsync(d->d, host, d->elems() * sizeof(float),
                              cudaMemcpyHostToDevice, ctx->stream));
    *out = d;
  });
}

extern "C" sk_status sk_dense_write(sk_ctx* ctx, sk_dense* d, const float* host) {
  return guarded([&] {
    require_ctx(ctx);
    d->version += 1;  // invalidates derived copies (K4's packed operand)
    if (d->elems())
      SK_CUDA(cudaMemcpyAsync(d->d, host, d->elems() * sizeof(float),
                              cudaMemcpyHostToDevice, ctx->stream));
  });
}

extern "C" sk_status sk_dense_download(sk_ctx* ctx, const sk_dense* d, float* host) {
  return guarded([&] {
    require_ctx(ctx);
    if (d->elems())
      SK_CUDA(cudaMemcpyAsync(host, d->d, d->elems() * sizeof(float),
                              cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  });
}

extern "C" sk_status sk_dense_download_async(sk_ctx* ctx, const sk_dense* d, float* host) {
  return guarded([&] {
    require_ctx(ctx);
    if (d->elems())
      SK_CUDA(cudaMemcpyAsync(host, d->d, d->elems() * sizeof(float),
                              cudaMemcpyDeviceToHost, ctx->stream));
  });
}

extern "C" sk_status sk_dense_shape(const sk_dense* d, uint32_t* rows, uint32_t* cols) {
  return guarded([&] {
    if (rows) *rows = d->rows;
    if (cols) *cols = d->cols;
  });
}

extern "C" float* sk_dense_device_ptr(const sk_dense* d) { return d ? d->d : nullptr; }

extern "C" sk_status sk_dense_identity(sk_ctx* ctx, uint32_t n, sk_dense** out) {
  return guarded([&] {
    require_ctx(ctx);
    sk_dense* d = new_dense(ctx, n, n);
    fill(ctx, d->d, d->elems(), 0.0f);
    if (n) SK_LAUNCH(k_identity, ceil_div(n, 256), 256, 0, ctx->stream, d->d, n);
    *out = d;
  });
}

extern "C" sk_status sk_dense_free(sk_dense* d) {
  return guarded([&] {
    if (!d) return;
    dfree(d->ctx, d->d);
    if (d->pack.buf) dfree(d->ctx, d->pack.buf);
    delete d;
  });
}

// ==== CSR =========================================================================

extern "C" sk_status sk_csr_shape(const sk_csr* a, uint32_t* rows, uint32_t* cols,
                                  size_t* nnz) {
  return guarded([&] {
    if (rows) *rows = a->rows;
    if (cols) *cols = a->cols;
    if (nnz) *nnz = a->nnz;
  });
}

extern "C" sk_status sk_csr_extract(sk_ctx* ctx, const sk_csr* a, uint32_t* rp,
                                    uint32_t* ci, float* v) {
  return guarded([&] {
    csr_ready(ctx, a);
    require_ctx(ctx);
    if (rp)
      SK_CUDA(cudaMemcpyAsync(rp, a->rp, (size_t(a->rows) + 1) * 4,
                              cudaMemcpyDeviceToHost, ctx->stream));
    if (ci && a->nnz)
      SK_CUDA(cudaMemcpyAsync(ci, a->ci, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (v && a->nnz)
      SK_CUDA(cudaMemcpyAsync(v, a->v, a->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  });
}

extern "C" sk_status sk_csr_free(sk_csr* a) {
  return guarded([&] { csr_release(a); });
}

// ==== model ===========================================================================

extern "C" sk_status sk_model_create(sk_ctx* ctx, uint32_t layers,
                                     const sk_csr* const* weights,
                                     const float* const* biases, sk_model** out) {
  return guarded([&] {
    require_ctx(ctx);
    // dnn.cpp:23-51
    if (layers == 0) fail(SK_ERR_INVALID_ARGUMENT, "model must have at least one layer");
    if (!biases)
      fail(SK_ERR_INVALID_ARGUMENT, "model has " + std::to_string(layers) +
                                        " weight matrices but 0 bias vectors");
    const uint32_t m = weights[0]->rows;
    for (uint32_t k = 0; k < layers; ++k) {
      const sk_csr* w = weights[k];
      csr_ready(ctx, w);
      if (w->rows != m || w->cols != m)
        fail(SK_ERR_DIMENSION, "layer " + std::to_string(k) + " weight is " +
                                   dim_string(w->rows, w->cols) + "; all layers must be " +
                                   dim_string(m, m));
      if (!biases[k])
        fail(SK_ERR_DIMENSION, "layer " + std::to_string(k) + " bias length 0 does not match " +
                                   std::to_string(m) + " neurons");
    }
    auto* md = new sk_model;
    md->ctx = ctx;
    md->layers = layers;
    md->neurons = m;
    md->bias_host.resize(size_t(layers) * m);
    md->bias_nonpos.resize(layers);
    md->bias_negmin.resize(layers);
    for (uint32_t k = 0; k < layers; ++k) {
      auto* w = const_cast<sk_csr*>(weights[k]);
      w->refs.fetch_add(1);
      md->w.push_back(w);
      std::memcpy(md->bias_host.data() + size_t(k) * m, biases[k], size_t(m) * 4);
      bool nonpos = true;
      double negmin = INFINITY;
      for (uint32_t i = 0; i < m; ++i) {
        const float bi = biases[k][i];
        nonpos &= (bi <= 0.0f);
        if (bi <= 0.0f) negmin = std::min(negmin, -double(bi));
      }
      md->bias_nonpos[k] = nonpos;
      md->bias_negmin[k] = negmin;
    }
    md->bias = dalloc<float>(ctx, md->bias_host.size());
    SK_CUDA(cudaMemcpyAsync(md->bias, md->bias_host.data(), md->bias_host.size() * 4,
                            cudaMemcpyHostToDevice, ctx->stream));
    sync(ctx);  // host bias copy may be released by the caller
    *out = md;
  });
}

extern "C" sk_status sk_model_shape(const sk_model* m, uint32_t* layers, uint32_t* neurons) {
  return guarded([&] {
    if (layers) *layers = m->layers;
    if (neurons) *neurons = m->neurons;
  });
}

extern "C" sk_status sk_model_free(sk_model* m) {
  return guarded([&] {
    if (!m) return;
    for (sk_csr* w : m->w) csr_release(w);
    dfree(m->ctx, m->bias);
    dfree(m->ctx, m->d_wptr);
    dfree(m->ctx, m->d_wstats);
    dfree(m->ctx, m->d_bias_nonpos);
    dfree(m->ctx, m->d_nonpos_run);
    for (sk_csr* t : m->wT) csr_release(t);
    delete m;
  });
}

// ==== DNN: dense activations ===========================================================

static float opt_clip(const sk_fwd_opts* o) { return o ? o->clip : 0.0f; }

static void require_input(uint32_t neurons, const sk_dense* y) {
  // dnn.cpp:55-61
  if (y->rows != neurons || y->cols < 1)
    fail(SK_ERR_DIMENSION, "input batch is " + dim_string(y->rows, y->cols) + ", expected " +
                               std::to_string(neurons) + " rows and n >= 1 columns");
}

extern "C" sk_status sk_layer_step(sk_ctx* ctx, const sk_csr* w, const float* bias,
                                   const sk_dense* y, const sk_fwd_opts* opt,
                                   sk_dense** out) {
  return guarded([&] {
    csr_ready(ctx, w);
    require_ctx(ctx);
    // dnn.cpp:89-98
    if (w->cols != y->rows)
      fail(SK_ERR_DIMENSION, "weight is " + dim_string(w->rows, w->cols) + " but input has " +
                                 std::to_string(y->rows) + " rows");
    if (!bias)
      fail(SK_ERR_DIMENSION, "bias length 0 does not match " + std::to_string(w->rows) +
                                 " output rows");
    float* db = dalloc<float>(ctx, w->rows);
    upload_staged(ctx, db, bias, size_t(w->rows) * 4);  // the host bias is only lent
    sk_dense* o = new_dense(ctx, w->rows, y->cols);
    timing_mark(ctx, SK_KT_SPMM);  // K1 is the layer's only kernel (measurement hook)
    launch_layer_dense(ctx, w, db, y->d, y->cols, opt_clip(opt), o->d);
    timing_mark(ctx);
    dfree(ctx, db);
    *out = o;
  });
}

static sk_dense* forward_dense(sk_ctx* ctx, const sk_model* m, const sk_dense* y0,
                               float clip) {
  require_input(m->neurons, y0);
  const uint32_t n = y0->cols;
  sk_dense* a = new_dense(ctx, m->neurons, n);
  sk_dense* b = m->layers > 1 ? new_dense(ctx, m->neurons, n) : nullptr;
  // one persistent launch for all layers; layer k writes buffer k & 1
  dense_forward_engine(ctx, m, 0, y0->d, n, clip, a->d, b ? b->d : nullptr);
  sk_dense* result = ((m->layers - 1) & 1) ? b : a;
  sk_dense* spare = (result == a) ? b : a;
  if (spare) sk_dense_free(spare);
  return result;
}

extern "C" sk_status sk_relu_forward(sk_ctx* ctx, const sk_model* m, const sk_dense* y0,
                                     const sk_fwd_opts* opt, sk_dense** out) {
  return guarded([&] {
    require_ctx(ctx);
    *out = forward_dense(ctx, m, y0, opt_clip(opt));
  });
}

extern "C" sk_status sk_relu_forward_host(sk_ctx* ctx, const sk_model* m, uint32_t n,
                                          const float* y0, const sk_fwd_opts* opt,
                                          float* yL) {
  return guarded([&] {
    require_ctx(ctx);
    sk_dense in;
    in.ctx = ctx;
    in.rows = m->neurons;
    in.cols = n;
    in.d = dalloc<float>(ctx, in.elems());
    SK_CUDA(cudaMemcpyAsync(in.d, y0, in.elems() * 4, cudaMemcpyHostToDevice, ctx->stream));
    sk_dense* r = forward_dense(ctx, m, &in, opt_clip(opt));
    SK_CUDA(cudaMemcpyAsync(yL, r->d, r->elems() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    dfree(ctx, in.d);
    sk_dense_free(r);
    sync(ctx);
  });
}

extern "C" sk_status sk_relu_forward_sparse(sk_ctx* ctx, const sk_model* m, const sk_csr* y0,
                                            const sk_fwd_opts* opt, sk_csr** out,
                                            uint64_t* nnz_trace) {
  return guarded([&] {
    csr_ready(ctx, y0);
    require_ctx(ctx);
    if (y0->rows != m->neurons || y0->cols < 1)
      fail(SK_ERR_DIMENSION, "input batch is " + dim_string(y0->rows, y0->cols) +
                                 ", expected " + std::to_string(m->neurons) +
                                 " rows and n >= 1 columns");
    *out = sparse_forward_impl(ctx, m, y0, opt_clip(opt), nnz_trace);
  });
}

extern "C" uint64_t sk_layer_seed(uint64_t seed, uint32_t layer) {
  return splitmix_at(seed, 1000ull + layer);
}

extern "C" sk_status sk_sparse_layer(sk_ctx* ctx, const sk_csr* w, const float* bias,
                                     const sk_csr* y, float clip, sk_csr** out) {
  return guarded([&] {
    csr_ready(ctx, w);
    csr_ready(ctx, y);
    require_ctx(ctx);
    if (w->cols != y->rows)
      fail(SK_ERR_DIMENSION, "weight is " + dim_string(w->rows, w->cols) + " but input has " +
                                 std::to_string(y->rows) + " rows");
    if (!bias)
      fail(SK_ERR_DIMENSION, "bias length 0 does not match " + std::to_string(w->rows) +
                                 " output rows");
    float* db = dalloc<float>(ctx, w->rows);
    SK_CUDA(cudaMemcpyAsync(db, bias, size_t(w->rows) * 4, cudaMemcpyHostToDevice, ctx->stream));
    uint64_t dense_rows = 0;  // rows whose untouched positions survive: 0 + b_i > 0 or NaN
    double negmin = INFINITY;  // min of -b_i over b_i <= 0 (the order-free path's threshold)
    for (uint32_t i = 0; i < w->rows; ++i) {
      dense_rows += !(bias[i] <= 0.0f);
      if (bias[i] <= 0.0f) negmin = std::min(negmin, -double(bias[i]));
    }
    sk_csr* o = sparse_layer_impl(ctx, w, db, y, clip, dense_rows, negmin);
    dfree(ctx, db);
    sync(ctx);
    *out = o;
  });
}

extern "C" sk_status sk_sparse_layer_dev(sk_ctx* ctx, const sk_csr* w, const float* d_bias,
                                         uint64_t dense_rows, double negmin, const sk_csr* y,
                                         float clip, sk_csr** out) {
  return guarded([&] {
    csr_ready(ctx, w);
    csr_ready(ctx, y);
    require_ctx(ctx);
    if (w->cols != y->rows)
      fail(SK_ERR_DIMENSION, "weight is " + dim_string(w->rows, w->cols) + " but input has " +
                                 std::to_string(y->rows) + " rows");
    if (!d_bias && w->rows)
      fail(SK_ERR_DIMENSION, "bias length 0 does not match " + std::to_string(w->rows) +
                                 " output rows");
    *out = sparse_layer_impl(ctx, w, d_bias, y, clip, dense_rows, negmin);
  });
}

struct sk_staged {
  sk::StagedLayer* st;
};

extern "C" sk_status sk_sparse_layer_stage(sk_ctx* ctx, const sk_csr* w, const float* d_bias,
                                           uint64_t dense_rows, double negmin, const sk_csr* y,
                                           float clip, sk_staged** out, uint64_t* nnz) {
  return guarded([&] {
    csr_ready(ctx, w);
    csr_ready(ctx, y);
    require_ctx(ctx);
    if (w->cols != y->rows)
      fail(SK_ERR_DIMENSION, "weight is " + dim_string(w->rows, w->cols) + " but input has " +
                                 std::to_string(y->rows) + " rows");
    if (!d_bias && w->rows)
      fail(SK_ERR_DIMENSION, "bias length 0 does not match " + std::to_string(w->rows) +
                                 " output rows");
    StagedLayer* st = stage_new(ctx);
    try {
      sparse_layer_impl(ctx, w, d_bias, y, clip, dense_rows, negmin, st);
    } catch (...) {
      stage_free(st);
      throw;
    }
    *nnz = stage_nnz(st);
    *out = new sk_staged{st};
  });
}

extern "C" sk_status sk_staged_publish(sk_ctx* ctx, sk_staged* st, uint32_t ndst,
                                       uint32_t* const* dst_rp, uint32_t* const* dst_ci,
                                       float* const* dst_v, uint32_t row_off, uint64_t nnz_off,
                                       int write_last) {
  return guarded([&] {
    require_ctx(ctx);
    if (!st) fail(SK_ERR_INVALID_ARGUMENT, "null staged layer");
    if (ndst > 8) fail(SK_ERR_INVALID_ARGUMENT, "at most 8 destinations (one NVLink box)");
    if (nnz_off + stage_nnz(st->st) > 0xFFFFFFFFull)
      fail(SK_ERR_INVALID_ARGUMENT, "exchange exceeds the 32-bit index range");
    try {
      stage_publish(st->st, ndst, dst_rp, dst_ci, dst_v, row_off, nnz_off, write_last);
    } catch (...) {
      stage_free(st->st);
      delete st;
      throw;
    }
    stage_free(st->st);  // (stream-ordered: the spans are reused only by later work)
    delete st;
  });
}

extern "C" sk_status sk_staged_free(sk_staged* st) {
  return guarded([&] {
    if (!st) return;
    stage_free(st->st);
    delete st;
  });
}

extern "C" sk_status sk_csr_device_arrays(const sk_csr* a, uint32_t** rp, uint32_t** ci,
                                          float** v) {
  return guarded([&] {
    if (a && a->ready) SK_CUDA(cudaEventSynchronize(a->ready));  // no stream to order
    if (rp) *rp = a->rp;
    if (ci) *ci = a->ci;
    if (v) *v = a->v;
  });
}

extern "C" sk_status sk_csr_from_device(sk_ctx* ctx, uint32_t rows, uint32_t cols, size_t nnz,
                                        const uint32_t* rp, const uint32_t* ci, const float* v,
                                        sk_csr** out) {
  return guarded([&] {
    require_ctx(ctx);
    sk_csr* a = new_csr(ctx, rows, cols, nnz);
    SK_CUDA(cudaMemcpyAsync(a->rp, rp, (size_t(rows) + 1) * 4, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    if (nnz) {
      SK_CUDA(cudaMemcpyAsync(a->ci, ci, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      SK_CUDA(cudaMemcpyAsync(a->v, v, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    *out = a;
  });
}

extern "C" sk_status sk_memcpy_d2d(sk_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    require_ctx(ctx);
    if (bytes) SK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  });
}
