// Internals shared by the libsk_b200 translation units.
//
// Design notes (see DESIGN.md for the full picture):
//  * Every handle remembers the context whose stream allocated it; memory is
//    stream-ordered (cudaMallocAsync / cudaFreeAsync) from the device's default
//    memory pool with an unlimited release threshold, so per-call allocations
//    are pool hits, not driver calls.
//  * Errors are reported as sk_status plus a thread-local message.  Errors a
//    kernel discovers (GF(2) domain violations) are written to a device error
//    word owned by the context and read back after the kernel, mirroring the
//    reference's exceptions thrown from inside worker threads
//    (proj/src/detail/parallel.hpp:55-70).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <climits>
#include <vector>

#include "sk_api.h"

namespace sk {

// ---- status plumbing ----------------------------------------------------------

struct Failure {
  sk_status code;
  std::string msg;
};

[[noreturn]] inline void fail(sk_status code, const std::string& msg) {
  throw Failure{code, msg};
}

void set_last_error(const std::string& msg);

#define SK_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      if (e_ == cudaErrorMemoryAllocation)                                   \
        ::sk::fail(SK_ERR_OOM, std::string("device allocation failed: ") +   \
                                   cudaGetErrorString(e_));                  \
      ::sk::fail(SK_ERR_CUDA, std::string(#call) + ": " +                    \
                                  cudaGetErrorString(e_));                   \
    }                                                                        \
  } while (0)

extern std::atomic<uint64_t> g_launches;

// Every kernel launch goes through this so the count is exact.
#define SK_LAUNCH(kernel, grid, block, smem, stream, ...)                    \
  do {                                                                       \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);              \
    ::sk::g_launches.fetch_add(1, std::memory_order_relaxed);                \
    SK_CUDA(cudaGetLastError());                                             \
  } while (0)

template <typename F>
sk_status guarded(F&& f) {
  try {
    f();
    return SK_OK;
  } catch (const Failure& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return SK_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SK_ERR;
  }
}

inline std::string dim_string(uint32_t r, uint32_t c) {
  return std::to_string(r) + "x" + std::to_string(c);
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return unsigned((a + b - 1) / b); }

}  // namespace sk

// ---- handles ------------------------------------------------------------------

struct sk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int num_sms = 148;
  size_t total_mem = 0;      // device memory size (queried once: cudaMemGetInfo takes a
                             // driver lock, so hot paths only call it when they must)
  int* d_err = nullptr;      // device error word (0 = ok)
  uint64_t* d_u64 = nullptr; // small device scratch for counters/flags (64 slots)
  uint64_t* h_u64 = nullptr; // pinned mirror of d_u64
  // Mailbox: mapped pinned host memory a one-warp kernel posts a few words into
  // (word 0 = sequence flag, payload from word kMboxHdr); the host polls the flag
  // instead of issuing device->host copies + a stream synchronise (see Fetch).
  uint32_t* mbox = nullptr;    // host address
  uint32_t* mbox_dev = nullptr;  // the same memory as the device sees it
  uint32_t mbox_seq = 0;
  // Optional per-layer timing of the dominant kernel (CUDA events recorded on
  // this stream around each layer's SpGEMM launch); see sk_ctx_set_timing.
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // 2 per layer
  std::vector<int> ev_tag;      // SK_KT_* per pair
  cudaEvent_t watch[2] = {nullptr, nullptr};  // sk_ctx_timer_start/stop
  char* pin = nullptr;                      // pinned staging ring (upload_staged)
  cudaEvent_t pin_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int pin_next = 0;
  size_t ev_used = 0;
  // Optional per-layer %globaltimer stamps written by the sparse engine.
  long long* stamps = nullptr;
  uint32_t stamps_cap = 0;
  std::vector<unsigned char> last_paths;  // per layer of the last sparse forward (SK_PATH_*)
  // Density-adaptive sparse forward: switch to the dense engine when a layer's
  // output has more than dense_above * m * n entries, back to the sparse engine
  // below sparse_below * m * n (sk_ctx_set_density_switch; dense_above <= 0 = off).
  double dense_above = 1.0 / 32;
  double sparse_below = 1.0 / 128;
  // Kernel selection (sk_ctx_set_tuning; 0 = automatic) and what the last
  // exact-layer launch ran (sk_ctx_last_exact).
  sk_tuning tune = {0, 0, 0, 0, 0, 0, 0, 0.0, 0, 0};
  sk_exact_info last_exact = {0, 0, 0, 0, 0, 0, 0, 0};
  // Grow-only scratch arena for the temporaries of one forward call (window
  // tables, item counts, scratch spans, ping-pong buffers): per-call pool
  // allocations of ~1 GB cost milliseconds of host time with the GPU idle.
  // Reuse is stream-ordered (set_stream synchronises the previous stream).
  uint8_t* arena = nullptr;
  size_t arena_cap = 0, arena_top = 0, arena_high = 0;
  int arena_depth = 0;
  std::vector<void*> arena_spill;  // overflow allocations of the current call
};

// K4's split-and-packed copy of a weight operand (tf32 hi / lo halves in the
// UMMA K-major tile layout), cached on the handle it was made from.
struct PackCache {
  float* buf = nullptr;      // hi then lo
  uint64_t version = ~0ull;  // the owner's version it was made from
};

struct sk_dense {
  sk_ctx* ctx = nullptr;
  uint32_t rows = 0, cols = 0;
  float* d = nullptr;
  size_t elems() const { return size_t(rows) * cols; }
  uint64_t version = 0;  // bumped by every in-place write (sk_dense_write)
  PackCache pack;        // as K4's A operand (dense_mxm_baseline / dense_layer_step)
};

// Per-matrix value statistics (the exactness test of the sparse engine): the
// smallest power of two every nonzero value is a multiple of ("granularity",
// lowbit exponent), the smallest e with |v| < 2^e, non-finite values, the
// longest row, and the min/max value bit patterns (equal: constant values).
struct ValueStats {
  int lowbit;     // min over nonzero values
  int ehi;        // max over nonzero values
  int nonfinite;  // any Inf/NaN
  int maxdeg;     // max stored entries per row (weights only)
  unsigned int vmin, vmax;  // min / max bit pattern over all stored values (equal: constant)
  unsigned int absmax;      // bit pattern of max |v| over finite values
  unsigned int rowsum;      // weights: bit pattern of an upper bound on max_i sum_k |w_ik|
};
#define SK_VALUESTATS_INIT {INT_MAX, INT_MIN, 0, 0, 0xFFFFFFFFu, 0u, 0u, 0u}

// Value statistics of a constant-valued matrix (every one of nnz stored values
// is c), on the host: the same rules as the device reduction (k_value_stats).
ValueStats const_value_stats(float c, size_t nnz);

// Every CSR column array carries kCiPad words of slack after its nnz entries,
// so a kernel may read the aligned 16-byte block holding its last entries
// without leaving the allocation.  (Measured for the exact layer's piece
// gathers -- two 16-byte loads per 4-entry piece instead of four scalar ones:
// cfg4 1.085 -> 1.131 ms, cfg5 2.36 -> 2.52 ms; not used there.)
constexpr size_t kCiPad = 8;

struct sk_csr {
  sk_ctx* ctx = nullptr;
  uint32_t rows = 0, cols = 0;
  size_t nnz = 0;
  uint32_t* rp = nullptr;  // rows+1
  uint32_t* ci = nullptr;  // nnz
  float* v = nullptr;      // nnz
  std::atomic<int> refs{1};
  // value statistics, computed once (handles are immutable: the zero-copy
  // device view is read-only) or known at construction (constant values)
  bool stats_valid = false;
  ValueStats stats;
  // its statistics as a weight (value statistics + row bounds), cached likewise
  bool wstats_valid = false;
  ValueStats wstats;
  // set by the stream-asynchronous constructor: the arrays are complete once
  // this event has fired (every consumer orders its stream after it)
  cudaEvent_t ready = nullptr;
  // K1t's chunk-tiled copy of the weights (values in 64 x 32 tiles + presence
  // masks), built on first use and cached like the statistics (k_spmm.cu)
  float* tile_vals = nullptr;
  uint32_t* tile_mask = nullptr;
  // K4's packed copy of the densified weights (dense_relu_forward)
  PackCache pack;
};



struct sk_model {
  sk_ctx* ctx = nullptr;
  uint32_t layers = 0, neurons = 0;
  std::vector<sk_csr*> w;       // shared (ref-counted) layer weights
  float* bias = nullptr;        // device, layers*neurons
  std::vector<float> bias_host; // layers*neurons
  std::vector<uint8_t> bias_nonpos;  // per layer: every b <= 0 (no NaN)
  std::vector<double> bias_negmin;   // per layer: min of -b_i over b_i <= 0 (inf: none)
  const void** d_wptr = nullptr;     // device [rp[L], ci[L], v[L]] for the engine
  void* d_wstats = nullptr;          // device per-layer value statistics (exactness test)
  uint8_t* d_bias_nonpos = nullptr;
  uint32_t* d_nonpos_run = nullptr;  // per layer k: consecutive layers from k with every b <= 0
  int weights_finite = -1;           // every weight finite (-1 = not computed yet)
  std::vector<ValueStats> wstats_host;  // host copy of d_wstats
  std::vector<sk_csr*> wT;              // per layer W^T (out-edges), built on first ESC use
  size_t clu_worst = SIZE_MAX;          // K1c: largest per-CTA weight slice (SIZE_MAX: not yet)
  std::vector<uint32_t> wT_maxdeg;      // longest W^T row
};

namespace sk {

// device memory (stream-ordered)
template <typename T>
T* dalloc(sk_ctx* ctx, size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  SK_CUDA(cudaMallocAsync(&p, n * sizeof(T), ctx->stream));
  return static_cast<T*>(p);
}
void dfree(sk_ctx* ctx, void* p);

// Arena scope (nestable): arena_begin / arena_end bracket one forward call;
// aalloc memory is valid until the outermost arena_end.
void arena_begin(sk_ctx* ctx);
void arena_end(sk_ctx* ctx);
void* arena_alloc_bytes(sk_ctx* ctx, size_t bytes);
template <typename T>
T* aalloc(sk_ctx* ctx, size_t n) {
  return static_cast<T*>(arena_alloc_bytes(ctx, (n ? n : 1) * sizeof(T)));
}

sk_dense* new_dense(sk_ctx* ctx, uint32_t rows, uint32_t cols);
sk_csr* new_csr(sk_ctx* ctx, uint32_t rows, uint32_t cols, size_t nnz);
void csr_release(sk_csr* a);
// Orders ctx's stream after an asynchronously built handle's copies (no-op
// for every other handle).
inline void csr_ready(sk_ctx* ctx, const sk_csr* a) {
  if (ctx && a && a->ready) SK_CUDA(cudaStreamWaitEvent(ctx->stream, a->ready, 0));
}

// Kernel attributes are per device (each device's primary context holds its
// own copy), so the "set once" state is keyed on (kernel, device) under a
// lock; occupancy queries are driver calls and are cached on the same key.
void kernel_smem_attr(sk_ctx* ctx, const void* kernel, int bytes);
int kernel_occupancy(sk_ctx* ctx, const void* kernel, int threads, size_t smem);
template <typename K>
inline void smem_attr(sk_ctx* ctx, K* kernel, int bytes = 200 * 1024) {
  kernel_smem_attr(ctx, reinterpret_cast<const void*>(kernel), bytes);
}
template <typename K>
inline int occupancy(sk_ctx* ctx, K* kernel, int threads, size_t smem) {
  return kernel_occupancy(ctx, reinterpret_cast<const void*>(kernel), threads, smem);
}

// Reads and clears the context's device error word (synchronising).
void check_device_error(sk_ctx* ctx, const char* op);
void sync(sk_ctx* ctx);

// Small device results read back through the context's mailbox.  A bulk
// host->device copy in flight on another stream delays every small
// device->host cudaMemcpyAsync by tens of microseconds each (measured with
// tools/micro/copy_interference.py: four 4-byte copies + a synchronise 36 -> 147 us
// beside a 32 MB upload), and cudaStreamSynchronize itself by ~20 us; a store into
// mapped host memory followed by a polled flag is not.  Stream-ordered like the
// copies it replaces: the post kernel runs after everything queued before it.
constexpr uint32_t kMboxHdr = 16;        // payload offset (words)
constexpr uint32_t kMboxWords = 1 << 15; // payload capacity (words)
struct PostSrc {
  const uint32_t* p[8];
  uint32_t n[8];
  int cnt;
};
struct Fetch {
  sk_ctx* ctx;
  PostSrc s;
  explicit Fetch(sk_ctx* c) : ctx(c) { s.cnt = 0; }
  Fetch& add(const void* dev, uint32_t words);
  // launches the post kernel, waits for it, returns the payload (words in add()
  // order; valid until the context's next fetch)
  const uint32_t* run();
};
// waits until the mailbox flag shows `seq` (a failed stream raises instead of spinning)
void mbox_wait(sk_ctx* ctx, uint32_t seq);
// Record a timing event pair slot (no-op unless ctx->timing); the opening
// mark of a pair carries the kernel's SK_KT_* tag.
void timing_mark(sk_ctx* ctx, int tag = SK_KT_OTHER);
void fill(sk_ctx* ctx, float* p, size_t n, float v);

// device scan helpers (CUB, stream-ordered temp storage)
void exclusive_scan_u32(sk_ctx* ctx, const uint32_t* in, uint32_t* out, size_t n);
// Host -> device copy of a small host buffer the caller only lends for the
// call (a bias vector): staged through a pinned ring slot, so the copy is
// stream-ordered and the call returns without waiting for the device.
void upload_staged(sk_ctx* ctx, void* dst, const void* src, size_t bytes);
void exclusive_scan_u64(sk_ctx* ctx, const uint64_t* in, uint64_t* out, size_t n);

// ---- semiring op tables (semiring.hpp:63-110), device side --------------------

enum DevErr : int { kErrNone = 0, kErrGf2Domain = 1 };

#ifdef __CUDACC__  // device op tables (host-only translation units skip them)
struct OpArith {
  static constexpr int kind = SK_ARITHMETIC;
  __device__ static float zero() { return 0.0f; }
  __device__ static float add(float a, float b, int*) { return __fadd_rn(a, b); }
  __device__ static float mul(float a, float b, int*) { return __fmul_rn(a, b); }
};
struct OpMaxPlus {
  static constexpr int kind = SK_MAX_PLUS;
  __device__ static float zero() { return -__int_as_float(0x7f800000); }
  __device__ static float add(float a, float b, int*) { return a < b ? b : a; }
  __device__ static float mul(float a, float b, int*) { return __fadd_rn(a, b); }
};
struct OpMinMax {
  static constexpr int kind = SK_MIN_MAX;
  __device__ static float zero() { return __int_as_float(0x7f800000); }
  __device__ static float add(float a, float b, int*) { return b < a ? b : a; }
  __device__ static float mul(float a, float b, int*) { return a < b ? b : a; }
};
struct OpGf2 {
  static constexpr int kind = SK_GF2;
  __device__ static float zero() { return 0.0f; }
  __device__ static bool ok(float v) { return v == 0.0f || v == 1.0f; }
  __device__ static float add(float a, float b, int* err) {
    if (!ok(a) || !ok(b)) atomicCAS(err, 0, kErrGf2Domain);
    return a == b ? 0.0f : 1.0f;
  }
  __device__ static float mul(float a, float b, int* err) {
    if (!ok(a) || !ok(b)) atomicCAS(err, 0, kErrGf2Domain);
    return (a == 1.0f && b == 1.0f) ? 1.0f : 0.0f;
  }
};

template <typename F>
void dispatch_semiring(sk_semiring s, F&& f) {
  switch (s) {
    case SK_ARITHMETIC: f(OpArith{}); return;
    case SK_MAX_PLUS: f(OpMaxPlus{}); return;
    case SK_MIN_MAX: f(OpMinMax{}); return;
    case SK_GF2: f(OpGf2{}); return;
  }
  fail(SK_ERR_INVALID_ARGUMENT, "unknown semiring kind " + std::to_string(int(s)));
}

#endif  // __CUDACC__

float semiring_zero_host(sk_semiring s);

#ifdef __CUDACC__
// ---- the layer epilogue (dnn.cpp:65-103 + optional clip) -----------------------
// z = acc + b (max-plus "times"); z = z<0 ? 0 : z (max-plus "plus" with 0,
// semiring.hpp:75 -- a select, so -0.0 and NaN pass through); clip by select.
__device__ __forceinline__ float layer_epilogue(float acc, float b, float clip) {
  float z = __fadd_rn(acc, b);
  z = (z < 0.0f) ? 0.0f : z;
  if (clip > 0.0f) z = (z > clip) ? clip : z;
  return z;
}

#endif  // __CUDACC__

// ---- SplitMix64 (rng.hpp:29-62), device side ------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t idx) {
  return mix64(seed + (idx + 1) * 0x9E3779B97F4A7C15ull);
}
#ifdef __CUDACC__
__device__ __forceinline__ double to_unit(uint64_t bits) {
  return __dmul_rn((double)(bits >> 11), 0x1.0p-53);
}
#endif  // __CUDACC__

// ---- internal entry points implemented in the .cu files ------------------------
sk_csr* csr_from_device_triples(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                const uint32_t* d_r, const uint32_t* d_c,
                                const float* d_v, size_t n,
                                const uint32_t* h_r, const uint32_t* h_c,
                                uint64_t* dup_index = nullptr);
sk_csr* csr_transpose(sk_ctx* ctx, const sk_csr* a);
// Thin layers by expand-sort-compress (k_esc.cu); every bias of layer k <= 0.
bool esc_applicable(sk_ctx* ctx, const sk_model* md, uint32_t k, const sk_csr* y, double ratio);
sk_csr* esc_layer(sk_ctx* ctx, const sk_model* md, const sk_csr* y, uint32_t k, float clip);
// The tiny ESC launched before its input's entry count reaches the host
// (k_esc.cu): the count is read from *d_nnz, the entries (in any order) from
// in_row / in_col / in_val; d_cnt[0] = output entries, d_cnt[1] = 1 if handled.
bool esc_tiny_possible(const sk_model* md, uint32_t k, const sk_csr* y);
sk_csr* esc_tiny_deferred(sk_ctx* ctx, const sk_model* md, uint32_t k, uint32_t n,
                          const uint32_t* in_row, const uint32_t* in_col, const float* in_val,
                          const uint32_t* d_nnz, float clip, uint32_t* d_cnt);
void ensure_model_tables(sk_ctx* ctx, sk_model* md);
void dense_forward_engine(sk_ctx* ctx, const sk_model* md, uint32_t k0, const float* y0,
                          uint32_t n, float clip, float* buf0, float* buf1,
                          unsigned long long* nnz = nullptr, unsigned long long stop_below = 0,
                          int* d_done = nullptr);
sk_csr* from_dense_impl(sk_ctx* ctx, const float* d, uint32_t rows, uint32_t cols);
void csr_scatter_dense(sk_ctx* ctx, const sk_csr* a, float* out);
void launch_layer_dense(sk_ctx* ctx, const sk_csr* w, const float* d_bias,
                        const float* y, uint32_t n, float clip, float* out);
void launch_mxm_csr_dense(sk_ctx* ctx, const sk_csr* a, const float* b,
                          uint32_t n, sk_semiring s, float* out);
sk_csr* mxm_csr_csr_impl(sk_ctx* ctx, const sk_csr* a, const sk_csr* b,
                         sk_semiring s);
// A staged column-shard layer (k_spgemm.cu): sparse_layer_impl with `stage`
// returns nullptr and leaves the block to stage_publish.
struct StagedLayer;
sk_csr* sparse_layer_impl(sk_ctx* ctx, const sk_csr* w, const float* d_bias, const sk_csr* y,
                          float clip, uint64_t dense_rows, double negmin = INFINITY,
                          StagedLayer* stage = nullptr);
StagedLayer* stage_new(sk_ctx* ctx);
uint64_t stage_nnz(const StagedLayer* st);
void stage_publish(StagedLayer* st, uint32_t nd, uint32_t* const* rp, uint32_t* const* ci,
                   float* const* v, uint32_t row_off, uint64_t nnz_off, int write_last);
void stage_free(StagedLayer* st);
void csr_publish_impl(sk_ctx* ctx, const sk_csr* blk, uint32_t nd, uint32_t* const* rp,
                      uint32_t* const* ci, float* const* v, uint32_t row_off, uint64_t nnz_off,
                      int write_last);
sk_csr* sparse_forward_impl(sk_ctx* ctx, const sk_model* m, const sk_csr* y0,
                            float clip, uint64_t* nnz_trace);
// W^T of a model layer (out-edges), built on first use and cached (k_esc.cu).
const sk_csr* model_layer_transpose(sk_ctx* ctx, sk_model* mm, uint32_t k);
// K6 (k_push.cu): the sample-major push layer; nullptr when the counters do not fit.
size_t push_smem(uint32_t m);
sk_csr* push_layer(sk_ctx* ctx, const sk_csr* wT, const sk_csr* y, uint32_t m, const float* bias,
                   float clip, float v, uint32_t cmin);
// C = A.B (+ bias, ReLU) on tcgen05 (3xTF32).  With `cache` (owned by A's
// handle, current for `version`), A's split/pack is reused across calls.
void launch_dense_gemm_tc(sk_ctx* ctx, const float* a, const float* b,
                          uint32_t M, uint32_t K, uint32_t N, const float* bias,
                          int relu, float* c, PackCache* cache = nullptr, uint64_t version = 0);

}  // namespace sk
