/* sk_api.h -- C-ABI of the B200-native sparse-DNN engine (libsk_b200.so).
 *
 * Drop-in boundary for the hot path of the reference library `semikern`
 * (/root/reference/proj).  The reference exposes a C++ value-type API in
 * namespace semikern; this header is the plain-C surface a binding (ctypes,
 * cgo, JNI, or the header-only C++ shim include/semikern_b200/semikern.hpp)
 * links against.  Every entry point cites the reference interface it replaces.
 *
 * Conventions
 *  - Orientation is the reference's: a weight matrix W_ref is m-by-m CSR whose
 *    row i lists the in-edges of output neuron i; activations Y are m-by-n
 *    neuron-major (neurons x samples), row-major (dnn.hpp:24-25).
 *  - Storage is the reference's: u32 row_ptr[rows+1], u32 col_idx[nnz] strictly
 *    increasing per row, f32 values[nnz] (matrix.hpp:29,74-116).
 *  - Handles (sk_csr, sk_dense, sk_model) own device memory and are immutable
 *    after creation, like the reference's value types; the caller frees every
 *    handle it receives.  Operations allocate new output handles.
 *  - Work is stream-ordered on the context's CUDA stream.  Calls that return
 *    host data (downloads, counts, error checks) synchronise that stream.
 *  - Errors: every call returns sk_status; sk_last_error() gives a
 *    thread-local message.  The codes map 1:1 onto the reference's exception
 *    classes (error.hpp:24-58): DIMENSION -> DimensionError, DOMAIN ->
 *    DomainError (raised from inside a kernel via a device error word),
 *    INVALID_ARGUMENT -> InvalidArgument, ERROR -> Error.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns SK_ERR_CUDA.
 */
#ifndef SK_API_H
#define SK_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sk_status {
  SK_OK = 0,
  SK_ERR = 1,                  /* semikern::Error */
  SK_ERR_DIMENSION = 2,        /* semikern::DimensionError */
  SK_ERR_DOMAIN = 3,           /* semikern::DomainError */
  SK_ERR_INVALID_ARGUMENT = 4, /* semikern::InvalidArgument */
  SK_ERR_PARSE = 5,            /* semikern::ParseError (Matrix Market reader) */
  SK_ERR_OOM = 6,              /* device allocation failed (cf. SkippedRun, bench.hpp:64-79) */
  SK_ERR_CUDA = 7              /* CUDA runtime failure / no device */
} sk_status;

/* Order of semikern::SemiringKind (semiring.hpp:34). */
typedef enum sk_semiring {
  SK_ARITHMETIC = 0,
  SK_MAX_PLUS = 1,
  SK_MIN_MAX = 2,
  SK_GF2 = 3
} sk_semiring;

typedef struct sk_ctx sk_ctx;
typedef struct sk_csr sk_csr;
typedef struct sk_dense sk_dense;
typedef struct sk_model sk_model;

/* Options of a forward pass; mirrors semikern::ForwardOptions (dnn.hpp:49-56)
 * plus the BASELINE clip.  `workers` is accepted and ignored: the GPU result is
 * bitwise independent of it, as the reference guarantees (dnn.hpp:75-76).
 * `clip` > 0 clamps activations from above after the ReLU (Graph-Challenge
 * style, BASELINE cfg3-5); 0 disables it (the reference has no clip). */
typedef struct sk_fwd_opts {
  int workers;
  int materialize_bias;
  float clip;
} sk_fwd_opts;

/* ---- library / context ------------------------------------------------- */
const char* sk_last_error(void);
const char* sk_version(void);
/* Number of kernel launches this process has issued through the library. */
uint64_t sk_kernel_launch_count(void);

sk_status sk_ctx_create(int device, sk_ctx** out);
sk_status sk_ctx_destroy(sk_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL = own. */
sk_status sk_ctx_set_stream(sk_ctx* ctx, void* cuda_stream);
void* sk_ctx_stream(const sk_ctx* ctx);
sk_status sk_ctx_synchronize(sk_ctx* ctx);
/* Measurement hook (no reference counterpart): when enabled, the library
 * records a CUDA-event pair on the context stream around every launch of the
 * dominant kernel (the per-layer SpGEMM / SpMM); sk_ctx_kernel_times returns
 * their durations in ms (synchronising) and resets the list. */
sk_status sk_ctx_set_timing(sk_ctx* ctx, int enable);
sk_status sk_ctx_kernel_times(sk_ctx* ctx, float* ms, size_t cap, size_t* count);
/* Same, plus which kernel each timed launch was (SK_KT_*). */
enum { SK_KT_OTHER = 0, SK_KT_EXACT = 1, SK_KT_ENGINE = 2, SK_KT_DENSE_ENGINE = 3,
       SK_KT_SPMM = 4, SK_KT_GEMM_TC = 5, SK_KT_SPGEMM = 6, SK_KT_PUSH = 7,
       SK_KT_STREAM = 8 };
sk_status sk_ctx_kernel_times_tagged(sk_ctx* ctx, float* ms, int* tags, size_t cap,
                                     size_t* count);

/* Stream stopwatch for callers that time whole API calls on the device (the
 * C++ shim's run_sweep, bench.cpp time_step analogue): start records an event
 * on the context's stream, stop records a second one, waits for it and
 * returns the milliseconds between them. */
sk_status sk_ctx_timer_start(sk_ctx* ctx);
sk_status sk_ctx_timer_stop(sk_ctx* ctx, float* ms);

/* With timing enabled, the sparse engine writes %globaltimer (ns) at the start
 * (entry 0) and at the end of every layer (entry k+1) of the last forward. */
sk_status sk_ctx_layer_stamps(sk_ctx* ctx, long long* ns, size_t n);
/* The path each layer of the last sparse forward (sk_relu_forward_sparse) took,
 * one code per layer: SK_PATH_EMPTY (empty input, every bias <= 0: no work),
 * SK_PATH_EXACT (order-free fixed-point layer), SK_PATH_ESC (expand-sort-
 * compress), SK_PATH_ENGINE (windowed sparse engine), SK_PATH_DENSE (dense
 * engine after the density switch).  Introspection only; results are bitwise
 * the same on every path.  No reference counterpart. */
enum { SK_PATH_EMPTY = 0, SK_PATH_EXACT = 1, SK_PATH_ESC = 2, SK_PATH_ENGINE = 3, SK_PATH_DENSE = 4 };
sk_status sk_ctx_layer_paths(sk_ctx* ctx, unsigned char* paths, size_t n);
/* Density-adaptive sparse forward (sk_relu_forward_sparse): the activations
 * move to the dense engine when a layer's output holds more than
 * dense_above * m * n entries and back to the sparse engine below
 * sparse_below * m * n.  Results are bitwise identical either way (the switch
 * is only taken when every weight is finite).  dense_above <= 0 disables it.
 * Defaults 1/32 and 1/128.  No reference counterpart (the reference's
 * activation type is fixed by the caller, dnn.hpp:77-78). */
sk_status sk_ctx_set_density_switch(sk_ctx* ctx, double dense_above, double sparse_below);
/* Per-context kernel selection (no reference counterpart; the reference has a
 * single code path).  Every choice computes the same ascending fold bit for
 * bit, so these only select WHICH kernel variant runs -- the parity tests force
 * each one.  0 in any integer field means "automatic" (the default).
 *   exact          1 (default) provably exact layers take the order-free kernel
 *                  (k_exact_layer); -1 never (windowed engine / ESC instead)
 *   exact_kernel   1 the generic k_exact_layer; 2 the specialised kernel
 *                  (taken only where its preconditions hold: 1024-sample
 *                  windows, constant increment, four 8-bit fields, every bias
 *                  <= 0 -- otherwise the generic kernel runs); 3 the
 *                  sample-major push kernel k_push_layer (where it applies:
 *                  constant positive products, every bias <= 0, 8-bit
 *                  counters of all out-neurons within 64 KB, a model layer;
 *                  measured slower than the windowed kernels, so never
 *                  automatic); 4 the specialised kernel with flattened
 *                  products instead of piece records (measured slower; where
 *                  the specialised kernel applies); 5 the stream kernel
 *                  k_exact_stream (K7: a row's in-edge slices bulk-copied into
 *                  shared memory per pass, where the specialised kernel's
 *                  preconditions hold and Y's column array is 16-byte aligned);
 *                  0 = the stream kernel where it applies, else the generic one
 *   exact_group    4, 8, 16, 32 or 64 windows per exact-layer work item (the
 *                  stream kernel: 1, 2, 4, 8 or 16 windows per pass)
 *   exact_records  64 or 192 piece records per batch (the stream kernel: a
 *                  staging buffer of 4x that many 16-byte units)
 *   window_log2    8..12: sample window of the windowed engine (default 10)
 *   exact_window_log2  8..12: sample window of the exact layer (default 10)
 *   esc            1 (default) thin layers take expand-sort-compress; -1 never
 *   esc_ratio      products per (row, window) below which ESC applies
 *                  (<= 0: default 8)
 *   exact_fields   the stream kernel's counter width: 4 or 8 bits (0: 4 where
 *                  the threshold and increment allow it; a 4-bit counter that
 *                  wraps makes the layer rerun with 8-bit ones)
 *   exact_layout   the stream kernel's view of Y: 1 a padded copy (rows
 *                  16-byte aligned); 2 its own column array where that is
 *                  16-byte aligned (a pass table and two side units per row are
 *                  built; else the copy); 3 the padded copy with every pass
 *                  slice's entries in accumulator-bank order (<= 8 passes, else
 *                  1; fewer shared-memory bank conflicts in the counter
 *                  atomics, measured not worth the sort: DESIGN.md K7);
 *                  0 = 2 for rows of > 96 entries on average, else 1 */
typedef struct sk_tuning {
  int exact;
  int exact_kernel;
  int exact_group;
  int exact_records;
  int window_log2;
  int exact_window_log2;
  int esc;
  double esc_ratio;
  int exact_fields;
  int exact_layout;
} sk_tuning;
sk_status sk_ctx_set_tuning(sk_ctx* ctx, const sk_tuning* t);
sk_status sk_ctx_get_tuning(const sk_ctx* ctx, sk_tuning* t);
/* What the last exact-layer launch on this context ran (introspection for the
 * parity tests): launches = exact-layer launches since the context was created;
 * kernel 1 generic / 2 specialised / 3 push / 4 flat / 5 stream; group = windows per item
 * (stream: per pass); records = piece records per batch (stream: 16-byte staging units); window_log2; fields = accumulator fields per word. */
typedef struct sk_exact_info {
  uint64_t launches;
  int kernel;
  int group;
  int records;
  int window_log2;
  int fields;
  int wraps;  /* stream kernel: launches rerun with 8-bit fields after a 4-bit one wrapped */
  int layout; /* stream kernel: 0 Y read in place, 1 the padded copy */
} sk_exact_info;
sk_status sk_ctx_last_exact(const sk_ctx* ctx, sk_exact_info* info);
/* Page-lock / unlock a caller host buffer for async copies. */
sk_status sk_host_register(void* p, size_t bytes);
sk_status sk_host_unregister(void* p);

/* ---- dense matrices (semikern::DenseMatrix, matrix.hpp:39-72) ----------- */
sk_status sk_dense_create(sk_ctx* ctx, uint32_t rows, uint32_t cols, float fill,
                          sk_dense** out);
sk_status sk_dense_upload(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                          const float* host, sk_dense** out);
/* Copy into an existing handle of the same shape (stream-ordered). */
sk_status sk_dense_write(sk_ctx* ctx, sk_dense* d, const float* host);
sk_status sk_dense_download(sk_ctx* ctx, const sk_dense* d, float* host);
/* Stream-ordered download; the caller synchronises. */
sk_status sk_dense_download_async(sk_ctx* ctx, const sk_dense* d, float* host);
sk_status sk_dense_shape(const sk_dense* d, uint32_t* rows, uint32_t* cols);
float* sk_dense_device_ptr(const sk_dense* d);
sk_status sk_dense_identity(sk_ctx* ctx, uint32_t n, sk_dense** out);
sk_status sk_dense_free(sk_dense* d);

/* ---- CSR matrices (semikern::CsrMatrix, matrix.hpp:74-116) ------------ */
/* csr_from_triples (matrix.hpp:144-150, matrix.cpp:145-189): any order; exact
 * 0.0 values dropped; out-of-range index or duplicate coordinate ->
 * SK_ERR_INVALID_ARGUMENT with the reference's message. Host triples. */
sk_status sk_csr_from_triples(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                              const uint32_t* row, const uint32_t* col,
                              const float* val, size_t n, sk_csr** out);
/* Validating (validate=1, matrix.cpp:89-119) or trusted (validate=0,
 * from_parts_unchecked, matrix.cpp:76-87) construction from host arrays. */
sk_status sk_csr_from_parts(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                            const uint32_t* row_ptr, const uint32_t* col_idx,
                            const float* values, int validate, sk_csr** out);
/* Pattern-only construction (no reference counterpart; the binary activation
 * matrices of the Graph Challenge inputs and gen_input carry no information in
 * their values): the host sends row_ptr and col_idx, every stored value is
 * `value` (filled on the device). Same validation as sk_csr_from_parts. */
sk_status sk_csr_from_pattern(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                              const uint32_t* row_ptr, const uint32_t* col_idx,
                              float value, int validate, sk_csr** out);
/* sk_csr_from_pattern without validation, on a caller stream (cudaStream_t):
 * the copies run there, overlapping work queued on the context's stream, and
 * every later use of the handle is ordered after them (an event on the handle).
 * The host arrays must stay valid (and should be page-locked) until then.  For
 * double-buffered input uploads.  No reference counterpart.
 * TRUSTED INPUT ONLY: nothing checks that row_ptr is non-decreasing with
 * row_ptr[rows] = nnz, or that each row's columns are strictly increasing and
 * below `cols` (the invariants of the reference's validating CsrMatrix
 * constructor, matrix.cpp:89-119).  The kernels index shared memory by column,
 * so a violating pattern is undefined behaviour -- validate it once with
 * sk_csr_from_pattern(..., validate = 1) when its origin is not trusted. */
sk_status sk_csr_from_pattern_async(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                    const uint32_t* row_ptr, const uint32_t* col_idx,
                                    float value, void* stream, sk_csr** out);
/* sk_csr_from_pattern_async with 16-bit column indices (cols <= 65536): half
 * the bytes over the host link for the activation patterns of batches up to
 * 65536 samples (the bench's 60000-sample inputs: 31.4 MB instead of 62.9 MB per
 * upload); widened to the handle's 32-bit column array on the device, on the
 * same stream.  Same trusted-input contract.  No reference counterpart. */
sk_status sk_csr_from_pattern16_async(sk_ctx* ctx, uint32_t rows, uint32_t cols,
                                      const uint32_t* row_ptr, const uint16_t* col_idx,
                                      float value, void* stream, sk_csr** out);
sk_status sk_csr_shape(const sk_csr* a, uint32_t* rows, uint32_t* cols,
                       size_t* nnz);
/* extractTuples / span accessors (matrix.hpp:99-108): D2H copy of the three
 * arrays; any pointer may be NULL. */
sk_status sk_csr_extract(sk_ctx* ctx, const sk_csr* a, uint32_t* row_ptr,
                         uint32_t* col_idx, float* values);
sk_status sk_csr_free(sk_csr* a);

/* to_dense (matrix.hpp:154-155), from_dense = select(!= 0) (matrix.hpp:158),
 * nnz (matrix.hpp:161). */
sk_status sk_to_dense(sk_ctx* ctx, const sk_csr* a, float ambient_zero,
                      sk_dense** out);
sk_status sk_from_dense(sk_ctx* ctx, const sk_dense* d, sk_csr** out);
sk_status sk_dense_nnz(sk_ctx* ctx, const sk_dense* d, size_t* out);

/* ---- element-wise (matrix.hpp:181-191; union semantics matrix.cpp:253-312) */
sk_status sk_ewise_dense(sk_ctx* ctx, int mul, const sk_dense* a,
                         const sk_dense* b, sk_semiring s, sk_dense** out);
sk_status sk_ewise_csr(sk_ctx* ctx, int mul, const sk_csr* a, const sk_csr* b,
                       sk_semiring s, sk_csr** out);
/* sparse (op) dense -> dense; sparse_is_left selects operand order. */
sk_status sk_ewise_mixed(sk_ctx* ctx, int mul, const sk_csr* sp,
                         const sk_dense* dn, int sparse_is_left, sk_semiring s,
                         sk_dense** out);

/* ---- mxm (matrix.hpp:202-218) ----------------------------------------- */
sk_status sk_mxm_csr_dense(sk_ctx* ctx, const sk_csr* a, const sk_dense* b,
                           sk_semiring s, sk_dense** out);
sk_status sk_mxm_dense_dense(sk_ctx* ctx, const sk_dense* a, const sk_dense* b,
                             sk_semiring s, sk_dense** out);
sk_status sk_mxm_csr_csr(sk_ctx* ctx, const sk_csr* a, const sk_csr* b,
                         sk_semiring s, sk_csr** out);
/* dense_mxm_baseline (matrix.hpp:217-218): tcgen05 tensor-core GEMM
 * (3xTF32, fp32-class accuracy; within kRelTol of the scalar product). */
sk_status sk_dense_mxm_baseline(sk_ctx* ctx, const sk_dense* a,
                                const sk_dense* b, sk_dense** out);

/* ---- DNN (dnn.hpp:31-89) ----------------------------------------------- */
/* DnnModel (dnn.hpp:31-47, dnn.cpp:23-51): L square CSR layers of one width
 * plus host bias vectors (copied).  Handles are borrowed, not consumed. */
sk_status sk_model_create(sk_ctx* ctx, uint32_t layers,
                          const sk_csr* const* weights,
                          const float* const* biases, sk_model** out);
sk_status sk_model_shape(const sk_model* m, uint32_t* layers, uint32_t* neurons);
sk_status sk_model_free(sk_model* m);

/* layer_step (dnn.hpp:66-72, dnn.cpp:86-103) as ONE fused kernel:
 * Z = W.Y (ascending-k fold) ; Z + b ; ReLU ; optional clip. Host bias. */
sk_status sk_layer_step(sk_ctx* ctx, const sk_csr* w, const float* bias,
                        const sk_dense* y, const sk_fwd_opts* opt,
                        sk_dense** out);
/* relu_forward (dnn.hpp:77-78, dnn.cpp:111-121) on dense activations. */
sk_status sk_relu_forward(sk_ctx* ctx, const sk_model* m, const sk_dense* y0,
                          const sk_fwd_opts* opt, sk_dense** out);
/* Host-to-host convenience: H2D(y0) -> relu_forward -> D2H(yL). */
sk_status sk_relu_forward_host(sk_ctx* ctx, const sk_model* m, uint32_t n,
                               const float* y0, const sk_fwd_opts* opt,
                               float* yL);
/* Sparse-activation forward (BASELINE cfg3-5): Y0 is an m-by-n CSR; every
 * layer is SpGEMM + bias + ReLU (+clip) + prune of exact zeros; result is the
 * CSR Y_L.  Values/pattern bitwise equal to the reference's
 * mxm(CsrMatrix,CsrMatrix) (matrix.cpp:452-521) followed by the layer
 * epilogue of dnn.cpp:65-103.  nnz_trace (optional, L+1 entries) receives
 * nnz(Y_k).  */
sk_status sk_relu_forward_sparse(sk_ctx* ctx, const sk_model* m,
                                 const sk_csr* y0, const sk_fwd_opts* opt,
                                 sk_csr** out, uint64_t* nnz_trace);
/* One sparse-activation layer with a RECTANGULAR weight block: W_ref rows are
 * a block of output neurons (m_blk x m), Y is m x n, the result m_blk x n.
 * Used by the column-sharded forward (each GPU owns a block of output
 * neurons, BASELINE cfg5); bias is host memory of length m_blk.  The layer
 * takes the order-free exact kernel when its partial sums are provably exact
 * (statistics of w cached on the handle), else the windowed SpGEMM; an empty
 * input with every bias <= 0 returns an empty result without a launch.
 * Bitwise the same either way. */
sk_status sk_sparse_layer(sk_ctx* ctx, const sk_csr* w, const float* bias,
                          const sk_csr* y, float clip, sk_csr** out);
/* sk_sparse_layer for callers that run the same weight block many times (the
 * column-sharded forward): the bias is already on the device (w->rows floats)
 * and its two summaries are precomputed -- dense_rows = the number of rows with
 * !(b_i <= 0) (their untouched positions survive), negmin = min over b_i <= 0
 * of -b_i (+inf when there is none).  Does not synchronise beyond what the
 * layer itself needs. */
sk_status sk_sparse_layer_dev(sk_ctx* ctx, const sk_csr* w, const float* d_bias,
                              uint64_t dense_rows, double negmin, const sk_csr* y, float clip,
                              sk_csr** out);
/* The column-sharded layer with its exchange fused into the output gather (no
 * reference counterpart; the boundary is dnn.cpp:117-119, where one layer's
 * output becomes the next one's input).  sk_sparse_layer_stage computes the
 * layer (sk_sparse_layer_dev semantics) up to its output count (*nnz) and
 * keeps the block in the context's scratch; sk_staged_publish then writes it
 * straight into `ndst` (<= 8) destinations -- entries at nnz_off, row pointers
 * at row_off shifted by nnz_off, the closing pointer when write_last -- with
 * the layer's own gather kernel (stores over NVLink into the peers' buffers),
 * and releases the staged layer; sk_staged_free releases it unpublished.  No
 * other call on the context may run between the two.  Layers that do not take
 * the order-free exact path are finished in the stage call and published from
 * the finished block. */
typedef struct sk_staged sk_staged;
sk_status sk_sparse_layer_stage(sk_ctx* ctx, const sk_csr* w, const float* d_bias,
                                uint64_t dense_rows, double negmin, const sk_csr* y, float clip,
                                sk_staged** out, uint64_t* nnz);
sk_status sk_staged_publish(sk_ctx* ctx, sk_staged* st, uint32_t ndst, uint32_t* const* dst_rp,
                            uint32_t* const* dst_ci, float* const* dst_v, uint32_t row_off,
                            uint64_t nnz_off, int write_last);
sk_status sk_staged_free(sk_staged* st);
/* Column-sharded exchange over peer memory (no reference counterpart).
 * sk_ipc_alloc: a cudaMalloc'd buffer of `bytes` and its 64-byte CUDA IPC
 * handle; sk_ipc_open maps a peer's handle (peer access over NVLink);
 * sk_ipc_close / sk_ipc_free release them.  sk_csr_publish writes the block
 * `blk` (rows [row_off, row_off + rows) of the next layer's input) into each of
 * `ndst` (<= 8) destinations with ONE kernel: col_idx / values at nnz_off, row
 * pointers at row_off shifted by nnz_off, and the closing row pointer when
 * write_last.  Stream-ordered on ctx's stream; the caller orders the readers
 * after every rank's publish (a collective barrier). */
sk_status sk_ipc_alloc(sk_ctx* ctx, size_t bytes, void** dptr, unsigned char* handle);
sk_status sk_ipc_open(sk_ctx* ctx, const unsigned char* handle, void** dptr);
sk_status sk_ipc_close(void* dptr);
sk_status sk_ipc_free(void* dptr);
sk_status sk_csr_publish(sk_ctx* ctx, const sk_csr* blk, uint32_t ndst,
                         uint32_t* const* dst_rp, uint32_t* const* dst_ci,
                         float* const* dst_v, uint32_t row_off, uint64_t nnz_off,
                         int write_last);
/* Zero-copy view of a handle's device arrays (valid while the handle lives).
 * Read-only: handles are immutable (the library caches per-matrix value
 * statistics). */
sk_status sk_csr_device_arrays(const sk_csr* a, uint32_t** row_ptr,
                               uint32_t** col_idx, float** values);
/* New handle from device arrays (copied; e.g. buffers owned by torch/NCCL). */
sk_status sk_csr_from_device(sk_ctx* ctx, uint32_t rows, uint32_t cols, size_t nnz,
                             const uint32_t* row_ptr, const uint32_t* col_idx,
                             const float* values, sk_csr** out);
/* Stream-ordered device-to-device copy on the context stream. */
sk_status sk_memcpy_d2d(sk_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Category set of a result: sorted indices of samples (columns) holding any
 * nonzero; returns the count; idx may be NULL to size. */
sk_status sk_categories_csr(sk_ctx* ctx, const sk_csr* y, uint32_t* idx,
                            size_t cap, size_t* count);
sk_status sk_categories_dense(sk_ctx* ctx, const sk_dense* y, uint32_t* idx,
                              size_t cap, size_t* count);

/* dense_layer_step / dense_relu_forward (dnn.hpp:85-89, dnn.cpp:123-149):
 * the dense comparator on tcgen05 tensor cores (3xTF32, fused bias+ReLU). */
sk_status sk_dense_layer_step(sk_ctx* ctx, const sk_dense* w, const float* bias,
                              const sk_dense* y, sk_dense** out);
sk_status sk_dense_relu_forward(sk_ctx* ctx, const sk_model* m,
                                const sk_dense* y0, sk_dense** out);

/* ---- Matrix Market exchange (matio.hpp:23-55, matio.cpp) ---------------
 * "real general" only: coordinate files yield a CSR (*kind = 0, *csr set),
 * array files a dense matrix (*kind = 1, *dense set).  The text is parsed on
 * the host with the reference's rules; the CSR is built on the device.
 * Malformed input -> SK_ERR_PARSE with "line N: <reference message>";
 * unreadable path -> SK_ERR "cannot open '<path>' for reading". */
sk_status sk_read_matrix(sk_ctx* ctx, const char* path, int* kind, sk_csr** csr,
                         sk_dense** dense);
/* read_matrix(std::istream&) analogue on an in-memory text. */
sk_status sk_read_matrix_text(sk_ctx* ctx, const char* text, size_t len, int* kind,
                              sk_csr** csr, sk_dense** dense);
/* write_matrix: exactly one of csr / dense; values as %.9g (binary32 round
 * trips).  sk_format_matrix writes into buf (NUL-terminated, truncated to
 * cap-1) and returns the full length in *len (the std::ostream overload). */
sk_status sk_write_matrix(sk_ctx* ctx, const sk_csr* csr, const sk_dense* dense,
                          const char* path);
sk_status sk_format_matrix(sk_ctx* ctx, const sk_csr* csr, const sk_dense* dense,
                           char* buf, size_t cap, size_t* len);

/* ---- BASELINE workload generators (device-side, bitwise equal to
 * oracle/sk_oracle.c) ----------------- */
/* Weight layer with exactly k nonzeros per row of W (Y.W orientation), in
 * reference orientation W_ref = W^T.  value NaN -> U[-1,1) values. */
sk_status sk_gen_layer_fixed(sk_ctx* ctx, uint32_t m, uint32_t k,
                             uint64_t layer_seed, float value, sk_csr** out);
/* Bernoulli(density) layer with U[-1,1) values (cfg2). */
sk_status sk_gen_layer_density(sk_ctx* ctx, uint32_t m, double density,
                               uint64_t layer_seed, sk_csr** out);
/* The reference's gen_weight (matgen.hpp:46, matgen.cpp:50-87) bitwise: m x m
 * CSR, entry (i,j) present with probability 1/inverse_sparsity, value
 * float(-1 + 4 u), zeros elided; GenSpec validation messages. Used by the
 * paper-style sweep (paper_1708_02937_b200/bench_sweep.py). */
sk_status sk_gen_weight(sk_ctx* ctx, uint32_t m, double inverse_sparsity,
                        uint64_t seed, sk_csr** out);
/* Dense U[0,1) neuron-major input = the reference gen_input formula. */
sk_status sk_gen_input_dense(sk_ctx* ctx, uint32_t m, uint32_t n,
                             uint64_t seed, sk_dense** out);
/* Binary input: every sample has exactly k active neurons (value 1.0);
 * neuron-major CSR m x n.  sample_offset shifts the sample counter (batch-row
 * shards generate their own slice of one global batch). */
sk_status sk_gen_input_binary(sk_ctx* ctx, uint32_t m, uint32_t n, uint32_t k,
                              uint64_t seed, uint64_t sample_offset,
                              sk_csr** out);
uint64_t sk_layer_seed(uint64_t seed, uint32_t layer);

#ifdef __cplusplus
}
#endif
#endif /* SK_API_H */
