/* TEST INFRASTRUCTURE ONLY -- CPU checker for the GPU path; see sk_oracle.h.
 *
 * Built with -ffp-contract=off: every a*b+c below is a separately rounded
 * multiply and add, as in the reference build.
 */
#include "sk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* Static contiguous row blocks over worker threads (the same partition idea as
 * proj/src/detail/parallel.hpp:29-43); results never depend on the count. */
static int g_threads = 0;

typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t begin, end;
} par_job;

static void* par_trampoline(void* p) {
  par_job* j = (par_job*)p;
  j->fn(j->ctx, j->begin, j->end);
  return NULL;
}

static void par_for(int64_t count, range_fn fn, void* ctx) {
  int nw = sko_threads();
  if (nw > count) nw = (int)(count > 0 ? count : 1);
  if (nw <= 1) {
    fn(ctx, 0, count);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nw);
  par_job* jobs = (par_job*)malloc(sizeof(par_job) * nw);
  for (int w = 0; w < nw; ++w) {
    jobs[w].fn = fn;
    jobs[w].ctx = ctx;
    jobs[w].begin = count * w / nw;
    jobs[w].end = count * (w + 1) / nw;
    pthread_create(&th[w], NULL, par_trampoline, &jobs[w]);
  }
  for (int w = 0; w < nw; ++w) pthread_join(th[w], NULL);
  free(th);
  free(jobs);
}

/* proj/include/semikern/rng.hpp:43-61 */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t sko_splitmix_at(uint64_t seed, uint64_t idx) {
  return mix64(seed + (idx + 1) * 0x9E3779B97F4A7C15ull);
}

double sko_to_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

/* tools/semikern_main.cpp:41-43 */
uint64_t sko_layer_seed(uint64_t seed, uint32_t layer) {
  return sko_splitmix_at(seed, 1000ull + layer);
}

static uint32_t bounded(uint64_t bits, uint32_t range) {
  return (uint32_t)(((unsigned __int128)bits * range) >> 64);
}

typedef struct {
  uint32_t cols, k;
  uint64_t seed, row_offset;
  uint32_t* out;
} fixed_ctx;

static void fixed_rows_range(void* p, int64_t begin, int64_t end) {
  const fixed_ctx* c = (const fixed_ctx*)p;
  const uint32_t cols = c->cols, k = c->k;
  const uint64_t seed = c->seed;
  uint32_t* cols_out = c->out;
  for (int64_t i = begin; i < end; ++i) {
    const uint64_t rs = sko_splitmix_at(seed, (uint64_t)i + c->row_offset);
    uint32_t* row = cols_out + (size_t)i * k;
    uint32_t have = 0;
    for (uint64_t t = 0; have < k; ++t) {
      const uint32_t c = bounded(sko_splitmix_at(rs, t), cols);
      /* binary search in the sorted prefix; insert if absent */
      uint32_t lo = 0, hi = have;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (row[mid] < c) lo = mid + 1; else hi = mid;
      }
      if (lo < have && row[lo] == c) continue;
      memmove(row + lo + 1, row + lo, (size_t)(have - lo) * sizeof(uint32_t));
      row[lo] = c;
      ++have;
    }
  }
}

void sko_gen_fixed_rows_off(uint32_t rows, uint32_t cols, uint32_t k, uint64_t seed,
                            uint64_t row_offset, uint32_t* cols_out) {
  fixed_ctx c = {cols, k, seed, row_offset, cols_out};
  par_for(rows, fixed_rows_range, &c);
}

void sko_gen_fixed_rows(uint32_t rows, uint32_t cols, uint32_t k, uint64_t seed,
                        uint32_t* cols_out) {
  sko_gen_fixed_rows_off(rows, cols, k, seed, 0, cols_out);
}

float sko_uniform_pm1(uint64_t seed, uint64_t idx) {
  const float v = (float)(-1.0 + 2.0 * sko_to_unit(sko_splitmix_at(seed, idx)));
  return v == 0.0f ? 1.0f : v;
}

void sko_csr_transpose(uint32_t rows, uint32_t cols, const uint32_t* rp,
                       const uint32_t* ci, const float* v, uint32_t* trp,
                       uint32_t* tci, float* tv) {
  memset(trp, 0, ((size_t)cols + 1) * sizeof(uint32_t));
  const size_t nnz = rp[rows];
  for (size_t e = 0; e < nnz; ++e) trp[ci[e] + 1]++;
  for (uint32_t c = 0; c < cols; ++c) trp[c + 1] += trp[c];
  uint32_t* fill = (uint32_t*)malloc(((size_t)cols + 1) * sizeof(uint32_t));
  memcpy(fill, trp, ((size_t)cols + 1) * sizeof(uint32_t));
  for (uint32_t r = 0; r < rows; ++r) {
    for (uint32_t e = rp[r]; e < rp[r + 1]; ++e) {
      const uint32_t dst = fill[ci[e]]++;
      tci[dst] = r;
      if (tv) tv[dst] = v[e];
    }
  }
  free(fill);
}

size_t sko_gen_layer_fixed(uint32_t m, uint32_t k, uint64_t layer_seed,
                           float value, uint32_t* rp, uint32_t* ci, float* v) {
  const size_t nnz = (size_t)m * k;
  uint32_t* wc = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  float* wv = (float*)malloc(nnz * sizeof(float));
  uint32_t* wrp = (uint32_t*)malloc(((size_t)m + 1) * sizeof(uint32_t));
  sko_gen_fixed_rows(m, m, k, sko_splitmix_at(layer_seed, 0), wc);
  const uint64_t vs = sko_splitmix_at(layer_seed, 1);
  const int uniform = value != value;
  for (size_t e = 0; e < nnz; ++e)
    wv[e] = uniform ? sko_uniform_pm1(vs, e) : value;
  for (uint32_t i = 0; i <= m; ++i) wrp[i] = i * k;
  sko_csr_transpose(m, m, wrp, wc, wv, rp, ci, v);
  free(wc);
  free(wv);
  free(wrp);
  return nnz;
}

size_t sko_gen_layer_density(uint32_t m, double density, uint64_t layer_seed,
                             uint32_t* rp, uint32_t* ci, float* v) {
  const uint64_t sel = sko_splitmix_at(layer_seed, 0);
  const uint64_t val = sko_splitmix_at(layer_seed, 1);
  size_t nnz = 0;
  rp[0] = 0;
  /* W_ref[j][i] = W[i][j]; entry (i,j) of W owns counter i*m+j. */
  for (uint32_t j = 0; j < m; ++j) {
    for (uint32_t i = 0; i < m; ++i) {
      const uint64_t idx = (uint64_t)i * m + j;
      if (sko_to_unit(sko_splitmix_at(sel, idx)) < density) {
        if (ci) {
          ci[nnz] = i;
          v[nnz] = sko_uniform_pm1(val, idx);
        }
        ++nnz;
      }
    }
    rp[j + 1] = (uint32_t)nnz;
  }
  return nnz;
}

/* proj/src/matgen.cpp:89-99 with stream kInput = 2 (matgen.cpp:38-43) */
typedef struct {
  uint64_t stream;
  float* y;
} input_ctx;

static void input_range(void* p, int64_t begin, int64_t end) {
  const input_ctx* c = (const input_ctx*)p;
  for (int64_t idx = begin; idx < end; ++idx)
    c->y[idx] = (float)sko_to_unit(sko_splitmix_at(c->stream, (uint64_t)idx));
}

void sko_gen_input_dense(uint32_t m, uint32_t n, uint64_t seed, float* y) {
  input_ctx c = {sko_splitmix_at(seed, 2), y};
  par_for((int64_t)m * n, input_range, &c);
}

void sko_gen_input_binary(uint32_t m, uint32_t n, uint32_t k, uint64_t seed,
                          uint64_t sample_offset, uint32_t* rp, uint32_t* ci,
                          float* v) {
  const size_t nnz = (size_t)n * k;
  uint32_t* bc = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  uint32_t* brp = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  sko_gen_fixed_rows_off(n, m, k, sko_splitmix_at(seed, 4), sample_offset, bc);
  for (uint32_t r = 0; r <= n; ++r) brp[r] = r * k;
  sko_csr_transpose(n, m, brp, bc, NULL, rp, ci, NULL);
  for (size_t e = 0; e < nnz; ++e) v[e] = 1.0f;
  free(bc);
  free(brp);
}

/* ---- layer recurrence ---- */

static inline float epilogue(float acc, float b, float clip) {
  float z = acc + b;           /* max-plus "times": proj/src/dnn.cpp:74-81 */
  z = (z < 0.0f) ? 0.0f : z;   /* max-plus "plus" with 0: semiring.hpp:75 */
  if (clip > 0.0f) z = (z > clip) ? clip : z;
  return z;
}

typedef struct {
  const uint32_t *rp, *ci;
  const float *wv, *bias, *y;
  float clip;
  uint32_t n;
  float* out;
} dense_ctx;

static void dense_range(void* p, int64_t begin, int64_t end) {
  const dense_ctx* c = (const dense_ctx*)p;
  const uint32_t *rp = c->rp, *ci = c->ci;
  const float *wv = c->wv, *bias = c->bias, *y = c->y;
  const float clip = c->clip;
  const uint32_t n = c->n;
  float* out = c->out;
  {
    float* acc = (float*)malloc((size_t)n * sizeof(float) + 4);
    for (int64_t i = begin; i < end; ++i) {
      for (uint32_t j = 0; j < n; ++j) acc[j] = 0.0f;
      for (uint32_t e = rp[i]; e < rp[i + 1]; ++e) {
        const float a = wv[e];
        const float* yrow = y + (size_t)ci[e] * n;
        for (uint32_t j = 0; j < n; ++j) acc[j] = acc[j] + a * yrow[j];
      }
      float* o = out + (size_t)i * n;
      for (uint32_t j = 0; j < n; ++j) o[j] = epilogue(acc[j], bias[i], clip);
    }
    free(acc);
  }
}

void sko_layer_dense(uint32_t m, uint32_t l, const uint32_t* rp,
                     const uint32_t* ci, const float* wv, const float* bias,
                     float clip, uint32_t n, const float* y, float* out) {
  (void)l;
  dense_ctx c = {rp, ci, wv, bias, y, clip, n, out};
  par_for(m, dense_range, &c);
}

typedef struct {
  const uint32_t *wrp, *wci;
  const float *wv, *bias;
  float clip;
  uint32_t n;
  const uint32_t *yrp, *yci;
  const float* yv;
  uint32_t** rc;
  float** rv;
  uint32_t* cnt;
} sparse_ctx;

static void sparse_range(void* p, int64_t begin, int64_t end) {
  const sparse_ctx* x = (const sparse_ctx*)p;
  const uint32_t *wrp = x->wrp, *wci = x->wci, *yrp = x->yrp, *yci = x->yci;
  const float *wv = x->wv, *bias = x->bias, *yv = x->yv;
  const float clip = x->clip;
  const uint32_t n = x->n;
  uint32_t** rc = x->rc;
  float** rv = x->rv;
  uint32_t* cnt = x->cnt;
  {
    float* acc = (float*)calloc((size_t)n + 1, sizeof(float));
    uint8_t* touched = (uint8_t*)calloc((size_t)n + 1, 1);
    for (int64_t i = begin; i < end; ++i) {
      /* Gustavson row i: ascending k, each Y row ascending samples. */
      for (uint32_t e = wrp[i]; e < wrp[i + 1]; ++e) {
        const float a = wv[e];
        const uint32_t k = wci[e];
        for (uint32_t q = yrp[k]; q < yrp[k + 1]; ++q) {
          const uint32_t s = yci[q];
          touched[s] = 1;
          acc[s] = acc[s] + a * yv[q];
        }
      }
      const float untouched = epilogue(0.0f, bias[i], clip);
      const int dense_row = untouched != 0.0f;
      uint32_t c = 0;
      uint32_t cap = 64;
      uint32_t* oc = (uint32_t*)malloc(cap * sizeof(uint32_t));
      float* ovv = (float*)malloc(cap * sizeof(float));
      for (uint32_t s = 0; s < n; ++s) {
        if (!touched[s] && !dense_row) continue;
        const float z = touched[s] ? epilogue(acc[s], bias[i], clip) : untouched;
        acc[s] = 0.0f;
        touched[s] = 0;
        if (z != 0.0f) {
          if (c == cap) {
            cap *= 2;
            oc = (uint32_t*)realloc(oc, cap * sizeof(uint32_t));
            ovv = (float*)realloc(ovv, cap * sizeof(float));
          }
          oc[c] = s;
          ovv[c] = z;
          ++c;
        }
      }
      rc[i] = oc;
      rv[i] = ovv;
      cnt[i + 1] = c;
    }
    free(acc);
    free(touched);
  }
}

size_t sko_layer_sparse(uint32_t m, uint32_t l, const uint32_t* wrp,
                        const uint32_t* wci, const float* wv, const float* bias,
                        float clip, uint32_t n, const uint32_t* yrp,
                        const uint32_t* yci, const float* yv, uint32_t** orp,
                        uint32_t** oci, float** ov) {
  (void)l;
  uint32_t** rc = (uint32_t**)calloc(m, sizeof(uint32_t*));
  float** rv = (float**)calloc(m, sizeof(float*));
  uint32_t* cnt = (uint32_t*)calloc((size_t)m + 1, sizeof(uint32_t));
  sparse_ctx x = {wrp, wci, wv, bias, clip, n, yrp, yci, yv, rc, rv, cnt};
  par_for(m, sparse_range, &x);
  for (uint32_t i = 0; i < m; ++i) cnt[i + 1] += cnt[i];
  const size_t nnz = cnt[m];
  uint32_t* c_out = (uint32_t*)malloc((nnz ? nnz : 1) * sizeof(uint32_t));
  float* v_out = (float*)malloc((nnz ? nnz : 1) * sizeof(float));
  for (uint32_t i = 0; i < m; ++i) {
    const uint32_t len = cnt[i + 1] - cnt[i];
    memcpy(c_out + cnt[i], rc[i], (size_t)len * sizeof(uint32_t));
    memcpy(v_out + cnt[i], rv[i], (size_t)len * sizeof(float));
    free(rc[i]);
    free(rv[i]);
  }
  free(rc);
  free(rv);
  *orp = cnt;
  *oci = c_out;
  *ov = v_out;
  return nnz;
}

/* Epilogue over an already-computed product Z (CSR of TOUCHED positions, as
 * the reference's mxm(CsrMatrix,CsrMatrix) returns, matrix.cpp:489-497):
 * z = Z + b_i -> ReLU -> clip, untouched positions give epilogue(0 + b_i). */
size_t sko_sparse_epilogue(uint32_t m, uint32_t n, const uint32_t* zrp,
                           const uint32_t* zci, const float* zv, const float* bias,
                           float clip, uint32_t** orp, uint32_t** oci, float** ov) {
  uint32_t* rp = (uint32_t*)malloc(((size_t)m + 1) * sizeof(uint32_t));
  size_t cap = zrp[m] + 16, nnz = 0;
  uint32_t* ci = (uint32_t*)malloc(cap * sizeof(uint32_t));
  float* v = (float*)malloc(cap * sizeof(float));
  rp[0] = 0;
  for (uint32_t i = 0; i < m; ++i) {
    const float untouched = epilogue(0.0f, bias[i], clip);
    const int dense_row = untouched != 0.0f;
    uint32_t q = zrp[i];
    const uint32_t qe = zrp[i + 1];
    if (dense_row && cap < nnz + n + 16) {
      cap = (nnz + n + 16) * 2;
      ci = (uint32_t*)realloc(ci, cap * sizeof(uint32_t));
      v = (float*)realloc(v, cap * sizeof(float));
    }
    if (!dense_row) {
      for (; q < qe; ++q) {
        const float z = epilogue(zv[q], bias[i], clip);
        if (z != 0.0f) { ci[nnz] = zci[q]; v[nnz] = z; ++nnz; }
      }
    } else {
      for (uint32_t s = 0; s < n; ++s) {
        float z;
        if (q < qe && zci[q] == s) z = epilogue(zv[q++], bias[i], clip);
        else z = untouched;
        if (z != 0.0f) { ci[nnz] = s; v[nnz] = z; ++nnz; }
      }
    }
    rp[i + 1] = (uint32_t)nnz;
  }
  *orp = rp;
  *oci = ci;
  *ov = v;
  return nnz;
}

void sko_free(void* p) { free(p); }

void sko_categories_sparse(uint32_t m, uint32_t n, const uint32_t* rp,
                           const uint32_t* ci, const float* v, uint8_t* flags) {
  memset(flags, 0, n);
  for (size_t e = 0; e < rp[m]; ++e)
    if (v[e] != 0.0f) flags[ci[e]] = 1;
}

void sko_categories_dense(uint32_t m, uint32_t n, const float* y,
                          uint8_t* flags) {
  memset(flags, 0, n);
  for (size_t i = 0; i < m; ++i)
    for (uint32_t j = 0; j < n; ++j)
      if (y[i * n + j] != 0.0f) flags[j] = 1;
}

int sko_threads(void) {
  if (g_threads > 0) return g_threads;
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

void sko_set_threads(int n) { g_threads = n; }
