/* TEST INFRASTRUCTURE ONLY -- the CPU checker for the GPU path.
 *
 * A plain-C restatement of the reference's hot path for the parts the
 * reference (/root/reference/proj) does not itself provide: the BASELINE
 * workload generators, the clip-at-32 epilogue, the sparse-activation layer
 * epilogue and the category-index set.  Everything the reference DOES provide
 * (relu_forward, mxm, csr_from_triples, gen_input ...) is checked against the
 * reference library itself (oracle/_ref, built by oracle/Makefile), and this
 * restatement is pinned bitwise against it in tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * legs may load this library.  The product (paper_1708_02937_b200) never does.
 *
 * Orientation is the reference's: W_ref is m-by-m CSR whose row i lists the
 * in-edges of output neuron i (proj/include/semikern/dnn.hpp:24-25); the
 * activation Y_ref is m-by-n neuron-major (neurons x samples).
 */
#ifndef SK_ORACLE_H
#define SK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64, counter-addressed (proj/include/semikern/rng.hpp:43-50). */
uint64_t sko_splitmix_at(uint64_t seed, uint64_t idx);
double sko_to_unit(uint64_t bits);

/* ---- BASELINE generators (shared definition with the GPU generators) ---- */

/* Per-layer seed, as the reference CLI derives it (tools/semikern_main.cpp:41-43). */
uint64_t sko_layer_seed(uint64_t seed, uint32_t layer);

/* rows x cols pattern with exactly k distinct columns per row, sorted.
 * Row i draws candidates mulhi(at(at(seed,i), t), cols) for t = 0,1,... and
 * rejects repeats.  cols_out has rows*k entries.  k <= cols required. */
void sko_gen_fixed_rows(uint32_t rows, uint32_t cols, uint32_t k, uint64_t seed,
                        uint32_t* cols_out);

/* Same, for rows row_offset .. row_offset+rows-1 of a larger matrix. */
void sko_gen_fixed_rows_off(uint32_t rows, uint32_t cols, uint32_t k, uint64_t seed,
                            uint64_t row_offset, uint32_t* cols_out);

/* Uniform[-1,1) float for entry index idx of value stream `seed`
 * (an exact 0.0f, probability 2^-53, is replaced by 1.0f so the entry stays
 * structurally present). */
float sko_uniform_pm1(uint64_t seed, uint64_t idx);

/* Transpose a CSR (rows x cols) into CSR (cols x rows); output columns come
 * out ascending because input rows are walked in order. */
void sko_csr_transpose(uint32_t rows, uint32_t cols, const uint32_t* rp,
                       const uint32_t* ci, const float* v, uint32_t* trp,
                       uint32_t* tci, float* tv);

/* Weight layer for the BASELINE configs, emitted in reference orientation
 * (W_ref = W^T).  mode 0: exactly k nonzeros per row of W (Y.W orientation)
 * with values `value` (k>0) or U[-1,1) (value != value, i.e. NaN);
 * returns nnz.  Arrays must hold m+1 / m*k entries. */
size_t sko_gen_layer_fixed(uint32_t m, uint32_t k, uint64_t layer_seed,
                           float value, uint32_t* rp, uint32_t* ci, float* v);

/* Bernoulli-density weight layer (cfg2), reference orientation, values
 * U[-1,1).  Two-call: pass rp only to size, then ci/v.  Returns nnz. */
size_t sko_gen_layer_density(uint32_t m, double density, uint64_t layer_seed,
                             uint32_t* rp, uint32_t* ci, float* v);

/* Dense U[0,1) input, neuron-major m x n: identical formula to the
 * reference's gen_input (proj/src/matgen.cpp:89-99). */
void sko_gen_input_dense(uint32_t m, uint32_t n, uint64_t seed, float* y);

/* Binary sparse input: each of n samples has exactly k active neurons out of
 * m (value 1.0), emitted neuron-major as CSR m x n.  rp: m+1, ci: n*k.
 * Sample s uses the counter of global sample s + sample_offset, so a
 * batch-row shard generates exactly its slice of the global batch. */
void sko_gen_input_binary(uint32_t m, uint32_t n, uint32_t k, uint64_t seed,
                          uint64_t sample_offset, uint32_t* rp, uint32_t* ci,
                          float* v);

/* ---- the layer recurrence ---- */

/* Dense-activation layer, reference fold order (proj/src/matrix.cpp:403-424,
 * proj/src/dnn.cpp:65-103) plus the optional clip:
 *   acc=+0; for e in row i ascending: acc = acc + w_e*y[k_e][j];
 *   z = acc + b_i; z = z<0 ? 0 : z; if clip: z = z>clip ? clip : z.
 * clip <= 0 (or NaN) disables the clip. out is m x n. */
void sko_layer_dense(uint32_t m, uint32_t l, const uint32_t* rp,
                     const uint32_t* ci, const float* wv, const float* bias,
                     float clip, uint32_t n, const float* y, float* out);

/* Sparse-activation layer: Y_ref CSR (l x n) in, Y'_ref CSR (m x n) out,
 * exact zeros pruned.  Fold per output is ascending k (as mxm_csr_csr,
 * proj/src/matrix.cpp:452-521).  Positions untouched by the product see
 * z = 0 + b_i, so a row with epilogue(0+b_i) != 0 comes out dense.
 * Output arrays are malloc'd; release with sko_free. Returns nnz. */
size_t sko_layer_sparse(uint32_t m, uint32_t l, const uint32_t* wrp,
                        const uint32_t* wci, const float* wv, const float* bias,
                        float clip, uint32_t n, const uint32_t* yrp,
                        const uint32_t* yci, const float* yv, uint32_t** orp,
                        uint32_t** oci, float** ov);

/* The layer epilogue alone, applied to the reference's mxm(CsrMatrix,
 * CsrMatrix) result (touched positions).  Same output contract as
 * sko_layer_sparse. */
size_t sko_sparse_epilogue(uint32_t m, uint32_t n, const uint32_t* zrp,
                           const uint32_t* zci, const float* zv, const float* bias,
                           float clip, uint32_t** orp, uint32_t** oci, float** ov);

void sko_free(void* p);

/* Category set: flags[s] = 1 iff sample s has any stored entry != 0. */
void sko_categories_sparse(uint32_t m, uint32_t n, const uint32_t* rp,
                           const uint32_t* ci, const float* v, uint8_t* flags);
void sko_categories_dense(uint32_t m, uint32_t n, const float* y,
                          uint8_t* flags);

/* Number of OpenMP threads the oracle will use. */
int sko_threads(void);
void sko_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
