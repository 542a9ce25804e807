// K7 (k_exact_stream.cu): the exact layer, one output row at a time, its in-edge
// slices streamed through registers with coalesced 16-byte loads.
#pragma once

#include <stddef.h>
#include <stdint.h>

struct sk_ctx;

namespace sk {

struct StreamArgs {
  const uint32_t* arp;  // W_ref row pointers (row i = in-edges of output neuron i)
  const uint32_t* aci;  // W_ref columns
  const uint32_t* bci;  // Y columns: Y's own array (launch_pass_table) or the padded copy
                        // (launch_pad_passes)
  const uint32_t* wpc;  // pass table: wpc[k*nP + j] = first entry of Y row k with sample >= j*SP
                        // (bits 0-29; bits 31 / 30: head / tail flags, launch_pass_table)
  uint32_t side;        // the side units' offset from bci in 16-byte units (signed)
  uint32_t m, n, nP, nW;  // output rows, samples, passes, 1024-sample windows
                          // (items: one per (row, pass), item_cnt[row * nP + pass])
  const float* bias;
  float clip;
  uint32_t q;             // the constant fixed-point increment
  uint32_t foff, clearw;  // field offset (sum + foff in each 8-bit field), cleared word
  float fx_scale, fx_unscale;
  uint32_t* item_cnt;     // per (row, pass)
  unsigned long long* item_off;
  uint32_t* sc_c;
  float* sc_v;
  uint32_t* sc_r;         // nullable: the row of each of the first 512 scratch entries
  unsigned long long* bump;
  unsigned long long* work;
  unsigned long long cap;
  int* overflow;
  int* wrap;              // 4-bit fields: a field wrapped (the layer is rerun with 8-bit ones)
};

// shared memory of one block for 2^fl accumulator words of fb-bit fields;
// threads per block
size_t stream_block_bytes(int fl, int fb, int ku);
int stream_block_threads();
// the kernel for 2^fl accumulator words (fl 8..11), ns in-edge slots per lane
// (in-degree <= 32 ns), fb-bit fields (8 or 4) and ku 16-byte units per lane
// and step (4 or 6)
const void* stream_kernel(int fl, int ns, int fb, int ku);
// The padded copy of an activation CSR's columns (rows 16-byte aligned, sentinel
// gaps; padded_size words) and its pass table (rows * nP + 1 words).
size_t padded_size(uint32_t rows, size_t nnz);
// short_rows: the mean row holds <= 96 entries (narrower chunks per warp)
void launch_pad_passes(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* pci, uint32_t* wpc, bool short_rows);
// The same padded copy with every pass slice's entries in bank order ((sample +
// 13 row) mod 32; <= 8 passes): K7's counter atomics meet fewer bank conflicts.
void launch_pad_banked(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* pci, uint32_t* wpc, bool short_rows);
// The pass table of an activation CSR read in place (16-byte aligned column
// array, nnz < 2^30) and the rows' side units (2 * rows 16-byte units).
void launch_pass_table(sk_ctx* ctx, const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                       uint32_t nP, int sh, uint32_t* wpc, void* side);
void launch_exact_stream(sk_ctx* ctx, const StreamArgs& p, int fl, int ns, int fb, int ku,
                         unsigned grid, size_t smem);

}  // namespace sk
