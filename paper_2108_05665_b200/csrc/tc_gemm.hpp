// tcgen05 split-precision (3xFP16 / 3xTF32) complex GEMM path (see tc_gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mtcg {

// One dense batched contraction on the tensor cores. A must be an
// intermediate table ([entry][M][K] complex, K-contiguous rows), read raw and
// split into TF32 hi/lo inside the kernel. B̂ hi/lo are built in
// bhat_hi/bhat_lo (scratch).
struct TcOp {
  int node;                       // plan node (diagnostics)
  int fa, fb, kc;                 // log2 M, N, K
  uint32_t nb;                    // items
  uint64_t a_entries;             // entries in A's table
  const float* a;                 // A table (floats, interleaved complex)
  const uint32_t* ia;
  const float2* b;                // B operand table base
  uint64_t b_item;
  const uint64_t* b_sstr;         // B slice projection: per-bit strides (null: none)
  int s_bits;
  const uint32_t* cur;            // device {slice index, root accumulates}
  int root;
  const uint32_t* ib;
  const uint32_t *tbn_lo, *tbn_hi, *tbk_lo, *tbk_hi;
  int tbn_bits, tbk_bits;
  float* bhat_hi;                 // scratch: units * 2N_eff * 2K floats (3xFP16: halves)
  float* bhat_lo;
  uint32_t* partials;             // scratch: 2 x 148 words of operand maxima (3xFP16)
  float2* out;
  const uint32_t* out_rows;
  uint64_t out_item;
  const uint32_t *tom_lo, *tom_hi, *ton_lo, *ton_hi;
  int tom_bits, ton_bits;
  int n_contig;                   // output n index contiguous (vector epilogue stores)
  int m_contig;                   // output m index contiguous (row-per-lane stores coalesce)
  uint64_t m_stride0;             // output stride of m bit 0 (complex elements)
  // Grouped mode (slots > 0): items sharing an A entry are one GEMM whose N
  // is the concatenation of `slots` item B blocks (padded with zero blocks).
  const uint32_t* grp_items;      // items ordered by A entry
  const uint32_t* grp_start;      // n_groups + 1 offsets
  uint32_t n_groups;
  uint32_t slots;
  // Gather mode (ga_tiles != null): tiles stack 128 / M items sharing a B
  // entry; ga_tiles = per tile {group, items...}, ga_groups = B entry per group
  const uint32_t* ga_tiles;
  uint32_t n_ga_tiles;
  const uint32_t* ga_groups;
  uint32_t n_ga_groups;
  // split-integer path (default): B̂ digit planes live in [bhat_hi, bhat_lo +
  // its size), column exponents in col_exp; A rows (K > 32 complex) are
  // quantized in place into digit planes with exponents in row_exp, unless
  // quantize_a is false (done once by the slice-reuse prologue).
  int8_t* col_exp;
  int8_t* row_exp;
  bool quantize_a;
};

// Launches the op's kernels on `st`; returns how many.
int tc_contract(const TcOp& op, cudaStream_t st);
// Split-integer path: the in-place A row quantization alone (slice-reuse
// prologue for ops whose A table is slice-invariant); returns launches.
int tc_quantize_a(const TcOp& op, cudaStream_t st);
// Tensor-core scheme: 0 = split integer (3 int8 digits, exact accumulation;
// default), 1 = 3xFP16, 2 = 3xTF32 (MTCG_TC_KIND=i8|f16|tf32).
int tc_kind();
// A rows of this op are quantized by a pre-pass (K > 32 complex) under the
// split-integer scheme.
inline bool tc_i8_prequant(int kc) { return kc > 5; }
bool tc_f16();                   // 3xFP16 split operands allowed (default) vs 3xTF32 only
bool tc_use_f16(const TcOp& op);  // this op takes the 3xFP16 path
int tc_tile_n(int n_real);

}  // namespace mtcg
