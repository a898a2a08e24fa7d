// tcgen05 3xTF32 complex GEMM path (see tc_gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mtcg {

// One dense batched contraction on the tensor cores. A must be an
// intermediate table ([entry][M][K] complex, K-contiguous rows); its entries
// are rounded to TF32 in place (A is dead after its parent's op) and their
// residuals written to a_lo. B̂ hi/lo are built in bhat_hi/bhat_lo.
struct TcOp {
  int fa, fb, kc;                 // log2 M, N, K
  uint32_t nb;                    // items
  uint64_t a_entries;             // entries in A's table
  float* a;                       // A table (floats, interleaved complex)
  float* a_lo;                    // scratch: a_entries * M * 2K floats
  const uint32_t* ia;
  const float2* b;                // B operand table base
  uint64_t b_item, b_slice;
  const uint32_t* ib;
  const uint32_t *tbn_lo, *tbn_hi, *tbk_lo, *tbk_hi;
  int tbn_bits, tbk_bits;
  float* bhat_hi;                 // scratch: nb * 2N * 2K floats
  float* bhat_lo;
  float2* out;
  const uint32_t* out_rows;
  uint64_t out_item;
  const uint32_t *tom_lo, *tom_hi, *ton_lo, *ton_hi;
  int tom_bits, ton_bits;
  int accumulate;
};

void tc_contract(const TcOp& op, cudaStream_t st);
size_t tc_smem_bytes(int bn);
int tc_tile_n(int n_real);

}  // namespace mtcg
