// Tile configurations of the batched contraction kernel, shared by the host
// planner (selection) and the device code (instantiation).
#pragma once

namespace mtcg {

struct TileConfig {
  int tm, tn, rm, rn;  // block tile M x N, per-thread register tile rm x rn
};

// Index 0 is the per-output-element kernel (no tiling) used for contractions
// with fewer than 256 outputs per item.
constexpr int kGenericConfig = 0;
constexpr int kNumTileConfigs = 11;
constexpr TileConfig kTileConfigs[kNumTileConfigs] = {
    {1, 1, 1, 1},      // 0: generic
    {128, 64, 8, 4},   // 1
    {128, 32, 8, 2},   // 2
    {128, 16, 4, 2},   // 3
    {256, 8, 8, 1},    // 4
    {256, 4, 4, 1},    // 5
    {256, 2, 2, 1},    // 6
    {256, 1, 1, 1},    // 7
    {64, 64, 4, 4},    // 8
    {32, 32, 2, 2},    // 9
    {16, 16, 1, 1},    // 10
};

// K elements staged per k-step (complex64 / complex128).
constexpr int kTileK64 = 16;
constexpr int kTileK128 = 8;

// Row-streaming kernel for skinny ops (N <= 8, K <= 32, M >= 256).
constexpr int kRowsConfig = 11;
// tcgen05 3xTF32 complex GEMM (dense ops, complex64 only; tc_gemm.cu).
constexpr int kTcConfig = 12;
// Row-streaming kernel over groups of items that share their A entry: each
// A row is read once and multiplied by every item's B of the group.
constexpr int kRowsGroupedConfig = 13;
// One warp per output element (lanes split K, shuffle reduction) for items
// with few outputs and a long K; complex64 only (the warp reduction changes
// the summation order, so complex128's reference order keeps the generic
// kernel).
constexpr int kDotConfig = 15;
// Member of a fused operand chain (planner.hpp Chain; reported by op_info —
// the chain's last op launches the chain kernel, the others nothing).
constexpr int kChainConfig = 16;
// Small M x N (M <= 16, 8 <= N <= 16) with a long K (>= 512), both operands
// K-contiguous intermediates, complex64: one CTA per item streams A and B
// through a cp.async ring, warps own 4 x 8 output blocks, lanes split K.
constexpr int kLongKConfig = 17;
// shared-memory budget for one group's B blocks (bytes)
constexpr int kGroupSmemBytes = 48 * 1024;

inline int select_config(int fa, int fb, int kc = 0) {
  // fa >= fb by construction (A is the side with more free legs).
  if (fb <= 4 && fa >= 8 && kc <= 5) return kRowsConfig;
  if (fa + fb < 8) return kGenericConfig;
  const int M = fa, N = fb;  // log2
  if (M >= 7) {
    if (N >= 6) return 1;
    if (N == 5) return 2;
    if (N == 4) return 3;
    if (M >= 8) {
      if (N == 3) return 4;
      if (N == 2) return 5;
      if (N == 1) return 6;
      return 7;
    }
    // M == 128 and N <= 8
    return N == 3 ? 3 : kGenericConfig;
  }
  if (M == 6) return N >= 6 ? 8 : (N >= 4 ? 9 : kGenericConfig);
  if (M == 5) return N >= 4 ? 9 : kGenericConfig;
  if (M == 4) return N >= 4 ? 10 : kGenericConfig;
  return kGenericConfig;
}

}  // namespace mtcg
