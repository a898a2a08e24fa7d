// Device side of the multi-tensor contraction engine (sm_100a).
//
// One batched launch per plan node per slice: every distinct (node, rank)
// contraction of the node (plan.hpp:103-111 `distinct`) is an item of the
// batch; operands are gathered from the children's HBM tables through
// per-item entry indices and bit-permutation offset tables, so leg
// permutations and slice projections (project_leg, tensor.cpp:255-282) are
// folded into the loads instead of materialised.
//
// Kernels
//   contract_tile     register/smem-tiled complex GEMM per item: A rows are
//                     K-contiguous (the planner stores every intermediate as
//                     [kept legs][legs the parent closes]); output written
//                     through per-tile offset tables, lanes along the output's
//                     contiguous dimension.
//   contract_rows[_grouped]  HBM-streaming skinny ops (N <= 16, K <= 32): a
//                     thread per A row, B in shared memory; grouped: every
//                     item sharing an A entry reads the row once.
//   contract_generic  one thread per output element, for items with < 256
//                     outputs; contract_dot: a warp per output (long K, C64).
//   chain_kernel      fused operand chains (planner.hpp Chain): a run of
//                     skinny ops applied to a shared-memory block of the
//                     running tensor, in the reference's per-step order.
//   tc_contract       tensor-core ops (tc_gemm.cu).
//   leaf_root         single-slot networks.
//   xeb_*             fused |amp|^2 -> compensated fp64 reductions.
//
// Precision: C64 uses fp32 FMA; C128 uses individually rounded fp64
// multiplies/adds in the reference order (tensor.cpp:186-245) and is
// bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "configs.hpp"
#include "device.hpp"
#include "tc_gemm.hpp"

namespace mtcg {

// One per handle. The intermediate arena is owned here and shared by every
// plan compiled on the handle (plans only keep per-slice intermediates in it
// and the handle is not reentrant), so repeated compiles of a workload do not
// pay cudaMalloc/cudaFree of a multi-GB region each time.
struct Engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  void* arena = nullptr;
  uint64_t arena_bytes = 0;
  void* pinned = nullptr;        // host staging for H2D/D2H (grown on demand)
  uint64_t pinned_bytes = 0;
  void* scratch = nullptr;       // device scratch for linear_xeb inputs
  uint64_t scratch_bytes = 0;
  // Device blobs of destroyed plans, reused by later uploads: cudaFree
  // synchronises the device and was measured to stall for 100s of ms.
  std::vector<std::pair<void*, uint64_t>> blob_pool;
};

namespace {
constexpr size_t kBlobPoolMax = 8;

void* blob_get(Engine* e, uint64_t bytes) {
  size_t best = e->blob_pool.size();
  for (size_t i = 0; i < e->blob_pool.size(); ++i) {
    const uint64_t sz = e->blob_pool[i].second;
    if (sz >= bytes && sz <= 2 * bytes + (1 << 20) &&
        (best == e->blob_pool.size() || sz < e->blob_pool[best].second))
      best = i;
  }
  if (best < e->blob_pool.size()) {
    void* p = e->blob_pool[best].first;
    e->blob_pool.erase(e->blob_pool.begin() + best);
    return p;
  }
  return nullptr;
}
}  // namespace

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t err__ = (x);                                                   \
    if (err__ != cudaSuccess)                                                  \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(err__));     \
  } while (0)

namespace {

// ---- complex arithmetic ----------------------------------------------------

template <class R>
struct V2;
template <>
struct V2<float> {
  using T = float2;
};
template <>
struct V2<double> {
  using T = double2;
};

// acc (+)= a * b. C64: fp32 FMA. C128 exact: the reference's
// pr = xr*yr - xi*yi, pi = xr*yi + xi*yr, each op rounded (no contraction),
// and the first product seeds the accumulator (tensor.cpp:196-213).
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b, bool) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b, bool first) {
  const double pr = __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
  const double pi = __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x));
  if (first) {
    acc.x = pr;
    acc.y = pi;
  } else {
    acc.x = __dadd_rn(acc.x, pr);
    acc.y = __dadd_rn(acc.y, pi);
  }
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  return make_float2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
template <class T>
__device__ __forceinline__ T czero();
template <>
__device__ __forceinline__ float2 czero<float2>() {
  return make_float2(0.f, 0.f);
}
template <>
__device__ __forceinline__ double2 czero<double2>() {
  return make_double2(0.0, 0.0);
}

// ---- kernel parameters ---------------------------------------------------------

struct DTable {
  const uint32_t* lo;
  const uint32_t* hi;
  int lo_bits;
  __device__ __forceinline__ uint32_t operator()(uint64_t x) const {
    return __ldg(lo + (x & ((1u << lo_bits) - 1))) + __ldg(hi + (x >> lo_bits));
  }
};

template <class T>
struct DevOp {
  const T* a;               // A table base
  const T* b;
  T* out;
  const uint32_t* ia;       // per item entry
  const uint32_t* ib;
  const uint32_t* out_rows; // root: item -> accumulator row, else null
  uint64_t a_item, b_item, out_item;
  uint64_t a_slice, b_slice;  // slice projection offsets (elements): resolved on device
  // Slice parameters live in device memory so one captured slice graph
  // serves every slice: cur = {slice index, root accumulates}, and a leaf
  // operand's projection offset is the sum of its per-bit strides over the
  // set bits of the slice index (multieval.cpp:322-329).
  const uint64_t* a_sstr;   // per-bit strides (null: operand not sliced)
  const uint64_t* b_sstr;
  const uint32_t* cur;
  int s_bits;
  int root;
  DTable tam, tak, tbn, tbk, tom, ton;
  uint32_t nb;
  int fa, fb, kc;
  int n_fast;               // epilogue lane order
  int accumulate;           // root: add into the accumulator
  int a_kcontig;            // rows kernel: A rows K-contiguous
  int b_kcontig;            // dot kernel: B rows K-contiguous too (direct loads)
  int o_ncontig;            // rows kernel: output n contiguous
  const uint32_t* grp_items;  // grouped rows kernel: items ordered by A entry
  const uint32_t* grp_start;  // ... CSR offsets per group
  uint32_t n_groups, grp_max;
  uint32_t grp_split;         // blocks sharing one group's items (few-group ops)
};

__device__ __forceinline__ uint64_t slice_offset_dev(const uint64_t* str, int bits, uint32_t s) {
  uint64_t o = 0;
  for (int b = 0; b < bits; ++b)
    if (s >> b & 1) o += __ldg(str + b);
  return o;
}

// Fill the slice-dependent fields of a kernel's private copy of its DevOp.
template <class T>
__device__ __forceinline__ void resolve_slice(DevOp<T>& op) {
  const uint32_t s = __ldg(op.cur);
  op.a_slice = op.a_sstr ? slice_offset_dev(op.a_sstr, op.s_bits, s) : 0;
  op.b_slice = op.b_sstr ? slice_offset_dev(op.b_sstr, op.s_bits, s) : 0;
  op.accumulate = op.root ? static_cast<int>(__ldg(op.cur + 1)) : 0;
}

__global__ void set_slice_kernel(uint32_t* cur, uint32_t s, uint32_t accumulate) {
  cur[0] = s;
  cur[1] = accumulate;
}

// ---- tiled batched contraction -------------------------------------------------

template <class R, int TM, int TN, int RM, int RN, int TK>
__global__ void __launch_bounds__((TM / RM) * (TN / RN))
    contract_tile(const DevOp<typename V2<R>::T> op_in) {
  DevOp<typename V2<R>::T> op = op_in;
  resolve_slice(op);
  using T = typename V2<R>::T;
  constexpr int NT = (TM / RM) * (TN / RN);
  constexpr int TXN = TN / RN;  // threads along n
  constexpr int TYM = TM / RM;  // threads along m
  constexpr bool kExact = sizeof(R) == 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);         // [TK][TM+1]
  T* Bs = As + TK * (TM + 1);                     // [TK][TN+1]
  uint32_t* aoff = reinterpret_cast<uint32_t*>(Bs + TK * (TN + 1));
  uint32_t* boff = aoff + TM;
  uint32_t* omo = boff + TN;
  uint32_t* ono = omo + TM;
  uint32_t* kao = ono + TN;
  uint32_t* kbo = kao + TK;

  const uint64_t M = uint64_t{1} << op.fa, N = uint64_t{1} << op.fb;
  const uint64_t K = uint64_t{1} << op.kc;
  const uint64_t tiles_m = (M + TM - 1) / TM, tiles_n = (N + TN - 1) / TN;
  const uint64_t tile = blockIdx.x + uint64_t{gridDim.x} * blockIdx.y;
  const uint64_t tn_i = tile % tiles_n;
  const uint64_t tm_i = (tile / tiles_n) % tiles_m;
  const uint64_t item = tile / (tiles_n * tiles_m);
  if (item >= op.nb) return;
  const uint64_t m0 = tm_i * TM, n0 = tn_i * TN;
  const int tid = threadIdx.x;

  const T* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item) : (uint32_t)item} * op.a_item + op.a_slice;
  const T* B = op.b + uint64_t{op.ib ? __ldg(op.ib + item) : (uint32_t)item} * op.b_item + op.b_slice;
  T* O = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + item)} : item) * op.out_item;

  for (int i = tid; i < TM; i += NT) {
    aoff[i] = m0 + i < M ? op.tam(m0 + i) : 0u;
    omo[i] = m0 + i < M ? op.tom(m0 + i) : 0u;
  }
  for (int i = tid; i < TN; i += NT) {
    boff[i] = n0 + i < N ? op.tbn(n0 + i) : 0u;
    ono[i] = n0 + i < N ? op.ton(n0 + i) : 0u;
  }

  int tx, ty;
  if (op.n_fast) {
    tx = tid % TXN;
    ty = tid / TXN;
  } else {
    ty = tid % TYM;
    tx = tid / TYM;
  }

  T acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = czero<T>();

  const int tk = static_cast<int>(K < TK ? K : TK);
  const int m_valid = static_cast<int>(M - m0 < TM ? M - m0 : TM);
  const int n_valid = static_cast<int>(N - n0 < TN ? N - n0 : TN);
  for (uint64_t k0 = 0; k0 < K; k0 += tk) {
    __syncthreads();  // previous chunk consumed; offsets visible
    for (int i = tid; i < tk; i += NT) {
      kao[i] = op.tak(k0 + i);
      kbo[i] = op.tbk(k0 + i);
    }
    __syncthreads();
    // A tile: k fastest across lanes (K-contiguous rows)
#pragma unroll 8
    for (int e = tid; e < TM * tk; e += NT) {
      const int row = e / tk, kk = e - row * tk;
      As[kk * (TM + 1) + row] = row < m_valid ? A[aoff[row] + kao[kk]] : czero<T>();
    }
#pragma unroll 8
    for (int e = tid; e < TN * tk; e += NT) {
      const int col = e / tk, kk = e - col * tk;
      Bs[kk * (TN + 1) + col] = col < n_valid ? B[boff[col] + kbo[kk]] : czero<T>();
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < tk; ++kk) {
      T av[RM], bv[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) av[i] = As[kk * (TM + 1) + ty + i * TYM];
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[j] = Bs[kk * (TN + 1) + tx + j * TXN];
      const bool first = kExact && k0 == 0 && kk == 0;
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) cmac(acc[i][j], av[i], bv[j], first);
    }
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int r = ty + i * TYM;
    if (r >= m_valid) continue;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int cidx = tx + j * TXN;
      if (cidx >= n_valid) continue;
      T* dst = O + omo[r] + ono[cidx];
      *dst = op.accumulate ? cadd(*dst, acc[i][j]) : acc[i][j];
    }
  }
}

// ---- skinny contractions: stream A rows, B resident in shared memory -----------
//
// For N <= 8 the op is a stream over A (M rows of K contiguous elements) and
// the output (M x N): HBM-bound. One thread per row (RPT rows per thread,
// strided by the block so every load/store instruction is warp-coalesced),
// the whole K x N block of B broadcast from shared memory, rows read with
// 16-byte vector loads when K-contiguous, outputs written as one vector run
// when the N legs are the output's lowest bits.

template <class T>
struct Vec4 {
  using type = float4;
};
template <>
struct Vec4<double2> {
  using type = double4;
};

template <class R, int K, int N, int RPT>
__global__ void __launch_bounds__(256, ((K <= 4 && N <= 4) || (K <= 8 && N <= 8 && sizeof(R) == 4) ? 3 : 2))
    contract_rows(const DevOp<typename V2<R>::T> op_in) {
  DevOp<typename V2<R>::T> op = op_in;
  resolve_slice(op);
  // RPT rows per thread computed together: each B row (N complex, one
  // broadcast smem read per element) feeds RPT x N multiply-adds; K streams
  // in chunks of KC so A never occupies more than RPT x KC registers.
  using T = typename V2<R>::T;
  constexpr int KC = K < 8 ? K : 8;
  __shared__ T Bs[K * N];
  __shared__ uint32_t kao[K];
  __shared__ uint32_t ono[N];
  const uint64_t item = blockIdx.y + uint64_t{gridDim.y} * blockIdx.z;
  if (item >= op.nb) return;
  const T* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item) : (uint32_t)item} * op.a_item + op.a_slice;
  const T* B = op.b + uint64_t{op.ib ? __ldg(op.ib + item) : (uint32_t)item} * op.b_item + op.b_slice;
  T* O = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + item)} : item) * op.out_item;
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e - k * N;
    Bs[e] = B[op.tbn(n) + op.tbk(k)];
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) kao[k] = op.tak(k);
  for (int n = threadIdx.x; n < N; n += blockDim.x) ono[n] = op.ton(n);
  __syncthreads();
  const uint64_t M = uint64_t{1} << op.fa;
  // each block streams several row chunks of its item (amortising the B /
  // offset-table setup above over more bytes)
  const uint64_t n_chunks = (M + 256 * RPT - 1) / (256 * RPT);
  for (uint64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
  const uint64_t base = chunk * (256 * RPT) + threadIdx.x;
  const T* rows[RPT];
  bool live[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const uint64_t m = base + j * 256;
    live[j] = m < M;
    rows[j] = A + (live[j] ? op.tam(m) : 0u);
  }
  T acc[RPT][N];
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int n = 0; n < N; ++n) acc[j][n] = czero<T>();
  // fully unrolled over the (<= 4) chunks so the next chunk's loads issue
  // under the current chunk's FMAs; the launch bound keeps 2 blocks per SM
#pragma unroll
  for (int k0 = 0; k0 < K; k0 += KC) {
    T av[RPT][KC];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (KC >= 2 && op.a_kcontig) {
        using V4 = typename Vec4<T>::type;
#pragma unroll
        for (int kk = 0; kk < KC; kk += 2) {
          const V4 v = live[j] ? *reinterpret_cast<const V4*>(rows[j] + k0 + kk) : V4{};
          av[j][kk] = T{v.x, v.y};
          av[j][kk + 1] = T{v.z, v.w};
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) av[j][kk] = live[j] ? rows[j][kao[k0 + kk]] : czero<T>();
      }
    }
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T bv[N];
#pragma unroll
      for (int n = 0; n < N; ++n) bv[n] = Bs[(k0 + kk) * N + n];
      const bool first = k0 == 0 && kk == 0;
#pragma unroll
      for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int n = 0; n < N; ++n) cmac(acc[j][n], av[j][kk], bv[n], first);
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!live[j]) continue;
    T* dst = O + op.tom(base + j * 256);
    if (N >= 2 && op.o_ncontig && !op.accumulate) {
      using V4 = typename Vec4<T>::type;
#pragma unroll
      for (int n = 0; n < N; n += 2)
        *reinterpret_cast<V4*>(dst + n) =
            V4{acc[j][n].x, acc[j][n].y, acc[j][n + 1].x, acc[j][n + 1].y};
    } else {
#pragma unroll
      for (int n = 0; n < N; ++n) {
        T* d = dst + ono[n];
        *d = op.accumulate ? cadd(*d, acc[j][n]) : acc[j][n];
      }
    }
  }
  }  // chunk loop
}

// ---- skinny contractions over groups of items sharing one A entry ---------------
//
// The items of a group differ only in B (and the output): each thread loads
// its RPT A rows once (K complex each, in registers), then loops over the
// group's items with every item's K x N block of B resident in shared memory.
// A is read from HBM once per distinct entry instead of once per item. Per
// output the k loop runs in the same order as contract_rows, so results are
// identical to it (and C128 stays bit-identical to the reference).

template <class R, int K, int N, int RPT>
__global__ void __launch_bounds__(256, (K <= 8 && sizeof(R) == 4 ? 3 : 2))
    contract_rows_grouped(const DevOp<typename V2<R>::T> op_in) {
  DevOp<typename V2<R>::T> op = op_in;
  resolve_slice(op);
  using T = typename V2<R>::T;
  using V4 = typename Vec4<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Bs = reinterpret_cast<T*>(smem_raw);                  // [g][K][N]
  uint32_t* kao = reinterpret_cast<uint32_t*>(Bs + op.grp_max * K * N);
  uint32_t* ono = kao + K;
  uint32_t* items = ono + N;                               // [g]
  const uint64_t gid = blockIdx.y + uint64_t{gridDim.y} * blockIdx.z;
  const uint64_t group = gid / op.grp_split;
  if (group >= op.n_groups) return;
  // this block's share of the group's items
  const uint32_t gs = __ldg(op.grp_start + group);
  const int gfull = static_cast<int>(__ldg(op.grp_start + group + 1) - gs);
  const int per = (gfull + static_cast<int>(op.grp_split) - 1) / static_cast<int>(op.grp_split);
  const int i0 = static_cast<int>(gid % op.grp_split) * per;
  const int g = min(per, gfull - i0);
  if (g <= 0) return;
  const uint32_t g0 = gs + static_cast<uint32_t>(i0);
  for (int i = threadIdx.x; i < g; i += blockDim.x) items[i] = __ldg(op.grp_items + g0 + i);
  __syncthreads();
  const uint32_t item0 = items[0];
  const T* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item0) : item0} * op.a_item + op.a_slice;
  for (int e = threadIdx.x; e < g * K * N; e += blockDim.x) {
    const int i = e / (K * N), r = e - i * (K * N);
    const int k = r / N, n = r - k * N;
    const uint32_t it = items[i];
    const T* B = op.b + uint64_t{op.ib ? __ldg(op.ib + it) : it} * op.b_item + op.b_slice;
    Bs[e] = B[op.tbn(n) + op.tbk(k)];
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) kao[k] = op.tak(k);
  for (int n = threadIdx.x; n < N; n += blockDim.x) ono[n] = op.ton(n);
  __syncthreads();
  const uint64_t M = uint64_t{1} << op.fa;
  const uint64_t n_chunks = (M + 256 * RPT - 1) / (256 * RPT);
  for (uint64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const uint64_t base = chunk * (256 * RPT) + threadIdx.x;
    bool live[RPT];
    uint32_t mo[RPT];
    T av[RPT][K];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const uint64_t m = base + j * 256;
      live[j] = m < M;
      const T* row = A + (live[j] ? op.tam(m) : 0u);
      mo[j] = live[j] ? op.tom(m) : 0u;
      if (K >= 2 && op.a_kcontig) {
#pragma unroll
        for (int kk = 0; kk < K; kk += 2) {
          const V4 v = live[j] ? *reinterpret_cast<const V4*>(row + kk) : V4{};
          av[j][kk] = T{v.x, v.y};
          av[j][kk + 1] = T{v.z, v.w};
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < K; ++kk) av[j][kk] = live[j] ? row[kao[kk]] : czero<T>();
      }
    }
    // per item, per pair of n: one 16-byte broadcast B load feeds 8 x RPT
    // FMAs (the shared-memory pipe, not the FMA pipe, bounds smaller ratios)
    constexpr int NP = N >= 2 ? 2 : 1;
    for (int i = 0; i < g; ++i) {
      const uint32_t it = items[i];
      T* O = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + it)} : it) * op.out_item;
      const T* Bi = Bs + i * K * N;
#pragma unroll
      for (int n0 = 0; n0 < N; n0 += NP) {
        T acc[RPT][NP];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          T bv[NP];
          if (NP == 2) {
            const V4 v = *reinterpret_cast<const V4*>(Bi + kk * N + n0);
            bv[0] = T{v.x, v.y};
            bv[NP - 1] = T{v.z, v.w};
          } else {
            bv[0] = Bi[kk * N + n0];
          }
#pragma unroll
          for (int j = 0; j < RPT; ++j)
#pragma unroll
            for (int n = 0; n < NP; ++n) {
              if (kk == 0) acc[j][n] = czero<T>();
              cmac(acc[j][n], av[j][kk], bv[n], kk == 0);
            }
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          if (!live[j]) continue;
          T* dst = O + mo[j];
          if (NP == 2 && op.o_ncontig && !op.accumulate) {
            *reinterpret_cast<V4*>(dst + n0) =
                V4{acc[j][0].x, acc[j][0].y, acc[j][NP - 1].x, acc[j][NP - 1].y};
          } else {
#pragma unroll
            for (int n = 0; n < NP; ++n) {
              T* d = dst + ono[n0 + n];
              *d = op.accumulate ? cadd(*d, acc[j][n]) : acc[j][n];
            }
          }
        }
      }
    }
  }  // chunk loop
}

// ---- one thread per output element ---------------------------------------------

template <class R>
__global__ void __launch_bounds__(256)
    contract_generic(const DevOp<typename V2<R>::T> op_in) {
  DevOp<typename V2<R>::T> op = op_in;
  resolve_slice(op);
  using T = typename V2<R>::T;
  const int r_out = op.fa + op.fb;
  const uint64_t total = uint64_t{op.nb} << r_out;
  const uint64_t K = uint64_t{1} << op.kc;
  const uint64_t omask = (uint64_t{1} << r_out) - 1;
  for (uint64_t e = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; e < total;
       e += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t item = e >> r_out, o = e & omask;
    const T* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item) : (uint32_t)item} * op.a_item +
                 op.a_slice + op.tam(o);
    const T* B = op.b + uint64_t{op.ib ? __ldg(op.ib + item) : (uint32_t)item} * op.b_item +
                 op.b_slice + op.tbn(o);
    T acc = czero<T>();
    for (uint64_t c = 0; c < K; ++c) cmac(acc, A[op.tak(c)], B[op.tbk(c)], c == 0);
    T* dst = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + item)} : item) * op.out_item + o;
    *dst = op.accumulate ? cadd(*dst, acc) : acc;
  }
}

// ---- fused operand chains (planner.hpp Chain) --------------------------------------
//
// One block = one final item x nu consecutive untouched-leg combinations u.
// The head's A block (nu x 2^|Q_in| elements) is loaded into shared memory,
// every step contracts the active touched legs with its small B in the
// reference's order (out = sum_c x[in_base(o) + in_c(c)] * b[b_base(o) + b_c(c)],
// the first product seeding the sum, as contract_pair) into the other
// buffer, and the tail's block is stored: the intermediate tables of the run
// never touch HBM.
template <class T>
struct ChainDev {
  const T* a;              // head's A table
  uint64_t a_item;
  T* out;                  // tail's output table
  uint64_t out_item;
  const uint32_t* entries; // [(steps + 1) x nb]
  uint32_t nb;
  int n_steps, q, inner_bits, outer_bits, n_ld, n_st;
  DTable tu_in, tu_out;    // outer combination -> block base offset
  // block maps, per index bit: shared-memory position and element offset
  uint32_t ld_p[12], ld_o[12], st_p[12], st_o[12];
  int ld_bits, st_bits;
  const uint32_t* cur;     // slice parameters (B operands that are sliced leaves)
  int s_bits;
  struct Step {
    const T* b;
    uint64_t b_item;
    const uint64_t* b_sstr;
    const uint32_t* tbl;
    int out_bits, kc, g_bits, f_bits;
    int tbl_rel;           // word offset of the step's tables from step 0's
  } steps[kMaxChainSteps];
  int tbl_words;           // all steps' tables
  int cpb_bits;            // log2 outer chunks per block
};

// One step over the block: work item (inner combination uu, kept-leg
// combination f) loads its K inputs once and writes its G outputs; K, G are
// compile-time so inputs (and small B tiles) live in registers.
template <class T, int KC, int GB>
__device__ __forceinline__ void chain_step(const T* X, T* Y, const T* Bs, const uint32_t* tb, int pitch,
                                           int inner_bits, int f_bits) {
  constexpr int K = 1 << KC, G = 1 << GB;
  // small B tiles in registers (complex64: up to 4 x 4 — else 16 broadcast
  // shared loads in a 4 x 4 work item's ~114 instructions)
  constexpr bool b_regs = K * G * sizeof(T) <= (sizeof(T) == 8 ? 128 : 64);
  const int F = 1 << f_bits;
  // kept legs keep their row positions: in_base[f] is also f's output base
  const uint32_t* in_base = tb;
  const uint32_t* out_g = tb + F;
  const uint32_t* in_c = out_g + G;
  // byte offsets: one add per shared access (an element index costs an add
  // and a scale)
  uint32_t ic[K], og[G];
#pragma unroll
  for (int c = 0; c < K; ++c) ic[c] = in_c[c] * static_cast<uint32_t>(sizeof(T));
#pragma unroll
  for (int g = 0; g < G; ++g) og[g] = out_g[g] * static_cast<uint32_t>(sizeof(T));
  T br[b_regs ? K * G : 1];
  if constexpr (b_regs) {
#pragma unroll
    for (int i = 0; i < K * G; ++i) br[i] = Bs[i];
  }
  const char* const Xb = reinterpret_cast<const char*>(X);
  char* const Yb = reinterpret_cast<char*>(Y);
  const int n = F << inner_bits;
  const int umask = (1 << inner_bits) - 1;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int uu = e & umask, f = e >> inner_bits;
    const uint32_t base = (uu * pitch + in_base[f]) * static_cast<uint32_t>(sizeof(T));
    const char* x = Xb + base;
    T xv[K];
#pragma unroll
    for (int c = 0; c < K; ++c) xv[c] = *reinterpret_cast<const T*>(x + ic[c]);
    char* y = Yb + base;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      T acc = czero<T>();
#pragma unroll
      for (int c = 0; c < K; ++c) cmac(acc, xv[c], b_regs ? br[c * G + g] : Bs[c * G + g], c == 0);
      *reinterpret_cast<T*>(y + og[g]) = acc;
    }
  }
}

template <class T>
__device__ __forceinline__ void chain_step_any(int kc, int gb, const T* X, T* Y, const T* Bs,
                                               const uint32_t* tb, int pitch, int inner_bits, int f_bits) {
#define MTCG_CHAIN_CASE(KC_, GB_) \
  case KC_ * 4 + GB_:             \
    chain_step<T, KC_, GB_>(X, Y, Bs, tb, pitch, inner_bits, f_bits); \
    break;
  switch (kc * 4 + gb) {
    MTCG_CHAIN_CASE(0, 0) MTCG_CHAIN_CASE(0, 1) MTCG_CHAIN_CASE(0, 2) MTCG_CHAIN_CASE(0, 3)
    MTCG_CHAIN_CASE(1, 0) MTCG_CHAIN_CASE(1, 1) MTCG_CHAIN_CASE(1, 2) MTCG_CHAIN_CASE(1, 3)
    MTCG_CHAIN_CASE(2, 0) MTCG_CHAIN_CASE(2, 1) MTCG_CHAIN_CASE(2, 2) MTCG_CHAIN_CASE(2, 3)
    MTCG_CHAIN_CASE(3, 0) MTCG_CHAIN_CASE(3, 1) MTCG_CHAIN_CASE(3, 2) MTCG_CHAIN_CASE(3, 3)
    default: break;
  }
#undef MTCG_CHAIN_CASE
}

// Each block walks `cpb` consecutive outer chunks of one item: the next
// chunk's elements are loaded into registers while the current one is
// contracted and stored (the load latency is the kernel's critical path; a
// block per chunk left most blocks outside their load phase).
constexpr int kChainThreads = 128;              // 16 elements per thread per 2048-element chunk
constexpr int kChainTBits = 7;                  // log2 kChainThreads
template <class R>
__global__ void __launch_bounds__(kChainThreads, sizeof(R) == 4 ? 5 : 3)
    chain_kernel(const __grid_constant__ ChainDev<typename V2<R>::T> d) {
  using T = typename V2<R>::T;
  extern __shared__ __align__(16) uint8_t chain_smem[];
  const int pitch = (1 << d.q) + 1;  // odd row pitch: rows start in different banks
  const int blk = pitch << d.inner_bits;
  T* const X0 = reinterpret_cast<T*>(chain_smem);
  T* const Y0 = X0 + blk;
  T* Bs = Y0 + blk;                                                    // B tiles, 64 per step
  uint32_t* tb = reinterpret_cast<uint32_t*>(Bs + 64 * d.n_steps);    // all steps' tables
  const int chunk_bits = d.outer_bits - d.cpb_bits;
  const uint32_t item = blockIdx.x >> chunk_bits;
  const uint64_t outer0 = (blockIdx.x & ((uint64_t{1} << chunk_bits) - 1)) << d.cpb_bits;
  // every step's tables (contiguous in the index blob) and B tile, once
  for (int i = threadIdx.x; i < d.tbl_words; i += blockDim.x) tb[i] = __ldg(d.steps[0].tbl + i);
  const uint32_t slice = d.cur ? __ldg(d.cur) : 0u;
  for (int l = 0; l < d.n_steps; ++l) {
    const auto& st = d.steps[l];
    const int KG = 1 << (st.kc + st.g_bits);
    if (threadIdx.x < KG) {
      const uint32_t* boff = st.tbl + (1 << st.f_bits) + (1 << st.g_bits) + (1 << st.kc);
      const uint64_t b_slice = st.b_sstr ? slice_offset_dev(st.b_sstr, d.s_bits, slice) : 0;
      const T* B = st.b + uint64_t{__ldg(d.entries + uint64_t{d.nb} * (l + 1) + item)} * st.b_item + b_slice;
      Bs[64 * l + threadIdx.x] = B[__ldg(boff + threadIdx.x)];
    }
  }
  const T* Aitem = d.a + uint64_t{__ldg(d.entries + item)} * d.a_item;
  T* Oitem = d.out + uint64_t{item} * d.out_item;
  constexpr int kU = 2048 / kChainThreads;  // elements per thread per chunk (2^(inner + |Q_in|) <= 2048)
  // element e = threadIdx.x + kChainThreads u of a map: the low kChainTBits
  // bits from the thread, bits kChainTBits-10 from u
  uint32_t lp = 0, lo = 0, sp = 0, so = 0;
#pragma unroll
  for (int i = 0; i < kChainTBits; ++i) {
    if (i < d.ld_bits && (threadIdx.x >> i & 1)) {
      lp += d.ld_p[i];
      lo += d.ld_o[i];
    }
    if (i < d.st_bits && (threadIdx.x >> i & 1)) {
      sp += d.st_p[i];
      so += d.st_o[i];
    }
  }
  // the per-u parts of the maps (bits >= kChainTBits, the same for every thread) live
  // in shared memory: [ld_o | ld_p | st_o | st_p][u] (registers for them
  // capped the kernel at 3 blocks per SM)
  uint32_t* hmap = tb + d.tbl_words;
  if (threadIdx.x < 4 * kU) {
    const int t = threadIdx.x / kU, u = threadIdx.x % kU;
    const uint32_t* tab = t == 0 ? d.ld_o : t == 1 ? d.ld_p : t == 2 ? d.st_o : d.st_p;
    const int bits = t < 2 ? d.ld_bits : d.st_bits;
    uint32_t x = 0;
    for (int i = 0; i < 11 - kChainTBits; ++i)
      if (kChainTBits + i < bits && (u >> i & 1)) x += tab[kChainTBits + i];
    hmap[threadIdx.x] = x;
  }
  __syncthreads();
  const uint32_t* hlo = hmap;
  const uint32_t* hlp = hmap + kU;
  const uint32_t* hso = hmap + 2 * kU;
  const uint32_t* hsp = hmap + 3 * kU;
  T v[kU];
  auto fetch = [&](uint64_t outer) {
    const T* A = Aitem + d.tu_in(outer) + lo;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (threadIdx.x + kChainThreads * u < d.n_ld) v[u] = A[hlo[u]];
  };
  fetch(outer0);
  const int n_chunks = 1 << d.cpb_bits;
  for (int k = 0; k < n_chunks; ++k) {
    __syncthreads();  // the previous chunk's results are stored
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (threadIdx.x + kChainThreads * u < d.n_ld) X0[lp + hlp[u]] = v[u];
    if (k + 1 < n_chunks) fetch(outer0 + k + 1);  // in flight during the steps
    T* X = X0;
    T* Y = Y0;
    for (int l = 0; l < d.n_steps; ++l) {
      const auto& st = d.steps[l];
      __syncthreads();
      chain_step_any<T>(st.kc, st.g_bits, X, Y, Bs + 64 * l, tb + st.tbl_rel, pitch, d.inner_bits, st.f_bits);
      T* t = X;
      X = Y;
      Y = t;
    }
    __syncthreads();
    T* O = Oitem + d.tu_out(outer0 + k) + so;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (threadIdx.x + kChainThreads * u < d.n_st) O[hso[u]] = X[sp + hsp[u]];
  }
}

// ---- one warp per output element (complex64, long K) ----------------------------

__global__ void __launch_bounds__(256)
    contract_dot(const DevOp<float2> op_in) {
  DevOp<float2> op = op_in;
  resolve_slice(op);
  const int r_out = op.fa + op.fb;
  const uint64_t total = uint64_t{op.nb} << r_out;
  const uint64_t K = uint64_t{1} << op.kc;
  const uint64_t omask = (uint64_t{1} << r_out) - 1;
  const int lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t{gridDim.x} * (blockDim.x / 32);
  for (uint64_t e = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) / 32; e < total; e += warps) {
    const uint64_t item = e >> r_out, o = e & omask;
    const float2* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item) : (uint32_t)item} * op.a_item +
                      op.a_slice + op.tam(o);
    const float2* B = op.b + uint64_t{op.ib ? __ldg(op.ib + item) : (uint32_t)item} * op.b_item +
                      op.b_slice + op.tbn(o);
    float2 acc = make_float2(0.f, 0.f);
    if (op.a_kcontig && op.b_kcontig) {
      // both rows K-contiguous: coalesced direct loads, 4 independent sums
      float2 acc1 = acc, acc2 = acc, acc3 = acc;
      uint64_t c = lane;
      for (; c + 96 < K; c += 128) {
        const float2 a0 = __ldg(A + c), a1 = __ldg(A + c + 32), a2 = __ldg(A + c + 64), a3 = __ldg(A + c + 96);
        const float2 b0 = __ldg(B + c), b1 = __ldg(B + c + 32), b2 = __ldg(B + c + 64), b3 = __ldg(B + c + 96);
        cmac(acc, a0, b0, false);
        cmac(acc1, a1, b1, false);
        cmac(acc2, a2, b2, false);
        cmac(acc3, a3, b3, false);
      }
      for (; c < K; c += 32) cmac(acc, __ldg(A + c), __ldg(B + c), false);
      acc.x += acc1.x + (acc2.x + acc3.x);
      acc.y += acc1.y + (acc2.y + acc3.y);
    } else {
      for (uint64_t c = lane; c < K; c += 32) cmac(acc, A[op.tak(c)], B[op.tbk(c)], false);
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, sh);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, sh);
    }
    if (lane == 0) {
      float2* dst = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + item)} : item) * op.out_item + o;
      *dst = op.accumulate ? cadd(*dst, acc) : acc;
    }
  }
}

// ---- small M x N, long K (complex64) ---------------------------------------------
// One CTA per item (grid-stride): A (M x K) and B (N x K), both K-contiguous,
// stream through a kLkStages-deep cp.async ring of kLkKT-wide K tiles (each
// operand element read from HBM once); warp w owns the 4 x 8 output block at
// m0 = 4 (w & 3), n0 = 8 (w >> 2); its lanes split each tile's K (lane,
// lane + 32) and a butterfly reduction combines them. Bound: HBM (16 x 16 x
// 16384 per item: 4 MB read for 16.8 M FMA).
constexpr int kLkKT = 64;      // complex K per stage
constexpr int kLkStages = 6;   // 6 x 16 KB ring

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(256, 2)
    contract_longk(const DevOp<float2> op_in) {
  DevOp<float2> op = op_in;
  resolve_slice(op);
  extern __shared__ float4 lk_smem[];
  float2* ring = reinterpret_cast<float2*>(lk_smem);  // [stage][A 16 rows | B 16 rows][kLkKT]
  const int M = 1 << op.fa, N = 1 << op.fb;
  const int n_tiles = 1 << (op.kc - 6);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = 4 * (warp & 3), n0 = 8 * (warp >> 2);
  const bool active = m0 < M && n0 < N;
  // loader: thread t copies 16 B (2 complex) at row t >> 4 (of 16), column
  // 2 (t & 15) and + 32 complex, for A then B
  const int lrow = tid >> 4, lcol = 2 * (tid & 15);
  for (uint64_t item = blockIdx.x; item < op.nb; item += gridDim.x) {
    const float2* A = op.a + uint64_t{op.ia ? __ldg(op.ia + item) : static_cast<uint32_t>(item)} * op.a_item + op.a_slice;
    const float2* B = op.b + uint64_t{op.ib ? __ldg(op.ib + item) : static_cast<uint32_t>(item)} * op.b_item + op.b_slice;
    const float2* arow = lrow < M ? A + op.tam(lrow) : nullptr;
    const float2* brow = lrow < N ? B + op.tbn(lrow) : nullptr;
    auto issue = [&](int t) {
      if (t < n_tiles) {
        float2* st = ring + (t % kLkStages) * (32 * kLkKT);
        const uint64_t k0 = uint64_t(t) * kLkKT;
        if (arow) {
          cp_async16(st + lrow * kLkKT + lcol, arow + k0 + lcol);
          cp_async16(st + lrow * kLkKT + lcol + 32, arow + k0 + lcol + 32);
        }
        if (brow) {
          cp_async16(st + (16 + lrow) * kLkKT + lcol, brow + k0 + lcol);
          cp_async16(st + (16 + lrow) * kLkKT + lcol + 32, brow + k0 + lcol + 32);
        }
      }
      cp_async_commit();
    };
    float2 acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < kLkStages - 1; ++t) issue(t);
    for (int t = 0; t < n_tiles; ++t) {
      cp_async_wait<kLkStages - 2>();
      __syncthreads();  // tile t visible to all; tile t - 1's slot free
      issue(t + kLkStages - 1);
      if (active) {
        const float2* st = ring + (t % kLkStages) * (32 * kLkKT);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = lane + 32 * h;
          float2 a[4], b[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = st[(m0 + i) * kLkKT + k];
#pragma unroll
          for (int j = 0; j < 8; ++j) b[j] = st[(16 + n0 + j) * kLkKT + k];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              acc[i][j].x = fmaf(a[i].x, b[j].x, fmaf(-a[i].y, b[j].y, acc[i][j].x));
              acc[i][j].y = fmaf(a[i].x, b[j].y, fmaf(a[i].y, b[j].x, acc[i][j].y));
            }
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring is reused by the next item
    if (active) {
      // butterfly over the lanes per element; lane l keeps element
      // (l >> 3, l & 7) of the block (no second copy of the sums live)
      float2 v = make_float2(0.f, 0.f);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          float2 t = acc[x][y];
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1) {
            t.x += __shfl_xor_sync(0xffffffffu, t.x, sh);
            t.y += __shfl_xor_sync(0xffffffffu, t.y, sh);
          }
          if (lane == x * 8 + y) v = t;
        }
      const int i = lane >> 3, j = lane & 7;
      if (m0 + i < M && n0 + j < N) {
        float2* dst = op.out + (op.out_rows ? uint64_t{__ldg(op.out_rows + item)} : item) * op.out_item +
                      op.tom(m0 + i) + op.ton(n0 + j);
        *dst = op.accumulate ? cadd(*dst, v) : v;
      }
    }
  }
}

// ---- single-slot network: every row's value is the projected leaf ----------------

template <class T>
__global__ void leaf_root(const T* leaves, uint64_t item, const uint32_t* row_value,
                          uint64_t rows, int r_out, DTable tout, const uint64_t* sstr, int s_bits,
                          const uint32_t* cur, T* acc) {
  const uint32_t s = __ldg(cur);
  const uint64_t slice_off = sstr ? slice_offset_dev(sstr, s_bits, s) : 0;
  const int accumulate = static_cast<int>(__ldg(cur + 1));
  const uint64_t total = rows << r_out;
  const uint64_t omask = (uint64_t{1} << r_out) - 1;
  for (uint64_t e = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; e < total;
       e += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t r = e >> r_out, o = e & omask;
    const T v = leaves[uint64_t{row_value[r]} * item + slice_off + tout(o)];
    acc[e] = accumulate ? cadd(acc[e], v) : v;
  }
}

// ---- XEB reductions ------------------------------------------------------------------

// Error-free pairwise combination of (sum, compensation) partials.
__device__ __forceinline__ void two_sum_add(double& s, double& c, double x) {
  const double t = s + x;
  if (fabs(s) >= fabs(x))
    c += (s - t) + x;
  else
    c += (x - t) + s;
  s = t;
}

template <class T>
__global__ void xeb_acc_kernel(const T* acc, const uint32_t* row_mult, uint64_t rows,
                               int r_out, double* partial) {
  const uint64_t total = rows << r_out;
  double s = 0.0, c = 0.0;
  for (uint64_t e = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; e < total;
       e += uint64_t{gridDim.x} * blockDim.x) {
    const T v = acc[e];
    const double re = v.x, im = v.y;
    const double p = re * re + im * im;  // std::norm
    const uint32_t mult = row_mult[e >> r_out];
    for (uint32_t q = 0; q < mult; ++q) two_sum_add(s, c, p);
  }
  __shared__ double ss[256], sc[256];
  ss[threadIdx.x] = s;
  sc[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = 0.0, bc = 0.0;
    for (int i = 0; i < blockDim.x; ++i) {
      two_sum_add(bs, bc, ss[i]);
      bc += sc[i];
    }
    partial[2 * blockIdx.x] = bs;
    partial[2 * blockIdx.x + 1] = bc;
  }
}

__global__ void xeb_probs_kernel(const double* probs, uint64_t count, int amplitudes,
                                 double* partial, int* negative) {
  double s = 0.0, c = 0.0;
  for (uint64_t e = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; e < count;
       e += uint64_t{gridDim.x} * blockDim.x) {
    double p;
    if (amplitudes) {
      const double re = probs[2 * e], im = probs[2 * e + 1];
      p = re * re + im * im;
    } else {
      p = probs[e];
    }
    if (p < 0.0) *negative = 1;
    two_sum_add(s, c, p);
  }
  __shared__ double ss[256], sc[256];
  ss[threadIdx.x] = s;
  sc[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = 0.0, bc = 0.0;
    for (int i = 0; i < blockDim.x; ++i) {
      two_sum_add(bs, bc, ss[i]);
      bc += sc[i];
    }
    partial[2 * blockIdx.x] = bs;
    partial[2 * blockIdx.x + 1] = bc;
  }
}

double finish_partials(const std::vector<double>& part) {
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < part.size(); i += 2) {
    const double x = part[i];
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
    c += part[i + 1];
  }
  return s + c;
}

// ---- launch helpers ---------------------------------------------------------------------

constexpr int kSmSlots = 148 * 8;
constexpr int kXebBlocks = 592;  // 4 x 148 SMs
constexpr int kMaxDevices = 64;

int current_device() {
  int d = 0;
  CK(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) throw CudaError("device ordinal out of range");
  return d;
}

template <class R, int TM, int TN, int RM, int RN>
void launch_tile(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  using T = typename V2<R>::T;
  constexpr int TK = sizeof(R) == 4 ? kTileK64 : kTileK128;
  constexpr int NT = (TM / RM) * (TN / RN);
  const size_t smem = sizeof(T) * (TK * (TM + 1) + TK * (TN + 1)) +
                      sizeof(uint32_t) * (2 * TM + 2 * TN + 2 * TK);
  auto kern = contract_tile<R, TM, TN, RM, RN, TK>;
  static bool attr_set[kMaxDevices] = {};  // per instantiation and device
  const int dev = current_device();
  if (!attr_set[dev]) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    attr_set[dev] = true;
  }
  const uint64_t M = uint64_t{1} << op.fa, N = uint64_t{1} << op.fb;
  const uint64_t tiles = ((M + TM - 1) / TM) * ((N + TN - 1) / TN) * op.nb;
  const uint64_t gx = std::min<uint64_t>(tiles, 65535);
  const uint64_t gy = (tiles + gx - 1) / gx;
  kern<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), NT, smem, st>>>(op);
}

template <class R, int K, int N>
void launch_rows_kn(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  // rows per thread: amortise B reads over more rows when N is small
  constexpr int RPT = sizeof(R) == 8 ? 1 : (N <= 4 ? 4 : 2);
  const uint64_t M = uint64_t{1} << op.fa;
  const uint64_t n_chunks = (M + 256 * RPT - 1) / (256 * RPT);
  // ~16 blocks per SM in total; each loops over n_chunks / gx chunks
  const uint64_t want = std::max<uint64_t>(1, (148 * 16 + op.nb - 1) / op.nb);
  const unsigned gx = static_cast<unsigned>(std::min<uint64_t>(n_chunks, want));
  const unsigned gy = std::min<uint32_t>(op.nb, 65535u);
  const unsigned gz = (op.nb + gy - 1) / gy;
  contract_rows<R, K, N, RPT><<<dim3(gx, gy, gz), 256, 0, st>>>(op);
}

template <class R, int K>
void launch_rows_k(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  switch (op.fb) {
    case 0: return launch_rows_kn<R, K, 1>(op, st);
    case 1: return launch_rows_kn<R, K, 2>(op, st);
    case 2: return launch_rows_kn<R, K, 4>(op, st);
    case 3: return launch_rows_kn<R, K, 8>(op, st);
    default: return launch_rows_kn<R, K, 16>(op, st);
  }
}

template <class R>
void launch_rows(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  switch (op.kc) {
    case 0: return launch_rows_k<R, 1>(op, st);
    case 1: return launch_rows_k<R, 2>(op, st);
    case 2: return launch_rows_k<R, 4>(op, st);
    case 3: return launch_rows_k<R, 8>(op, st);
    case 4: return launch_rows_k<R, 16>(op, st);
    default: return launch_rows_k<R, 32>(op, st);
  }
}

template <class R, int K, int N>
void launch_rows_grouped_kn(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  using T = typename V2<R>::T;
  // rows per thread: RPT x K complex of A in registers
  // (K = 8: two rows per thread and three blocks per SM beat four rows at two
  // blocks — cfg3 node 606 4.97 -> 4.39 ms)
  constexpr int RA = 16;
  constexpr int RPT0 = RA / K;
  constexpr int RPT = RPT0 < 1 ? 1 : (RPT0 > 8 ? 8 : RPT0);
  const size_t smem = sizeof(T) * op.grp_max * K * N + sizeof(uint32_t) * (K + N + op.grp_max);
  auto kern = contract_rows_grouped<R, K, N, RPT>;
  static bool attr_set[kMaxDevices] = {};  // per instantiation and device
  const int dev = current_device();
  if (!attr_set[dev]) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kGroupSmemBytes + 48 * 1024));
    attr_set[dev] = true;
  }
  const uint64_t M = uint64_t{1} << op.fa;
  const uint64_t n_chunks = (M + 256 * RPT - 1) / (256 * RPT);
  // few row chunks x groups: split each group's items over several blocks
  DevOp<T> o = op;
  o.grp_split = 1;
  if (n_chunks * op.n_groups < 2 * 148)
    o.grp_split = static_cast<uint32_t>(std::min<uint64_t>(
        op.grp_max, (2 * 148 + n_chunks * op.n_groups - 1) / (n_chunks * op.n_groups)));
  const uint64_t units = uint64_t{op.n_groups} * o.grp_split;
  const uint64_t want = std::max<uint64_t>(1, (148 * 16 + units - 1) / units);
  const unsigned gx = static_cast<unsigned>(std::min<uint64_t>(n_chunks, want));
  const unsigned gy = static_cast<unsigned>(std::min<uint64_t>(units, 65535u));
  const unsigned gz = static_cast<unsigned>((units + gy - 1) / gy);
  kern<<<dim3(gx, gy, gz), 256, smem, st>>>(o);
}

template <class R, int K>
void launch_rows_grouped_k(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  switch (op.fb) {
    case 0: return launch_rows_grouped_kn<R, K, 1>(op, st);
    case 1: return launch_rows_grouped_kn<R, K, 2>(op, st);
    case 2: return launch_rows_grouped_kn<R, K, 4>(op, st);
    case 3: return launch_rows_grouped_kn<R, K, 8>(op, st);
    default: return launch_rows_grouped_kn<R, K, 16>(op, st);
  }
}

template <class R>
void launch_rows_grouped(const DevOp<typename V2<R>::T>& op, cudaStream_t st) {
  switch (op.kc) {
    case 0: return launch_rows_grouped_k<R, 1>(op, st);
    case 1: return launch_rows_grouped_k<R, 2>(op, st);
    case 2: return launch_rows_grouped_k<R, 4>(op, st);
    case 3: return launch_rows_grouped_k<R, 8>(op, st);
    case 4: return launch_rows_grouped_k<R, 16>(op, st);
    default: return launch_rows_grouped_k<R, 32>(op, st);
  }
}

template <class R>
void launch_op(const DevOp<typename V2<R>::T>& op, int config, cudaStream_t st) {
  switch (config) {
    case kRowsConfig: return launch_rows<R>(op, st);
    case kRowsGroupedConfig: return launch_rows_grouped<R>(op, st);
    case kLongKConfig:
      if constexpr (sizeof(R) == 4) {
        const size_t smem = sizeof(float2) * kLkStages * 32 * kLkKT;
        static bool attr_set[kMaxDevices] = {};
        const int dev = current_device();
        if (!attr_set[dev]) {
          CK(cudaFuncSetAttribute(contract_longk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
          attr_set[dev] = true;
        }
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>(op.nb, kSmSlots * 2));
        contract_longk<<<blocks, 256, smem, st>>>(op);
        return;
      }
      throw CudaError("long-K kernel: complex64 only");
    case kDotConfig:
      if constexpr (sizeof(R) == 4) {
        const uint64_t warps = uint64_t{op.nb} << (op.fa + op.fb);
        const uint64_t blocks = std::min<uint64_t>((warps + 7) / 8, kSmSlots * 8);
        contract_dot<<<static_cast<unsigned>(blocks), 256, 0, st>>>(op);
        return;
      }
      [[fallthrough]];  // (complex128 never selects it)
    case kGenericConfig: {
      const uint64_t total = uint64_t{op.nb} << (op.fa + op.fb);
      const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, kSmSlots * 4);
      contract_generic<R><<<static_cast<unsigned>(blocks), 256, 0, st>>>(op);
      return;
    }
    case 1: return launch_tile<R, 128, 64, 8, 4>(op, st);
    case 2: return launch_tile<R, 128, 32, 8, 2>(op, st);
    case 3: return launch_tile<R, 128, 16, 4, 2>(op, st);
    case 4: return launch_tile<R, 256, 8, 8, 1>(op, st);
    case 5: return launch_tile<R, 256, 4, 4, 1>(op, st);
    case 6: return launch_tile<R, 256, 2, 2, 1>(op, st);
    case 7: return launch_tile<R, 256, 1, 1, 1>(op, st);
    case 8: return launch_tile<R, 64, 64, 4, 4>(op, st);
    case 9:
      // long K: 4 x 4 register tiles (8 shared loads per 16 complex MACs
      // instead of 4 per 4; 64 threads per 32 x 32 tile)
      if (op.kc >= 5) return launch_tile<R, 32, 32, 4, 4>(op, st);
      return launch_tile<R, 32, 32, 2, 2>(op, st);
    case 10: return launch_tile<R, 16, 16, 1, 1>(op, st);
    default: throw CudaError("unknown kernel configuration " + std::to_string(config));
  }
}

DTable dtable(const uint32_t* blob, const SplitTable& t) {
  DTable d;
  d.lo = blob + t.dev_off;
  d.hi = blob + t.dev_off + t.lo.size();
  d.lo_bits = t.lo_bits;
  return d;
}


// Stream assignment for a concurrent (DAG) capture of one slice: an op
// continues the stream whose last op is one of its dependencies when
// possible, otherwise takes the least recently used stream; dependencies on
// other streams become event waits.
struct DagIssue {
  DevicePlan& dp;
  cudaStream_t main;
  std::vector<cudaStream_t> streams;
  std::vector<int> stream_of;  // per op
  std::vector<int> last_op;    // per stream
  DagIssue(DevicePlan& d, cudaStream_t m) : dp(d), main(m) {
    streams.push_back(m);
    for (void* a : dp.aux_streams) streams.push_back(static_cast<cudaStream_t>(a));
    stream_of.assign(dp.c.ops.size(), -1);
    last_op.assign(streams.size(), -1);
    cudaEvent_t fork = static_cast<cudaEvent_t>(dp.join_events.back());
    CK(cudaEventRecord(fork, main));
    for (size_t k = 1; k < streams.size(); ++k) CK(cudaStreamWaitEvent(streams[k], fork, 0));
  }
  cudaStream_t begin(size_t oi) {
    const std::vector<int>& deps = dp.c.ops[oi].deps;
    int chosen = -1;
    for (int d : deps)
      if (stream_of[d] >= 0 && last_op[stream_of[d]] == d) chosen = stream_of[d];
    if (chosen < 0) {
      chosen = 0;
      for (size_t k = 1; k < streams.size(); ++k)
        if (last_op[k] < last_op[chosen]) chosen = static_cast<int>(k);
    }
    for (int d : deps)
      if (stream_of[d] >= 0 && stream_of[d] != chosen)
        CK(cudaStreamWaitEvent(streams[chosen], static_cast<cudaEvent_t>(dp.op_events[d]), 0));
    stream_of[oi] = chosen;
    last_op[chosen] = static_cast<int>(oi);
    return streams[chosen];
  }
  void end(size_t oi) {
    CK(cudaEventRecord(static_cast<cudaEvent_t>(dp.op_events[oi]), streams[stream_of[oi]]));
  }
  void join() {
    for (size_t k = 1; k < streams.size(); ++k) {
      cudaEvent_t j = static_cast<cudaEvent_t>(dp.join_events[k - 1]);
      CK(cudaEventRecord(j, streams[k]));
      CK(cudaStreamWaitEvent(main, j, 0));
    }
  }
};

// Launches one slice's ops; the slice index and the root's accumulate flag
// are read by the kernels from dp.d_cur (set by set_slice_kernel), so this
// launch sequence is the same for every slice and is captured once.
// Ops [op0, op1) only (default: all): the slice-reuse prologue and the
// per-slice ops are launched (and captured) separately.
// Shared memory of a chain block: 2 buffers x 2^(inner + q) elements.
template <class R>
void launch_chain(DevicePlan& dp, const Chain& ch, cudaStream_t st) {
  using T = typename V2<R>::T;
  const Compiled& c = dp.c;
  T* arena = static_cast<T*>(dp.d_arena);
  const T* leaves = static_cast<const T*>(dp.d_leaves);
  const Op& head = c.ops[ch.head];
  const Op& tail = c.ops[ch.tail];
  ChainDev<T> d;
  d.a = arena + head.a_base;
  d.a_item = head.a_item;
  d.out = arena + ch.out_base;
  d.out_item = tail.out_item;
  d.entries = dp.d_index + ch.entries_off;
  d.nb = tail.nb;
  d.n_steps = static_cast<int>(ch.steps.size());
  d.q = ch.q;
  d.inner_bits = ch.u_inner_bits;
  d.outer_bits = ch.u_bits - ch.u_inner_bits;
  d.ld_bits = static_cast<int>(ch.qin.size() / 2);
  d.st_bits = static_cast<int>(ch.qout.size() / 2);
  d.n_ld = 1 << d.ld_bits;
  d.n_st = 1 << d.st_bits;
  if (d.ld_bits > 11 || d.st_bits > 11) throw InternalError("chain block larger than 2048 elements");
  for (int i = 0; i < d.ld_bits; ++i) {
    d.ld_p[i] = ch.qin[2 * i];
    d.ld_o[i] = ch.qin[2 * i + 1];
  }
  for (int i = 0; i < d.st_bits; ++i) {
    d.st_p[i] = ch.qout[2 * i];
    d.st_o[i] = ch.qout[2 * i + 1];
  }
  d.tu_in = dtable(dp.d_tables, ch.tu_in);
  d.tu_out = dtable(dp.d_tables, ch.tu_out);
  d.cur = dp.d_cur;
  d.s_bits = dp.s_bits;
  for (size_t l = 0; l < ch.steps.size(); ++l) {
    const ChainStep& cs = ch.steps[l];
    const Op& op = c.ops[cs.op];
    auto& s = d.steps[l];
    s.b = op.b_leaf ? leaves + op.b_base : arena + op.b_base;
    s.b_item = op.b_item;
    s.b_sstr = dp.b_str_off[cs.op] < 0 ? nullptr : dp.d_sstr + dp.b_str_off[cs.op];
    s.tbl = dp.d_index + cs.tbl_off;
    s.out_bits = __builtin_ctz(cs.n_out);
    s.kc = cs.kc;
    s.g_bits = cs.g_bits;
    s.f_bits = cs.f_bits;
    s.tbl_rel = static_cast<int>(cs.tbl_off - ch.steps[0].tbl_off);
  }
  d.tbl_words = static_cast<int>(ch.steps.back().tbl_off + ch.steps.back().tbl.size() - ch.steps[0].tbl_off);
  const size_t smem = (2 * ((size_t{1} << d.q) + 1 << d.inner_bits) + 64 * ch.steps.size()) * sizeof(T) +
                      4 * static_cast<size_t>(d.tbl_words) + 4 * 4 * (2048 / kChainThreads);  // + the per-u map parts
  static size_t smem_set[kMaxDevices] = {};  // function attributes are per device
  const int dev = current_device();
  if (smem > 48 * 1024 && smem > smem_set[dev]) {
    CK(cudaFuncSetAttribute(chain_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    smem_set[dev] = smem;
  }
  // chunks per block: up to 8, keeping >= 4 blocks per SM's worth of work
  d.cpb_bits = 0;
  while (d.cpb_bits < 3 && d.outer_bits - d.cpb_bits > 0 &&
         (uint64_t{tail.nb} << (d.outer_bits - d.cpb_bits - 1)) >= 148 * 8)
    ++d.cpb_bits;
  const uint64_t blocks = uint64_t{tail.nb} << (d.outer_bits - d.cpb_bits);
  chain_kernel<R><<<static_cast<unsigned>(blocks), kChainThreads, smem, st>>>(d);
}

template <class R>
void launch_slice_ops(DevicePlan& dp, void* d_acc, cudaStream_t st_main, cudaEvent_t* op_events = nullptr,
                      DagIssue* dag = nullptr, size_t op0 = 0, size_t op1 = ~size_t{0}) {
  using T = typename V2<R>::T;
  Compiled& c = dp.c;
  T* arena = static_cast<T*>(dp.d_arena);
  const T* leaves = static_cast<const T*>(dp.d_leaves);
  T* acc = static_cast<T*>(d_acc);
  auto sstr = [&](int64_t off) -> const uint64_t* { return off < 0 ? nullptr : dp.d_sstr + off; };
  // Split-integer tensor-core ops whose A table is slice-invariant (slice
  // reuse): their A rows are quantized in place once, right after the
  // prologue (tc_quantize_a), not in every slice.
  const size_t n_pro = c.n_prologue_ops;
  auto prequant = [&](cudaStream_t st) {
    if constexpr (sizeof(R) == 4) {
      for (size_t j = n_pro; j < c.ops.size(); ++j) {
        const Op& q = c.ops[j];
        if (!q.a_prequant || q.nb == 0 || q.config != kTcConfig) continue;
        TcOp t{};
        t.node = q.node;
        t.fa = q.fa;
        t.fb = q.fb;
        t.kc = q.kc;
        t.a_entries = q.a_entries;
        t.a = reinterpret_cast<const float*>(arena + q.a_base);
        t.row_exp = reinterpret_cast<int8_t*>(arena + q.row_exp_off);
        dp.engine->launches += tc_quantize_a(t, st);
      }
    }
  };
  const size_t op_end = std::min(op1, c.ops.size());
  for (size_t oi = op0; oi < op_end; ++oi) {
    if (n_pro && oi == n_pro && op0 < n_pro && !dag) prequant(st_main);
    const Op& op = c.ops[oi];
    if (op.nb == 0) continue;
    if (op.chain >= 0 && !op.chain_tail) continue;  // evaluated by its chain's tail
    const cudaStream_t st = dag ? dag->begin(oi) : st_main;
    if (op_events) CK(cudaEventRecord(op_events[2 * oi], st));
    if (op.chain >= 0) {
      launch_chain<R>(dp, c.chains[op.chain], st);
      dp.engine->launches++;
      if (op_events) CK(cudaEventRecord(op_events[2 * oi + 1], st));
      if (dag) dag->end(oi);
      continue;
    }
    DevOp<T> d;
    d.a = op.a_leaf ? leaves + op.a_base : arena + op.a_base;
    d.b = op.b_leaf ? leaves + op.b_base : arena + op.b_base;
    d.out = op.root ? acc : arena + op.out_base;
    d.ia = dp.d_index + op.ia_off;
    d.ib = dp.d_index + op.ib_off;
    d.out_rows = op.root ? dp.d_index + op.out_rows_off : nullptr;
    d.a_item = op.a_item;
    d.b_item = op.b_item;
    d.out_item = op.out_item;
    d.a_slice = d.b_slice = 0;
    d.a_sstr = sstr(dp.a_str_off[oi]);
    d.b_sstr = sstr(dp.b_str_off[oi]);
    d.cur = dp.d_cur;
    d.s_bits = dp.s_bits;
    d.root = op.root ? 1 : 0;
    d.tam = dtable(dp.d_tables, op.tam);
    d.tak = dtable(dp.d_tables, op.tak);
    d.tbn = dtable(dp.d_tables, op.tbn);
    d.tbk = dtable(dp.d_tables, op.tbk);
    d.tom = dtable(dp.d_tables, op.tom);
    d.ton = dtable(dp.d_tables, op.ton);
    d.nb = op.nb;
    d.fa = op.fa;
    d.fb = op.fb;
    d.kc = op.kc;
    d.n_fast = op.store_n_fast ? 1 : 0;
    d.a_kcontig = op.a_kcontig ? 1 : 0;
    d.b_kcontig = op.b_kcontig ? 1 : 0;
    d.o_ncontig = op.o_ncontig ? 1 : 0;
    d.grp_items = dp.d_index + op.grp_items_off;
    d.grp_start = dp.d_index + op.grp_start_off;
    d.n_groups = op.grp_start.empty() ? 0 : static_cast<uint32_t>(op.grp_start.size() - 1);
    d.grp_max = op.grp_max;
    d.grp_split = 1;
    d.accumulate = 0;
    if constexpr (sizeof(R) == 4) {
      if (op.config == kTcConfig) {
        TcOp t;
        t.node = op.node;
        t.fa = op.fa;
        t.fb = op.fb;
        t.kc = op.kc;
        t.nb = op.nb;
        t.a_entries = op.a_entries;
        t.a = reinterpret_cast<const float*>(arena + op.a_base);
        t.ia = d.ia;
        t.b = reinterpret_cast<const float2*>(d.b);
        t.b_item = op.b_item;
        t.b_sstr = d.b_sstr;
        t.s_bits = d.s_bits;
        t.cur = d.cur;
        t.root = d.root;
        t.ib = d.ib;
        t.tbn_lo = d.tbn.lo;
        t.tbn_hi = d.tbn.hi;
        t.tbn_bits = d.tbn.lo_bits;
        t.tbk_lo = d.tbk.lo;
        t.tbk_hi = d.tbk.hi;
        t.tbk_bits = d.tbk.lo_bits;
        t.grp_items = op.grp_max ? d.grp_items : nullptr;
        t.grp_start = op.grp_max ? d.grp_start : nullptr;
        t.n_groups = op.grp_max ? d.n_groups : 0;
        t.slots = op.grp_max;
        const uint32_t ga_per = op.ga_tiles.empty() ? 0u : 1u + (128u >> op.fa);
        t.ga_tiles = op.ga_tiles.empty() ? nullptr : dp.d_index + op.ga_tiles_off;
        t.n_ga_tiles = ga_per ? static_cast<uint32_t>(op.ga_tiles.size() / ga_per) : 0u;
        t.ga_groups = op.ga_groups.empty() ? nullptr : dp.d_index + op.ga_groups_off;
        t.n_ga_groups = static_cast<uint32_t>(op.ga_groups.size());
        const uint64_t units = t.n_ga_groups ? uint64_t{t.n_ga_groups}
                               : op.grp_max ? uint64_t{d.n_groups} * op.grp_max : op.nb;
        const uint64_t bhat_elems = units << (op.fb + op.kc + 1);
        t.bhat_hi = reinterpret_cast<float*>(arena + op.scratch_off);
        t.bhat_lo = reinterpret_cast<float*>(arena + op.scratch_off + bhat_elems);
        t.partials = reinterpret_cast<uint32_t*>(arena + op.scratch_off + 2 * bhat_elems);
        t.col_exp = reinterpret_cast<int8_t*>(arena + op.scratch_off + 2 * bhat_elems + 4096 / sizeof(T));
        t.row_exp = op.a_prequant ? reinterpret_cast<int8_t*>(arena + op.row_exp_off)
                                  : t.col_exp + (units << op.fb);
        t.quantize_a = !op.a_prequant;
        t.out = reinterpret_cast<float2*>(d.out);
        t.out_rows = d.out_rows;
        t.out_item = op.out_item;
        t.tom_lo = d.tom.lo;
        t.tom_hi = d.tom.hi;
        t.tom_bits = d.tom.lo_bits;
        t.ton_lo = d.ton.lo;
        t.ton_hi = d.ton.hi;
        t.ton_bits = d.ton.lo_bits;
        // vector epilogue stores need adjacent column pairs only (ton(2j + 1)
        // = ton(2j) + 1), not a contiguous n range
        t.n_contig = (op.ton.bits >= 1 && (op.ton.lo_bits >= 1 ? op.ton.lo[1] : op.ton.hi[1]) == 1) ? 1 : 0;
        t.m_contig = op.o_mcontig ? 1 : 0;
        t.m_stride0 = op.tom.bits >= 1 ? (op.tom.lo_bits >= 1 ? op.tom.lo[1] : op.tom.hi[1]) : 1;
        dp.engine->launches += tc_contract(t, st);  // [absmax +] B̂ build + GEMM
        if (op_events) CK(cudaEventRecord(op_events[2 * oi + 1], st));
        if (dag) dag->end(oi);
        continue;
      }
    }
    launch_op<R>(d, op.config, st);
    dp.engine->launches++;
    if (op_events) CK(cudaEventRecord(op_events[2 * oi + 1], st));
    if (dag) dag->end(oi);
  }
  if (dag) dag->join();
  if (n_pro && op_end == n_pro && op0 < n_pro) prequant(st_main);
  const cudaStream_t st = st_main;
  if (c.has_leaf_root && c.n_rows > 0) {
    const LeafRoot& lr = c.leaf_root;
    const int r_out = static_cast<int>(c.out_legs.size());
    const uint64_t total = c.n_rows << r_out;
    const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, kSmSlots * 4);
    leaf_root<T><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        leaves + c.slot_base[lr.slot], lr.item, dp.d_index + lr.rows_off, c.n_rows, r_out,
        dtable(dp.d_tables, lr.tout), sstr(dp.lr_str_off), dp.s_bits, dp.d_cur, acc);
    dp.engine->launches++;
  }
  CK(cudaGetLastError());
}

void launch_slice(DevicePlan& dp, void* d_acc, cudaStream_t st, cudaEvent_t* op_events = nullptr,
                  DagIssue* dag = nullptr, size_t op0 = 0, size_t op1 = ~size_t{0}) {
  if (dp.c.precision == MTCG_C64)
    launch_slice_ops<float>(dp, d_acc, st, op_events, dag, op0, op1);
  else
    launch_slice_ops<double>(dp, d_acc, st, op_events, dag, op0, op1);
}

// Streams and events for concurrent capture (created once per plan).
// MTCG_STREAMS=<k> sets the stream count; default 1 (serial graph): with the
// first-fit arena most ops depend on their predecessor through memory reuse
// (cfg2: critical path 9.46 of 9.90 ms serialised), so extra streams only add
// event nodes until the allocator keeps independent subtrees apart.
void ensure_dag_resources(DevicePlan& dp) {
  if (!dp.join_events.empty()) return;
  const int k_env = std::getenv("MTCG_STREAMS") ? std::atoi(std::getenv("MTCG_STREAMS")) : 1;
  const int k = std::max(1, std::min(16, k_env));
  for (int i = 1; i < k; ++i) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    dp.aux_streams.push_back(s);
  }
  for (size_t i = 0; i < dp.c.ops.size(); ++i) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    dp.op_events.push_back(e);
  }
  for (int i = 0; i < k; ++i) {  // k - 1 joins + the fork
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    dp.join_events.push_back(e);
  }
}

void set_slice(DevicePlan& dp, uint64_t s, bool accumulate, cudaStream_t st) {
  set_slice_kernel<<<1, 1, 0, st>>>(dp.d_cur, static_cast<uint32_t>(s), accumulate ? 1u : 0u);
  dp.engine->launches++;
}

}  // namespace

// ---- engine / plan lifetime -----------------------------------------------------------

Engine* engine_create(int device) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) throw CudaError("CUDA device " + std::to_string(device) + " not present");
  CK(cudaSetDevice(device));
  auto* e = new Engine;
  e->device = device;
  CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  return e;
}

void engine_destroy(Engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->arena) cudaFree(e->arena);
  if (e->scratch) cudaFree(e->scratch);
  for (auto& [p, sz] : e->blob_pool) cudaFree(p);
  if (e->pinned) cudaFreeHost(e->pinned);
  cudaStreamDestroy(e->stream);
  delete e;
}

uint64_t engine_launches(const Engine* e) { return e->launches; }
uint64_t engine_arena_bytes(const Engine* e) { return e->arena_bytes; }
void* engine_stream(Engine* e) { return e->stream; }

DevicePlan::~DevicePlan() {
  if (engine) cudaSetDevice(engine->device);
  for (auto& [k, g] : graphs) {
    if (g.exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec));
    if (g.exec_pro) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec_pro));
  }
  for (void* e : op_events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* e : join_events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* s : aux_streams) cudaStreamDestroy(static_cast<cudaStream_t>(s));
  if (d_stage) {
    cudaStreamSynchronize(engine ? engine->stream : nullptr);
    cudaFree(d_stage);
  }
  if (d_blob) {
    if (engine) {
      engine->blob_pool.emplace_back(d_blob, blob_bytes);
      if (engine->blob_pool.size() > kBlobPoolMax) {
        cudaFree(engine->blob_pool.front().first);
        engine->blob_pool.erase(engine->blob_pool.begin());
      }
    } else {
      cudaFree(d_blob);
    }
  }
}

// Pinned host staging owned by the engine (grown on demand): every H2D/D2H
// of the one-shot path goes through it, so copies are truly asynchronous.
void* engine_pinned(Engine* e, uint64_t bytes) {
  if (e->pinned_bytes < bytes) {
    if (e->pinned) {
      CK(cudaStreamSynchronize(e->stream));
      CK(cudaFreeHost(e->pinned));
      e->pinned = nullptr;
      e->pinned_bytes = 0;
    }
    const uint64_t want = std::max<uint64_t>(bytes, 1 << 20);
    CK(cudaMallocHost(&e->pinned, want));
    e->pinned_bytes = want;
  }
  return e->pinned;
}

void ensure_arena(DevicePlan& dp);

std::unique_ptr<DevicePlan> upload_plan(Engine* e, Compiled&& c) {
  CK(cudaSetDevice(e->device));
  auto dp = std::make_unique<DevicePlan>();
  dp->engine = e;
  dp->c = std::move(c);
  Compiled& cc = dp->c;
  const size_t eb = cc.elem_bytes;
  // One device allocation and one copy for everything the plan keeps
  // resident: leaves (in the plan precision) | offset tables | index arrays |
  // row multiplicities | XEB partials.
  auto up = [](uint64_t x) { return (x + 255) / 256 * 256; };
  const uint64_t o_leaves = 0;
  const uint64_t o_tables = up(o_leaves + std::max<uint64_t>(cc.leaf_elems * eb, 16));
  const uint64_t o_index = up(o_tables + 4 * std::max<size_t>(cc.table_blob.size(), 1));
  const uint64_t o_mult = up(o_index + 4 * std::max<size_t>(cc.index_blob.size(), 1));
  // per-bit slice strides of sliced leaf operands
  std::vector<uint64_t> sstr;
  auto put_strides = [&](const std::vector<uint64_t>& v) -> int64_t {
    if (std::none_of(v.begin(), v.end(), [](uint64_t x) { return x != 0; })) return -1;
    const int64_t off = static_cast<int64_t>(sstr.size());
    sstr.insert(sstr.end(), v.begin(), v.end());
    return off;
  };
  dp->s_bits = static_cast<int>(cc.sliced.size());
  dp->a_str_off.assign(cc.ops.size(), -1);
  dp->b_str_off.assign(cc.ops.size(), -1);
  for (size_t i = 0; i < cc.ops.size(); ++i) {
    if (cc.ops[i].a_leaf) dp->a_str_off[i] = put_strides(cc.ops[i].a_slice_stride);
    if (cc.ops[i].b_leaf) dp->b_str_off[i] = put_strides(cc.ops[i].b_slice_stride);
  }
  if (cc.has_leaf_root) dp->lr_str_off = put_strides(cc.leaf_root.slice_stride);
  const uint64_t o_sstr = up(o_mult + 4 * std::max<size_t>(cc.row_mult.size(), 1));
  const uint64_t o_cur = up(o_sstr + 8 * std::max<size_t>(sstr.size(), 1));
  const uint64_t o_xeb = up(o_cur + 8);
  const uint64_t total = up(o_xeb + sizeof(double) * 2 * kXebBlocks);
  uint8_t* h = static_cast<uint8_t*>(engine_pinned(e, total));
  CK(cudaStreamSynchronize(e->stream));  // staging may still feed an earlier copy
  if (cc.precision == MTCG_C64) {
    float* f = reinterpret_cast<float*>(h + o_leaves);
    for (uint64_t i = 0; i < 2 * cc.leaf_elems; ++i) f[i] = static_cast<float>(cc.leaf_values[i]);
  } else {
    std::memcpy(h + o_leaves, cc.leaf_values.data(), cc.leaf_values.size() * sizeof(double));
  }
  std::memcpy(h + o_tables, cc.table_blob.data(), 4 * cc.table_blob.size());
  std::memcpy(h + o_index, cc.index_blob.data(), 4 * cc.index_blob.size());
  std::memcpy(h + o_mult, cc.row_mult.data(), 4 * cc.row_mult.size());
  std::memcpy(h + o_sstr, sstr.data(), 8 * sstr.size());
  std::memset(h + o_cur, 0, 8);
  dp->d_blob = blob_get(e, total);
  if (dp->d_blob) {
    // a pooled blob may still be read by work its old plan queued on any
    // stream (cudaFree would have waited for it too)
    CK(cudaDeviceSynchronize());
  } else {
    CK(cudaMalloc(&dp->d_blob, total));
  }
  dp->blob_bytes = total;
  CK(cudaMemcpyAsync(dp->d_blob, h, o_xeb, cudaMemcpyHostToDevice, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  uint8_t* d = static_cast<uint8_t*>(dp->d_blob);
  dp->d_leaves = d + o_leaves;
  dp->d_tables = reinterpret_cast<uint32_t*>(d + o_tables);
  dp->d_index = reinterpret_cast<uint32_t*>(d + o_index);
  dp->d_row_mult = reinterpret_cast<uint32_t*>(d + o_mult);
  dp->d_sstr = reinterpret_cast<uint64_t*>(d + o_sstr);
  dp->d_cur = reinterpret_cast<uint32_t*>(d + o_cur);
  dp->d_xeb_part = reinterpret_cast<double*>(d + o_xeb);
  ensure_arena(*dp);
  return dp;
}

// The intermediate arena is the handle's, shared by its plans and grown to
// the largest one on demand: a plan resolves it before every run (a later,
// larger plan may have moved it) and drops graphs captured on the old one.
void ensure_arena(DevicePlan& dp) {
  Engine* e = dp.engine;
  const uint64_t need = dp.c.arena_elems * static_cast<uint64_t>(dp.c.elem_bytes);
  if (!need) return;
  if (e->arena_bytes < need) {
    if (e->arena) {
      CK(cudaDeviceSynchronize());  // no plan's work may still use it
      CK(cudaFree(e->arena));
      e->arena = nullptr;
      e->arena_bytes = 0;
    }
    CK(cudaMalloc(&e->arena, need));
    e->arena_bytes = need;
  }
  if (dp.d_arena != e->arena) {
    dp.d_arena = e->arena;
    for (auto& [k, g] : dp.graphs) {
      if (g.exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec));
      if (g.exec_pro) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec_pro));
    }
    dp.graphs.clear();
  }
}

// The captured graphs of a plan for accumulator d_acc (slice body, and the
// prologue when the plan has one), created on first use; null when graphs
// are disabled (MTCG_NO_GRAPHS=1).
DevicePlan::GraphEntry* plan_graphs(DevicePlan& dp, void* d_acc, cudaStream_t st) {
  if (std::getenv("MTCG_NO_GRAPHS")) return nullptr;
  const size_t n_pro = dp.c.n_prologue_ops;
  auto capture = [&](size_t op0, size_t op1, void*& exec_out, uint64_t& kernels_out) {
    const uint64_t before = dp.engine->launches;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      DagIssue dag(dp, st);
      launch_slice(dp, d_acc, st, nullptr, &dag, op0, op1);
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    CK(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ierr = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(ierr);
    exec_out = exec;
    kernels_out = dp.engine->launches - before;
    dp.engine->launches = before;  // counted when replayed
  };
  auto it = dp.graphs.find(d_acc);
  if (it == dp.graphs.end()) {
    ensure_dag_resources(dp);
    DevicePlan::GraphEntry e;
    capture(n_pro, ~size_t{0}, e.exec, e.kernels);
    if (n_pro) capture(0, n_pro, e.exec_pro, e.kernels_pro);
    it = dp.graphs.emplace(d_acc, e).first;
  }
  return &it->second;
}

// One slice of a row-chunked evaluation: the request-independent prologue
// (when with_prologue: the first chunk of the slice) and the chunk's body.
void run_slice_chunk(DevicePlan& dp, uint64_t s, void* d_acc, bool accumulate, bool with_prologue,
                     void* stream) {
  CK(cudaSetDevice(dp.engine->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : dp.engine->stream;
  ensure_arena(dp);
  const size_t n_pro = dp.c.n_prologue_ops;
  DevicePlan::GraphEntry* ge = plan_graphs(dp, d_acc, st);
  set_slice(dp, s, accumulate, st);
  if (with_prologue && n_pro) {
    if (ge) {
      CK(cudaGraphLaunch(static_cast<cudaGraphExec_t>(ge->exec_pro), st));
      dp.engine->launches += ge->kernels_pro;
    } else {
      launch_slice(dp, d_acc, st, nullptr, nullptr, 0, n_pro);
    }
  }
  if (ge) {
    CK(cudaGraphLaunch(static_cast<cudaGraphExec_t>(ge->exec), st));
    dp.engine->launches += ge->kernels;
  } else {
    launch_slice(dp, d_acc, st, nullptr, nullptr, n_pro);
  }
}

void run_slices(DevicePlan& dp, uint64_t s0, uint64_t s1, void* d_acc, bool accumulate,
                void* stream, void* d_out_slices) {
  CK(cudaSetDevice(dp.engine->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : dp.engine->stream;
  if (s0 >= s1) return;
  ensure_arena(dp);
  // One slice's launches are captured as a CUDA graph on first use (per
  // accumulator) and replayed for every slice after a set-slice kernel: the
  // host issues 2 launches per slice. MTCG_NO_GRAPHS=1 launches directly.
  // With slice reuse the invariant ops (ops [0, n_pro)) form a second graph
  // run once per call, before the first slice: the arena is shared by the
  // handle's plans, so their resident tables are rebuilt on every run. A
  // row-chunked plan's prologue runs every slice (run_slice_chunk).
  const size_t n_pro = dp.c.row_prologue ? 0 : dp.c.n_prologue_ops;
  if (dp.c.row_prologue && dp.c.n_prologue_ops) {
    const uint64_t slice_bytes = dp.c.n_rows * dp.c.row_elems * static_cast<uint64_t>(dp.c.elem_bytes);
    for (uint64_t s = s0; s < s1; ++s) {
      run_slice_chunk(dp, s, d_acc, !d_out_slices && (accumulate || s > s0), true, stream);
      if (d_out_slices && slice_bytes)
        CK(cudaMemcpyAsync(static_cast<uint8_t*>(d_out_slices) + (s - s0) * slice_bytes, d_acc, slice_bytes,
                           cudaMemcpyDeviceToDevice, st));
    }
    return;
  }
  DevicePlan::GraphEntry* ge = plan_graphs(dp, d_acc, st);
  if (n_pro) {
    set_slice(dp, s0, accumulate, st);
    if (ge) {
      CK(cudaGraphLaunch(static_cast<cudaGraphExec_t>(ge->exec_pro), st));
      dp.engine->launches += ge->kernels_pro;
    } else {
      launch_slice(dp, d_acc, st, nullptr, nullptr, 0, n_pro);
    }
  }
  // per-slice outputs: every slice overwrites d_acc (staging) and is copied
  // to its own slot of d_out_slices
  const uint64_t slice_bytes = dp.c.n_rows * dp.c.row_elems * static_cast<uint64_t>(dp.c.elem_bytes);
  for (uint64_t s = s0; s < s1; ++s) {
    set_slice(dp, s, !d_out_slices && (accumulate || s > s0), st);
    if (ge) {
      CK(cudaGraphLaunch(static_cast<cudaGraphExec_t>(ge->exec), st));
      dp.engine->launches += ge->kernels;
    } else {
      launch_slice(dp, d_acc, st, nullptr, nullptr, n_pro);
    }
    if (d_out_slices && slice_bytes)
      CK(cudaMemcpyAsync(static_cast<uint8_t*>(d_out_slices) + (s - s0) * slice_bytes, d_acc, slice_bytes,
                         cudaMemcpyDeviceToDevice, st));
  }
}

namespace {
// acc = (accumulate ? acc : parts[0]) + parts[1] + ... + parts[n - 1], one
// rounded add per part in part order: the reference's slice fold
// (multieval.cpp:498-513, add_into :369-372), and exactly what the root
// epilogue's accumulation computes when the slices run on one device.
template <class T>
__global__ void fold_kernel(const T* parts, uint64_t n_parts, uint64_t n_elem, T* acc, int accumulate) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n_elem;
       i += uint64_t{gridDim.x} * blockDim.x) {
    T a = accumulate ? acc[i] : parts[i];
    for (uint64_t p = accumulate ? 0 : 1; p < n_parts; ++p) {
      const T b = parts[p * n_elem + i];
      a.x = a.x + b.x;
      a.y = a.y + b.y;
    }
    acc[i] = a;
  }
}
}  // namespace

void fold_slices(Engine* e, int precision, const void* d_parts, uint64_t n_parts, uint64_t n_elem, void* d_acc,
                 bool accumulate, void* stream) {
  CK(cudaSetDevice(e->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : e->stream;
  if (!n_parts || !n_elem) return;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n_elem + 255) / 256, kSmSlots * 4));
  if (precision == MTCG_C64)
    fold_kernel<<<blocks, 256, 0, st>>>(static_cast<const float2*>(d_parts), n_parts, n_elem,
                                         static_cast<float2*>(d_acc), accumulate ? 1 : 0);
  else
    fold_kernel<<<blocks, 256, 0, st>>>(static_cast<const double2*>(d_parts), n_parts, n_elem,
                                         static_cast<double2*>(d_acc), accumulate ? 1 : 0);
  e->launches++;
  CK(cudaGetLastError());
}

int engine_device(const Engine* e) { return e->device; }

void time_ops(DevicePlan& dp, uint64_t slice, void* d_acc, bool accumulate, void* stream,
              float* op_ms) {
  CK(cudaSetDevice(dp.engine->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : dp.engine->stream;
  ensure_arena(dp);
  const size_t n = dp.c.ops.size();
  std::vector<cudaEvent_t> ev(2 * n);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  set_slice(dp, slice, accumulate, st);
  launch_slice(dp, d_acc, st, ev.data());
  CK(cudaStreamSynchronize(st));
  for (size_t i = 0; i < n; ++i) {
    op_ms[i] = 0.f;
    const Op& op = dp.c.ops[i];
    if (op.nb && (op.chain < 0 || op.chain_tail)) CK(cudaEventElapsedTime(&op_ms[i], ev[2 * i], ev[2 * i + 1]));
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

double xeb_device(DevicePlan& dp, const void* d_acc, int n_qubits, void* stream) {
  CK(cudaSetDevice(dp.engine->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : dp.engine->stream;
  const Compiled& c = dp.c;
  const int r_out = static_cast<int>(c.out_legs.size());
  const uint64_t total = c.n_rows << r_out;
  const int blocks = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, kXebBlocks)));
  // partials: preallocated in the plan's blob; read back through the
  // engine's pinned staging — no allocation on the timed path
  double* h_part = static_cast<double*>(engine_pinned(dp.engine, sizeof(double) * 2 * kXebBlocks));
  if (c.precision == MTCG_C64)
    xeb_acc_kernel<float2><<<blocks, 256, 0, st>>>(static_cast<const float2*>(d_acc),
                                                   dp.d_row_mult, c.n_rows, r_out, dp.d_xeb_part);
  else
    xeb_acc_kernel<double2><<<blocks, 256, 0, st>>>(static_cast<const double2*>(d_acc),
                                                    dp.d_row_mult, c.n_rows, r_out, dp.d_xeb_part);
  dp.engine->launches++;
  CK(cudaMemcpyAsync(h_part, dp.d_xeb_part, sizeof(double) * 2 * blocks,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const std::vector<double> part(h_part, h_part + 2 * blocks);
  const double count = static_cast<double>(c.n_requests) * static_cast<double>(c.row_elems);
  return std::ldexp(finish_partials(part) / count, n_qubits) - 1.0;
}

double xeb_probs(Engine* e, const double* probs, uint64_t count, int n_qubits, bool amplitudes) {
  CK(cudaSetDevice(e->device));
  cudaStream_t st = e->stream;
  const uint64_t words = amplitudes ? 2 * count : count;
  const int blocks = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((count + 255) / 256, kXebBlocks)));
  // device scratch: [inputs | partials | negative flag], cached on the engine
  const uint64_t in_bytes = (sizeof(double) * words + 255) / 256 * 256;
  const uint64_t need = in_bytes + sizeof(double) * 2 * kXebBlocks + 256;
  if (e->scratch_bytes < need) {
    if (e->scratch) {
      CK(cudaStreamSynchronize(st));
      CK(cudaFree(e->scratch));
      e->scratch = nullptr;
      e->scratch_bytes = 0;
    }
    CK(cudaMalloc(&e->scratch, need));
    e->scratch_bytes = need;
  }
  uint8_t* base = static_cast<uint8_t*>(e->scratch);
  double* d_in = reinterpret_cast<double*>(base);
  double* d_part = reinterpret_cast<double*>(base + in_bytes);
  int* d_neg = reinterpret_cast<int*>(base + in_bytes + sizeof(double) * 2 * kXebBlocks);
  // inputs go through pinned staging (one host memcpy + one async DMA)
  uint8_t* h = static_cast<uint8_t*>(engine_pinned(e, std::max<uint64_t>(sizeof(double) * words, need - in_bytes)));
  CK(cudaStreamSynchronize(st));
  std::memcpy(h, probs, sizeof(double) * words);
  CK(cudaMemsetAsync(d_neg, 0, sizeof(int), st));
  CK(cudaMemcpyAsync(d_in, h, sizeof(double) * words, cudaMemcpyHostToDevice, st));
  xeb_probs_kernel<<<blocks, 256, 0, st>>>(d_in, count, amplitudes ? 1 : 0, d_part, d_neg);
  e->launches++;
  CK(cudaGetLastError());
  // partials + flag back through the same staging (the H2D above is ordered
  // before this D2H on the stream, so reusing the buffer is safe)
  CK(cudaMemcpyAsync(h, d_part, sizeof(double) * 2 * kXebBlocks + sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double* hp = reinterpret_cast<const double*>(h);
  std::vector<double> part(hp, hp + 2 * blocks);
  int neg = 0;
  std::memcpy(&neg, h + sizeof(double) * 2 * kXebBlocks, sizeof(int));
  if (neg) throw DataError("negative probability");
  return std::ldexp(finish_partials(part) / static_cast<double>(count), n_qubits) - 1.0;
}

void* device_alloc(Engine* e, uint64_t bytes) {
  CK(cudaSetDevice(e->device));
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<uint64_t>(bytes, 16)));
  return p;
}

void device_free(Engine* e, void* p) {
  cudaSetDevice(e->device);
  if (p) cudaFree(p);
}

void copy_to_host(Engine* e, void* dst, const void* src, uint64_t bytes, void* stream) {
  CK(cudaSetDevice(e->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : e->stream;
  void* h = engine_pinned(e, bytes);
  CK(cudaStreamSynchronize(e->stream));
  CK(cudaMemcpyAsync(h, src, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(dst, h, bytes);
}

}  // namespace mtcg
