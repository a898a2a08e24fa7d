// Device build of the tuple index (the reference's
// build_tuple_index, plan.cpp:292-333). Same output as the host builder in
// planner.cpp — rows in lexicographic tuple order, per-node dense ranks
// ordered by (rank_left, rank_right), the (rank_left, rank_right) pair of
// every distinct rank — computed with radix sorts on the GPU:
//
//   rows   the informative tuple columns (slots with more than one value)
//          come bit-packed into 64-bit words (first column most significant;
//          packed on the host while the tuples are validated, TupleWords);
//          a stable LSD radix sort over the words (request index as the
//          payload) orders the requests lexicographically, ties by request
//          index — so a row's representative is its first request, as on the
//          host. Adjacent-difference flags + a scan number the rows.
//   ranks  nodes are processed by height: every node of one height forms a
//          segment of `rows` keys (segment << kb | rank_l * distinct_r +
//          rank_r) and one radix sort per height orders all segments at once.
//          Dense ranks are a flag scan minus the segment's first scan value;
//          the first element of each run writes the pair of that rank.
//
// Only the host-visible results come back (one compacted copy): the rows,
// distinct counts, every internal node's pairs, every leaf's value list and
// the root's rank per row. Per-node rank arrays stay on the device.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <numeric>

#include "device.hpp"
#include "planner.hpp"

namespace mtcg {

namespace {

#define IK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw CudaError(std::string("tuple index: ") + #x + ": " + cudaGetErrorString(e_));  \
  } while (0)

constexpr int kThreads = 256;

unsigned blocks_for(uint64_t n) {
  return static_cast<unsigned>(std::min<uint64_t>((n + kThreads - 1) / kThreads, 148ull * 64));
}

// word values of the requests in the current order (LSD passes after the first)
__global__ void gather_word(const uint64_t* __restrict__ word, const uint32_t* __restrict__ order, uint64_t k,
                            uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k; i += uint64_t{gridDim.x} * blockDim.x)
    out[i] = word[order[i]];
}

// flag[i] = request order[i] starts a new row (its tuple differs from order[i-1])
__global__ void row_flags(const uint64_t* __restrict__ words, int n_words, const uint32_t* __restrict__ order,
                          uint64_t k, uint32_t* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k; i += uint64_t{gridDim.x} * blockDim.x) {
    uint32_t f = i == 0;
    if (!f)
      for (int w = 0; w < n_words && !f; ++w) f = words[w * k + order[i]] != words[w * k + order[i - 1]];
    flag[i] = f;
  }
}

// rows from the flag scan: row_of_request, row_first (= first request of a row)
__global__ void row_assign(const uint32_t* __restrict__ scan, const uint32_t* __restrict__ flag,
                           const uint32_t* __restrict__ order, uint64_t k, uint32_t* __restrict__ row_of_request,
                           uint32_t* __restrict__ row_first) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < k; i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = scan[i] - 1;
    row_of_request[order[i]] = r;
    if (flag[i]) row_first[r] = order[i];
  }
}

// One segment (node) of a height level. kind 0: leaf over informative column
// `col`; 1: single-valued leaf (every key 0); 2: internal node. Rank arrays
// live in slots (a node's slot is recycled once its parent has run).
struct Seg {
  int kind;
  int wd, sh, nbits;          // kind 0: the column's word, bit offset, width
  int node, right;            // right: internal nodes' right child (pairs)
  int slot, lslot, rslot;     // rank array slots (own, children)
};

__global__ void level_keys(const Seg* __restrict__ segs, int n_segs, uint64_t rows, int kb,
                           const uint64_t* __restrict__ words, uint64_t k, const uint32_t* __restrict__ row_first,
                           const uint32_t* __restrict__ rank, const uint32_t* __restrict__ distinct,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ pos) {
  const uint64_t n = uint64_t(n_segs) * rows;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t s = i / rows, r = i - s * rows;
    const Seg g = segs[s];
    uint64_t key = 0;
    if (g.kind == 0)
      key = (words[uint64_t(g.wd) * k + row_first[r]] >> g.sh) & ((uint64_t{1} << g.nbits) - 1);
    else if (g.kind == 2)
      key = uint64_t(rank[uint64_t(g.lslot) * rows + r]) * distinct[g.right] + rank[uint64_t(g.rslot) * rows + r];
    keys[i] = (kb < 64 ? s << kb : 0) | key;
    pos[i] = static_cast<uint32_t>(i);
  }
}

__global__ void level_flags(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x)
    flag[i] = i == 0 || keys[i] != keys[i - 1];
}

// Ranks, distinct counts and the pairs of one batch. Segment s occupies the
// sorted range [s*rows, (s+1)*rows) (keys are prefixed by the segment); its
// distinct keys are the run starts, numbered by the batch's flag scan; they
// go to the global pair list at *total + scan - 1 (batches back to back).
__global__ void level_assign(const Seg* __restrict__ segs, uint64_t rows, int kb, const uint64_t* __restrict__ keys,
                             const uint32_t* __restrict__ pos, const uint32_t* __restrict__ scan, uint64_t n,
                             uint32_t* __restrict__ rank, uint32_t* __restrict__ distinct,
                             uint64_t* __restrict__ node_off, const uint64_t* __restrict__ total,
                             uint2* __restrict__ pairs) {
  const uint64_t mask = kb < 64 ? (uint64_t{1} << kb) - 1 : ~uint64_t{0};
  const uint64_t t0 = *total;
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t s = pos[i] / rows, r = pos[i] - s * rows;
    const uint64_t start = s * rows;
    const uint32_t b0 = scan[start];
    const uint32_t rk = scan[i] - b0;
    const Seg g = segs[s];
    rank[uint64_t(g.slot) * rows + r] = rk;
    if (i == 0 || keys[i] != keys[i - 1]) {
      const uint64_t key = keys[i] & mask;
      uint2 v;
      if (g.kind == 2) {
        const uint64_t dr = distinct[g.right];
        v = make_uint2(static_cast<uint32_t>(key / dr), static_cast<uint32_t>(key % dr));
      } else {
        v = make_uint2(static_cast<uint32_t>(key), 0u);
      }
      pairs[t0 + scan[i] - 1] = v;
    }
    if (i == start) node_off[g.node] = t0 + b0 - 1;
    if (i == start + rows - 1) distinct[g.node] = rk + 1;
  }
}

__global__ void advance_total(uint64_t* total, const uint32_t* scan, uint64_t n) { *total += scan[n - 1]; }

int bits_for(uint64_t span) {  // bits to hold values in [0, span)
  int b = 0;
  while (b < 64 && (uint64_t{1} << b) < span) ++b;
  return b;
}

// Per-device scratch kept across builds (grow-only; one build at a time per
// device): re-allocating and first-touching GBs per compile costs more than
// the sorts themselves.
struct DevScratch {
  std::mutex mu;
  uint8_t* base = nullptr;
  size_t cap = 0;
};
DevScratch g_scratch[64];

struct ScratchUnavailable {};

struct Scratch {
  cudaStream_t st;
  DevScratch& d;
  size_t used = 0;
  Scratch(cudaStream_t s, DevScratch& ds, size_t need) : st(s), d(ds) {
    if (d.cap < need) {
      if (d.base) IK(cudaFree(d.base));
      d.base = nullptr;
      d.cap = 0;
      if (cudaMalloc(&d.base, need) != cudaSuccess) {
        cudaGetLastError();  // clear: the caller falls back to the host builder
        d.base = nullptr;
        throw ScratchUnavailable();
      }
      d.cap = need;
    }
  }
  template <class T>
  T* get(uint64_t n) {
    const size_t b = (std::max<uint64_t>(n, 1) * sizeof(T) + 255) & ~size_t{255};
    if (used + b > d.cap) throw InternalError("tuple index: scratch estimate exceeded");
    T* p = reinterpret_cast<T*>(d.base + used);
    used += b;
    return p;
  }
};

struct Cub {
  cudaStream_t st;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  static size_t need(uint64_t n_sort, uint64_t n_scan) {
    size_t a = 0, b = 0;
    IK(cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const uint64_t*>(nullptr),
                                       static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                       static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n_sort), 0, 64));
    IK(cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<const uint32_t*>(nullptr),
                                     static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n_scan)));
    return std::max(a, b);
  }
  void sort(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, int end_bit) {
    size_t b = temp_bytes;
    IK(cub::DeviceRadixSort::SortPairs(temp, b, kin, kout, vin, vout, static_cast<int64_t>(n), 0,
                                       std::max(end_bit, 1), st));
  }
  void scan(const uint32_t* in, uint32_t* out, uint64_t n) {
    size_t b = temp_bytes;
    IK(cub::DeviceScan::InclusiveSum(temp, b, in, out, static_cast<int64_t>(n), st));
  }
};

__global__ void iota_u32(uint32_t* v, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

}  // namespace

bool build_tuple_index_device(const mtcg_problem& p, const std::vector<int>& postorder, const TupleWords& lay,
                              const std::vector<uint64_t>& tuple_words, int device, TupleIndex& ti) {
  const uint64_t k = p.n_requests;
  if (k == 0 || k >= (uint64_t{1} << 31) || device < 0 || device >= 64) return false;
  const bool tdbg = std::getenv("MTCG_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  const int m = p.n_slots;
  const int n = p.n_nodes;
  std::vector<int> column_of(m, -1);
  const int w = static_cast<int>(lay.informative.size());
  for (int c = 0; c < w; ++c) column_of[lay.informative[c]] = c;
  const int nw = static_cast<int>(lay.span.size());

  // --- host schedule: heights, key-width bounds, batches, rank slots --------
  // (rows <= k: bounds use k; the row count only shrinks the launches)
  std::vector<int> height(n, 0);
  int max_h = 0;
  for (int node : postorder)
    if (p.node_slot[node] < 0) {
      height[node] = 1 + std::max(height[p.node_left[node]], height[p.node_right[node]]);
      max_h = std::max(max_h, height[node]);
    }
  std::vector<uint64_t> ub(n, 1), span(n, 1);
  std::vector<std::vector<Seg>> levels(max_h + 1);
  for (int node : postorder) {
    Seg g{};
    g.node = node;
    g.right = -1;
    if (p.node_slot[node] >= 0) {
      const int col = column_of[p.node_slot[node]];
      g.kind = col >= 0 ? 0 : 1;
      if (col >= 0) {
        g.wd = lay.word[col];
        g.sh = lay.shift[col];
        g.nbits = lay.bits[col];
      }
      span[node] = col >= 0 ? static_cast<uint64_t>(p.slot_n_values[p.node_slot[node]]) : 1;
    } else {
      g.kind = 2;
      g.right = p.node_right[node];
      const unsigned __int128 sp = static_cast<unsigned __int128>(ub[p.node_left[node]]) * ub[p.node_right[node]];
      span[node] = sp > ~uint64_t{0} ? ~uint64_t{0} : static_cast<uint64_t>(sp);
    }
    ub[node] = std::min<uint64_t>(span[node], k);
    levels[height[node]].push_back(g);
  }
  uint64_t pair_bound = 0;
  for (int x = 0; x < n; ++x) pair_bound += ub[x];
  const uint64_t batch_cap = std::max<uint64_t>(k, uint64_t{1} << 24);  // elements per sort
  struct Batch {
    size_t s0;
    int ns, kb;
  };
  std::vector<Seg> all;
  std::vector<Batch> batches;
  for (auto& L : levels)
    for (size_t a0 = 0; a0 < L.size();) {
      size_t a1 = a0;
      int kb = 0;
      while (a1 < L.size()) {
        const int kb2 = std::max(kb, bits_for(span[L[a1].node]));
        if (a1 > a0 && (kb2 + bits_for(a1 - a0 + 1) > 64 || (a1 - a0 + 1) * k > batch_cap)) break;
        kb = kb2;
        ++a1;
      }
      batches.push_back({all.size(), static_cast<int>(a1 - a0), kb});
      all.insert(all.end(), L.begin() + a0, L.begin() + a1);
      a0 = a1;
    }
  // rank slots: taken when a node's batch runs, returned after its parent's
  std::vector<int> slot_of(n, -1), free_slots;
  int n_rank_slots = 0;
  for (const Batch& b : batches) {
    for (int a = 0; a < b.ns; ++a) {
      Seg& g = all[b.s0 + a];
      if (free_slots.empty()) free_slots.push_back(n_rank_slots++);
      g.slot = free_slots.back();
      free_slots.pop_back();
      slot_of[g.node] = g.slot;
      if (g.kind == 2) {
        g.lslot = slot_of[p.node_left[g.node]];
        g.rslot = slot_of[p.node_right[g.node]];
      }
    }
    for (int a = 0; a < b.ns; ++a) {
      const Seg& g = all[b.s0 + a];
      if (g.kind == 2) {
        free_slots.push_back(g.lslot);
        free_slots.push_back(g.rslot);
      }
    }
  }
  uint64_t max_cnt = k;
  for (const Batch& b : batches) max_cnt = std::max<uint64_t>(max_cnt, uint64_t(b.ns) * k);
  auto al = [](uint64_t b) { return (b + 255) & ~uint64_t{255}; };
  const size_t need = al(uint64_t(std::max(nw, 1)) * k * 8) +
                      2 * al(k * 8) + 6 * al(k * 4) + al(uint64_t(n_rank_slots) * k * 4) + al(all.size() * sizeof(Seg)) +
                      2 * al(max_cnt * 8) + 4 * al(max_cnt * 4) + al(pair_bound * 8) + al(n * 8) + al(n * 4) + al(8) +
                      al(Cub::need(max_cnt, max_cnt)) + 4096;

  int prev = 0;
  IK(cudaGetDevice(&prev));
  IK(cudaSetDevice(device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev};
  cudaStream_t st;
  // highest priority: the index usually runs while the previous
  // evaluation's kernels still occupy the GPU
  int prio_lo = 0, prio_hi = 0;
  IK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  IK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio_hi));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sguard{st};
  std::lock_guard<std::mutex> lock(g_scratch[device].mu);
  // the device's free memory bounds the index: without room for its scratch
  // (k x live nodes ranks, sort buffers) the host builder takes over
  try {
    Scratch probe(st, g_scratch[device], need);
  } catch (const ScratchUnavailable&) {
    return false;
  }
  Scratch S(st, g_scratch[device], need);
  Cub cub{st};
  cub.temp_bytes = Cub::need(max_cnt, max_cnt);
  cub.temp = S.get<uint8_t>(cub.temp_bytes);
  ti = TupleIndex{};

  uint64_t* d_words = S.get<uint64_t>(uint64_t(std::max(nw, 1)) * k);
  if (nw) IK(cudaMemcpyAsync(d_words, tuple_words.data(), uint64_t(nw) * k * 8, cudaMemcpyHostToDevice, st));
  uint64_t* d_ka = S.get<uint64_t>(k);
  uint64_t* d_kb = S.get<uint64_t>(k);
  uint32_t* d_order = S.get<uint32_t>(k);
  uint32_t* d_order2 = S.get<uint32_t>(k);
  uint32_t* d_flag = S.get<uint32_t>(k);
  uint32_t* d_scan = S.get<uint32_t>(k);
  uint32_t* d_row_of_request = S.get<uint32_t>(k);
  uint32_t* d_row_first = S.get<uint32_t>(k);
  iota_u32<<<blocks_for(k), kThreads, 0, st>>>(d_order, k);
  // LSD: least significant word first; stable sorts keep the earlier order
  for (int x = nw - 1; x >= 0; --x) {
    const int used = lay.word_bits[x];
    gather_word<<<blocks_for(k), kThreads, 0, st>>>(d_words + uint64_t(x) * k, d_order, k, d_ka);
    cub.sort(d_ka, d_kb, d_order, d_order2, k, used);
    std::swap(d_order, d_order2);
  }
  row_flags<<<blocks_for(k), kThreads, 0, st>>>(d_words, nw, d_order, k, d_flag);
  cub.scan(d_flag, d_scan, k);
  row_assign<<<blocks_for(k), kThreads, 0, st>>>(d_scan, d_flag, d_order, k, d_row_of_request, d_row_first);
  uint32_t rows32 = 0;
  IK(cudaMemcpyAsync(&rows32, d_scan + (k - 1), 4, cudaMemcpyDeviceToHost, st));
  IK(cudaStreamSynchronize(st));
  const uint64_t rows = rows32;
  const auto t_rows = std::chrono::steady_clock::now();

  // --- per-node ranks: one radix sort per batch of equal-height nodes -------
  uint32_t* d_rank = S.get<uint32_t>(uint64_t(n_rank_slots) * k);
  Seg* d_all = S.get<Seg>(all.size());
  uint64_t* d_k1 = S.get<uint64_t>(max_cnt);
  uint64_t* d_k2 = S.get<uint64_t>(max_cnt);
  uint32_t* d_p1 = S.get<uint32_t>(max_cnt);
  uint32_t* d_p2 = S.get<uint32_t>(max_cnt);
  uint32_t* d_f = S.get<uint32_t>(max_cnt);
  uint32_t* d_s = S.get<uint32_t>(max_cnt);
  uint2* d_pairs = S.get<uint2>(pair_bound);
  uint64_t* d_node_off = S.get<uint64_t>(n);
  uint32_t* d_distinct = S.get<uint32_t>(n);
  uint64_t* d_total = S.get<uint64_t>(1);
  IK(cudaMemsetAsync(d_total, 0, 8, st));
  IK(cudaMemcpyAsync(d_all, all.data(), all.size() * sizeof(Seg), cudaMemcpyHostToDevice, st));
  for (const Batch& b : batches) {
    const uint64_t cnt = uint64_t(b.ns) * rows;
    level_keys<<<blocks_for(cnt), kThreads, 0, st>>>(d_all + b.s0, b.ns, rows, b.kb, d_words, k, d_row_first, d_rank,
                                                     d_distinct, d_k1, d_p1);
    cub.sort(d_k1, d_k2, d_p1, d_p2, cnt, std::min(64, b.kb + bits_for(b.ns)));
    level_flags<<<blocks_for(cnt), kThreads, 0, st>>>(d_k2, cnt, d_f);
    cub.scan(d_f, d_s, cnt);
    level_assign<<<blocks_for(cnt), kThreads, 0, st>>>(d_all + b.s0, rows, b.kb, d_k2, d_p2, d_s, cnt, d_rank,
                                                       d_distinct, d_node_off, d_total, d_pairs);
    advance_total<<<1, 1, 0, st>>>(d_total, d_s, cnt);
  }
  // --- results to the host --------------------------------------------------
  ti.distinct.resize(n);
  std::vector<uint64_t> node_off(n);
  uint64_t total = 0;
  IK(cudaMemcpyAsync(ti.distinct.data(), d_distinct, n * 4, cudaMemcpyDeviceToHost, st));
  IK(cudaMemcpyAsync(node_off.data(), d_node_off, n * 8, cudaMemcpyDeviceToHost, st));
  IK(cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, st));
  IK(cudaStreamSynchronize(st));
  const auto t_levels = std::chrono::steady_clock::now();
  if (total > pair_bound) throw InternalError("tuple index: pair bound exceeded");
  // host staging kept across builds (fresh pages cost more than the copies)
  static thread_local std::vector<uint32_t> pairs, row_of_request;
  pairs.resize(2 * total);
  row_of_request.resize(k);
  ti.row_tuple_first.resize(rows);
  ti.root_rank.resize(rows);
  IK(cudaMemcpyAsync(pairs.data(), d_pairs, total * 8, cudaMemcpyDeviceToHost, st));
  IK(cudaMemcpyAsync(row_of_request.data(), d_row_of_request, k * 4, cudaMemcpyDeviceToHost, st));
  IK(cudaMemcpyAsync(ti.row_tuple_first.data(), d_row_first, rows * 4, cudaMemcpyDeviceToHost, st));
  IK(cudaMemcpyAsync(ti.root_rank.data(), d_rank + uint64_t(slot_of[p.root]) * rows, rows * 4,
                     cudaMemcpyDeviceToHost, st));
  IK(cudaStreamSynchronize(st));
  auto t1 = std::chrono::steady_clock::now();
  ti.rank_value.assign(n, {});
  ti.pair_l.assign(n, {});
  ti.pair_r.assign(n, {});
  for (int a = 0; a < n; ++a) {
    const uint32_t* q = pairs.data() + 2 * node_off[a];
    const uint32_t d = ti.distinct[a];
    if (p.node_slot[a] >= 0) {
      auto& v = ti.rank_value[a];
      v.resize(d);
      for (uint32_t i = 0; i < d; ++i) v[i] = q[2 * i];
    } else {
      auto& l = ti.pair_l[a];
      auto& r = ti.pair_r[a];
      l.resize(d);
      r.resize(d);
      for (uint32_t i = 0; i < d; ++i) {
        l[i] = q[2 * i];
        r[i] = q[2 * i + 1];
      }
    }
  }
  ti.rows = rows;
  ti.row_of_request.assign(row_of_request.begin(), row_of_request.end());
  ti.rank.assign(n, nullptr);
  ti.rank[p.root] = ti.root_rank.data();
  if (tdbg)
    std::fprintf(stderr, "[mtcg]   device index phases: upload+rows %.3f, levels %.3f, download %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t_rows - t0).count(),
                 std::chrono::duration<double, std::milli>(t_levels - t_rows).count(),
                 std::chrono::duration<double, std::milli>(t1 - t_levels).count());
  if (tdbg)
    std::fprintf(stderr, "[mtcg]   device tuple index %.3f ms (unpack %.3f ms; %d words, %llu rows, %zu batches, %d rank slots)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(),
                 nw, static_cast<unsigned long long>(rows), batches.size(), n_rank_slots);
  return true;
}

}  // namespace mtcg
