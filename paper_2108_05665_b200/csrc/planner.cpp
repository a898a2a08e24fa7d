// Host compilation of a multi-tensor evaluation (see planner.hpp).
//
// Reference behaviour reproduced here (paths under /root/reference/proj):
//   validation            index_plan plan.cpp:201-259, check_inputs
//                         multieval.cpp:284-297, slice_spec :332-348,
//                         check_legs tensor.cpp:31-40
//   tuple index           build_tuple_index plan.cpp:292-333
//   contraction shapes    shared_legs multieval.cpp:57-64 (every shared leg
//                         is closed, :97), contraction_result_legs
//                         tensor.cpp:100-130
//   counts                predicted_cost tensor.cpp:132-148, Session
//                         node_contractions multieval.cpp:258
//
// B200-specific choices (not in the reference): every distinct (node, rank)
// is evaluated once in one batched launch per node (level batching instead of
// the recursive left/right caches, multieval.cpp:213-274 — the values are
// pure functions of (node, rank), so results and counts are unchanged);
// intermediate layouts are chosen per node so the parent contraction reads
// K-contiguous rows; the HBM arena is planned statically.
#include "planner.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <numeric>
#include <thread>

#include "configs.hpp"

namespace mtcg {

namespace {

std::string fmt(const char* f, long long a = 0, long long b = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b);
  return buf;
}

struct PlanIdx {
  std::vector<int> parent, postorder;
};

// index_plan (plan.cpp:201-259): the plan must be a tree whose leaves are a
// permutation of the slots.
PlanIdx index_plan(const mtcg_problem& p) {
  const int n = p.n_nodes;
  if (p.root < 0 || p.root >= n) throw DataError("plan has no root");
  PlanIdx ix;
  ix.parent.assign(n, -2);
  std::vector<int> inorder;
  std::vector<std::pair<int, int>> stack{{p.root, 0}};
  ix.parent[p.root] = -1;
  while (!stack.empty()) {
    auto& [node, phase] = stack.back();
    if (p.node_slot[node] >= 0) {
      if (p.node_slot[node] >= p.n_slots)
        throw DataError(fmt("leaf slot %lld out of range", p.node_slot[node]));
      inorder.push_back(p.node_slot[node]);
      ix.postorder.push_back(node);
      stack.pop_back();
      continue;
    }
    const int l = p.node_left[node], r = p.node_right[node];
    if (l < 0 || r < 0 || l >= n || r >= n) throw DataError("malformed plan node");
    if (phase < 2) {
      const int child = phase == 0 ? l : r;
      phase += 1;
      if (ix.parent[child] != -2) throw DataError("plan is not a tree");
      ix.parent[child] = node;
      stack.push_back({child, 0});
    } else {
      ix.postorder.push_back(node);
      stack.pop_back();
    }
  }
  std::vector<char> seen(p.n_slots, 0);
  for (int s : inorder) {
    if (seen[s]) throw DataError(fmt("slot %lld appears twice in plan", s));
    seen[s] = 1;
  }
  if (static_cast<int>(inorder.size()) != p.n_slots)
    throw DataError(fmt("plan covers %lld slots, diagram has %lld",
                        static_cast<long long>(inorder.size()), p.n_slots));
  return ix;
}



// build_tuple_index (plan.cpp:292-333). Rows are the distinct request tuples
// in lexicographic order; rank[node][row] is the dense rank of the row's
// restriction to the node's leaves, ordered by (rank_left, rank_right).
// Same ranks as the reference; faster: tuples are compared on the slots that
// have more than one value only (every other column is 0 in every tuple),
// and ranks come from marking the keys each row produces (keys of a node lie
// in [0, distinct[left] * distinct[right])) and sorting only the distinct ones.
TupleIndex build_tuple_index(const mtcg_problem& p, const PlanIdx& ix) {
  TupleIndex ti;
  const uint64_t k = p.n_requests;
  const int m = p.n_slots;
  const uint32_t* T = p.tuples;
  std::vector<int> informative;
  for (int j = 0; j < m; ++j)
    if (p.slot_n_values[j] > 1) informative.push_back(j);
  const size_t w = informative.size();
  static thread_local std::vector<uint32_t> compact;  // scratch kept across compiles
  compact.resize(k * w);
  for (uint64_t i = 0; i < k; ++i)
    for (size_t c = 0; c < w; ++c) compact[i * w + c] = T[i * m + informative[c]];
  const uint32_t* Cp = compact.data();
  // Lexicographic order by an LSD radix sort (one stable counting pass per
  // informative column, value ranges are the slots' value counts): O(k w)
  // instead of a comparison sort. Sorted rows also keep the per-node key
  // passes below cache-friendly.
  // Consecutive informative columns are packed into one digit while the
  // product of their value ranges stays <= 4096 (lexicographic within the
  // group), and the digits stored digit-major: ~w/6 passes over small
  // sequential arrays instead of w passes of strided reads (k = 10^5:
  // 160 -> ~15 ms).
  std::vector<std::pair<size_t, size_t>> groups;  // [c0, c1)
  std::vector<uint32_t> group_span;
  for (size_t c0 = 0; c0 < w;) {
    uint64_t span = 1;
    size_t c1 = c0;
    while (c1 < w && span * static_cast<uint64_t>(p.slot_n_values[informative[c1]]) <= 4096)
      span *= static_cast<uint64_t>(p.slot_n_values[informative[c1++]]);
    if (c1 == c0) span = static_cast<uint64_t>(p.slot_n_values[informative[c1++]]);  // a single wide slot
    groups.push_back({c0, c1});
    group_span.push_back(static_cast<uint32_t>(span));
    c0 = c1;
  }
  static thread_local std::vector<uint32_t> digits;
  digits.resize(groups.size() * k);
  for (size_t g = 0; g < groups.size(); ++g)
    for (uint64_t i = 0; i < k; ++i) {
      uint32_t d = 0;
      for (size_t c = groups[g].first; c < groups[g].second; ++c)
        d = d * static_cast<uint32_t>(p.slot_n_values[informative[c]]) + Cp[i * w + c];
      digits[g * k + i] = d;
    }
  std::vector<uint64_t> order(k), tmp(k);
  std::iota(order.begin(), order.end(), 0);
  std::vector<uint64_t> count;
  for (size_t g = groups.size(); g-- > 0;) {
    const uint64_t span = group_span[g];
    const uint32_t* dg = digits.data() + g * k;
    count.assign(span + 1, 0);
    for (uint64_t i = 0; i < k; ++i) ++count[dg[i] + 1];
    for (uint64_t v = 0; v < span; ++v) count[v + 1] += count[v];
    for (uint64_t i = 0; i < k; ++i) tmp[count[dg[order[i]]]++] = order[i];
    order.swap(tmp);
  }
  auto lex_eq = [&](uint64_t a, uint64_t b) {
    return std::equal(Cp + a * w, Cp + a * w + w, Cp + b * w);
  };
  ti.row_of_request.assign(k, 0);
  for (uint64_t i = 0; i < k; ++i) {
    if (i == 0 || !lex_eq(order[i - 1], order[i]))
      ti.row_tuple_first.push_back(static_cast<uint32_t>(order[i]));
    ti.row_of_request[order[i]] = ti.row_tuple_first.size() - 1;
  }
  ti.rows = ti.row_tuple_first.size();
  const uint64_t rows = ti.rows;
  // One buffer for all nodes' rank arrays, kept per thread across compiles:
  // re-allocating ~n_nodes x rows words per compile page-faults fresh memory
  // every time (ms of jitter on the one-shot path).
  static thread_local std::vector<uint32_t> rank_pool;
  if (rank_pool.size() < uint64_t{static_cast<uint64_t>(p.n_nodes)} * rows)
    rank_pool.resize(uint64_t{static_cast<uint64_t>(p.n_nodes)} * rows);
  ti.rank.assign(p.n_nodes, nullptr);
  for (int node = 0; node < p.n_nodes; ++node) ti.rank[node] = rank_pool.data() + uint64_t{static_cast<uint64_t>(node)} * rows;
  ti.rank_value.assign(p.n_nodes, {});
  ti.distinct.assign(p.n_nodes, 0);
  ti.pair_l.assign(p.n_nodes, {});
  ti.pair_r.assign(p.n_nodes, {});
  // informative columns of the distinct rows, slot-major (sequential reads)
  std::vector<int> column_of(m, -1);
  for (size_t c = 0; c < w; ++c) column_of[informative[c]] = static_cast<int>(c);
  static thread_local std::vector<uint32_t> cols;
  cols.resize(w * rows);
  for (uint64_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < w; ++c)
      cols[c * rows + r] = Cp[static_cast<uint64_t>(ti.row_tuple_first[r]) * w + c];
  static thread_local std::vector<uint64_t> keys;
  keys.resize(rows);
  static thread_local std::vector<uint32_t> mark;  // all-zero between nodes and compiles
  std::vector<uint64_t> touched;
  const uint64_t mark_limit = 16 * rows + 4096;
  const bool tdbg = std::getenv("MTCG_TIMING") != nullptr;
  double t_keys = 0, t_rank = 0;
  for (int node : ix.postorder) {
    auto c0 = std::chrono::steady_clock::now();
    uint32_t* rk = ti.rank[node];
    uint64_t span;  // keys lie in [0, span)
    if (p.node_slot[node] >= 0) {
      const int c = column_of[p.node_slot[node]];
      if (c < 0) {  // single-valued slot: every row has value 0
        std::fill(rk, rk + rows, 0u);
        ti.distinct[node] = rows ? 1 : 0;
        if (rows) ti.rank_value[node].assign(1, 0u);
        continue;
      }
      for (uint64_t r = 0; r < rows; ++r) keys[r] = cols[c * rows + r];
      span = static_cast<uint64_t>(p.slot_n_values[p.node_slot[node]]);
    } else {
      const uint32_t* rl = ti.rank[p.node_left[node]];
      const uint32_t* rr = ti.rank[p.node_right[node]];
      const uint64_t dl = ti.distinct[p.node_left[node]];
      const uint64_t dr = ti.distinct[p.node_right[node]];
      if (rows && (dl == 1 || dr == 1)) {
        // one child is the same for every row: key = the other child's rank,
        // already dense — share its rank array (read-only from here on)
        const bool left_varies = dr == 1;
        ti.rank[node] = const_cast<uint32_t*>(left_varies ? rl : rr);
        const uint64_t d = left_varies ? dl : dr;
        ti.distinct[node] = static_cast<uint32_t>(d);
        auto& pl = ti.pair_l[node];
        auto& pr = ti.pair_r[node];
        pl.resize(d);
        pr.resize(d);
        for (uint64_t i = 0; i < d; ++i) {
          pl[i] = left_varies ? static_cast<uint32_t>(i) : 0u;
          pr[i] = left_varies ? 0u : static_cast<uint32_t>(i);
        }
        t_keys += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
        continue;
      }
      for (uint64_t r = 0; r < rows; ++r) keys[r] = rl[r] * dr + rr[r];
      span = ti.distinct[p.node_left[node]] * dr;
    }
    auto c1 = std::chrono::steady_clock::now();
    // Dense ranks in key order. Keys order like the reference's
    // (rank_l << 32 | rank_r) since rank_r < distinct[right].
    touched.clear();
    if (span <= mark_limit) {
      if (mark.size() < span) mark.resize(span, 0);
      if (span <= 4 * rows + 1024) {
        // counting pass: mark the present keys, then number them in key order
        for (uint64_t r = 0; r < rows; ++r) mark[keys[r]] = 1;
        uint32_t cnt = 0;
        for (uint64_t key = 0; key < span; ++key)
          if (mark[key]) {
            mark[key] = ++cnt;
            touched.push_back(key);
          }
      } else {
        for (uint64_t r = 0; r < rows; ++r)
          if (!mark[keys[r]]) {
            mark[keys[r]] = 1;
            touched.push_back(keys[r]);
          }
        std::sort(touched.begin(), touched.end());
        for (size_t i = 0; i < touched.size(); ++i) mark[touched[i]] = static_cast<uint32_t>(i + 1);
      }
      for (uint64_t r = 0; r < rows; ++r) rk[r] = mark[keys[r]] - 1;
      for (uint64_t key : touched) mark[key] = 0;
    } else {
      touched = keys;
      std::sort(touched.begin(), touched.end());
      touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
      for (uint64_t r = 0; r < rows; ++r)
        rk[r] = static_cast<uint32_t>(
            std::lower_bound(touched.begin(), touched.end(), keys[r]) - touched.begin());
    }
    auto c2 = std::chrono::steady_clock::now();
    t_keys += std::chrono::duration<double, std::milli>(c1 - c0).count();
    t_rank += std::chrono::duration<double, std::milli>(c2 - c1).count();
    ti.distinct[node] = static_cast<uint32_t>(touched.size());
    if (p.node_slot[node] >= 0) {
      ti.rank_value[node].assign(touched.begin(), touched.end());
    } else {
      // (rank_left, rank_right) of every distinct rank: the batch entries
      const uint64_t dr = ti.distinct[p.node_right[node]];
      auto& pl = ti.pair_l[node];
      auto& pr = ti.pair_r[node];
      pl.resize(touched.size());
      pr.resize(touched.size());
      for (size_t i = 0; i < touched.size(); ++i) {
        pl[i] = static_cast<uint32_t>(touched[i] / dr);
        pr[i] = static_cast<uint32_t>(touched[i] % dr);
      }
    }
  }
  if (tdbg) std::fprintf(stderr, "[mtcg]   keys %.3f ms, ranks %.3f ms\n", t_keys, t_rank);
  return ti;
}

bool contains(const std::vector<uint32_t>& v, uint32_t x) {
  return std::find(v.begin(), v.end(), x) != v.end();
}

// Stride (elements) of each leg in a row-major layout.
uint64_t stride_in(const std::vector<uint32_t>& layout, uint32_t leg) {
  uint64_t s = 1;
  for (size_t i = layout.size(); i-- > 0;) {
    if (layout[i] == leg) return s;
    s <<= 1;
  }
  throw InternalError("leg not in layout");
}

}  // namespace

void SplitTable::build(const std::vector<uint64_t>& strides) {
  bits = static_cast<int>(strides.size());
  lo_bits = std::min(bits, 10);
  const int hi_bits = bits - lo_bits;
  lo.assign(size_t{1} << lo_bits, 0);
  hi.assign(size_t{1} << hi_bits, 0);
  // off(x) = off(x without its lowest set bit) + stride of that bit: O(size)
  for (uint64_t x = 1; x < lo.size(); ++x)
    lo[x] = static_cast<uint32_t>(lo[x & (x - 1)] + strides[__builtin_ctzll(x)]);
  for (uint64_t x = 1; x < hi.size(); ++x)
    hi[x] = static_cast<uint32_t>(hi[x & (x - 1)] + strides[lo_bits + __builtin_ctzll(x)]);
}

namespace {
// MTCG_TIMING=1 prints the host compile phases to stderr.
struct PhaseTimer {
  bool on = std::getenv("MTCG_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mtcg] %-14s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// MTCG_TIMING=1: per-section totals accumulated over the ops loop.
struct SectionTimer {
  bool on = std::getenv("MTCG_TIMING") != nullptr;
  double ms[8] = {};
  std::chrono::steady_clock::time_point t;
  void start() {
    if (on) t = std::chrono::steady_clock::now();
  }
  void lap(int i) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    ms[i] += std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
  }
  void print(const char* const* names, int n) const {
    if (!on) return;
    for (int i = 0; i < n; ++i) std::fprintf(stderr, "[mtcg]   %-14s %8.3f ms\n", names[i], ms[i]);
  }
};
}  // namespace

namespace {
// check_inputs' tuple range check (multieval.cpp:284-297; the first offending
// entry in request-major order names the slot), fused with the bit-packing of
// the tuples for the device tuple index (words != nullptr, layout `lay`);
// split over host threads for large batches.
void check_tuples(const mtcg_problem& p, const TupleWords* lay, std::vector<uint64_t>* words) {
  const uint64_t k = p.n_requests;
  const int m = p.n_slots;
  const size_t nw = lay ? lay->span.size() : 0;
  if (words) words->resize(std::max<size_t>(nw, 1) * k);
  uint64_t* out = words ? words->data() : nullptr;
  auto range = [&](uint64_t i0, uint64_t i1) -> uint64_t {  // first bad flat index or ~0
    for (uint64_t i = i0; i < i1; ++i) {
      const uint32_t* t = p.tuples + i * m;
      for (int j = 0; j < m; ++j)
        if (t[j] >= static_cast<uint32_t>(p.slot_n_values[j])) return i * m + j;
      if (out)
        for (size_t x = 0; x < nw; ++x) {
          uint64_t v = 0;
          for (int c = lay->span[x].first; c < lay->span[x].second; ++c)
            v = (v << lay->bits[c]) | t[lay->informative[c]];
          out[x * k + i] = v;
        }
    }
    return ~uint64_t{0};
  };
  uint64_t bad = ~uint64_t{0};
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned nt = k * static_cast<uint64_t>(m) >= (uint64_t{1} << 22) ? hw : 1;
  if (nt == 1) {
    bad = range(0, k);
  } else {
    uint64_t first[16];
    std::thread th[16];
    for (unsigned t = 0; t < nt; ++t)
      th[t] = std::thread([&, t] { first[t] = range(k * t / nt, k * (t + 1) / nt); });
    for (unsigned t = 0; t < nt; ++t) {
      th[t].join();
      bad = std::min(bad, first[t]);
    }
  }
  if (bad != ~uint64_t{0})
    throw DataError(fmt("request tuple indexes past slot %lld's value set", static_cast<long long>(bad % m)));
}

std::vector<int> informative_slots(const mtcg_problem& p) {
  std::vector<int> v;
  for (int j = 0; j < p.n_slots; ++j)
    if (p.slot_n_values[j] > 1) v.push_back(j);
  return v;
}
}  // namespace

TupleWords tuple_word_layout(const mtcg_problem& p) {
  TupleWords L;
  L.informative = informative_slots(p);
  const int w = static_cast<int>(L.informative.size());
  for (int c = 0; c < w; ++c) {
    uint64_t nv = static_cast<uint64_t>(p.slot_n_values[L.informative[c]]);
    int b = 0;
    while ((uint64_t{1} << b) < nv) ++b;
    L.bits.push_back(static_cast<uint8_t>(b));
  }
  L.word.assign(w, 0);
  L.shift.assign(w, 0);
  for (int c0 = 0; c0 < w;) {
    int c1 = c0, used = 0;
    while (c1 < w && used + L.bits[c1] <= 64) used += L.bits[c1++];
    const int x = static_cast<int>(L.span.size());
    int sh = used;
    for (int c = c0; c < c1; ++c) {  // first column most significant
      sh -= L.bits[c];
      L.word[c] = x;
      L.shift[c] = sh;
    }
    L.span.push_back({c0, c1});
    L.word_bits.push_back(used);
    c0 = c1;
  }
  return L;
}

namespace {
// Item indices 0..n-1 stably ordered by key[i] (keys < the key range): a
// counting sort (the grouping / gather orders of every op; comparison sorts
// were the largest part of host compile at 10^5 requests).
std::vector<uint32_t> order_by_key(const std::vector<uint32_t>& key) {
  uint32_t range = 0;
  for (uint32_t k : key) range = std::max(range, k + 1);
  std::vector<uint32_t> count(static_cast<size_t>(range) + 1, 0), out(key.size());
  for (uint32_t k : key) ++count[k + 1];
  for (uint32_t v = 0; v < range; ++v) count[v + 1] += count[v];
  for (uint32_t i = 0; i < key.size(); ++i) out[count[key[i]]++] = i;
  return out;
}
}  // namespace

TupleIndex tuple_index(const mtcg_problem& p, int device) {
  const PlanIdx ix = index_plan(p);
  TupleIndex ti;
  const TupleWords lay = tuple_word_layout(p);
  std::vector<uint64_t> words;
  check_tuples(p, &lay, device >= 0 ? &words : nullptr);
  if (device < 0 || !build_tuple_index_device(p, ix.postorder, lay, words, device, ti)) ti = build_tuple_index(p, ix);
  return ti;
}

Compiled compile_problem(const mtcg_problem& p, const mtcg_options& opt,
                         uint64_t cap_bytes, const std::vector<char>* request_dependent_slots,
                         int index_device) {
  PhaseTimer timer;
  Compiled c;
  c.precision = opt.precision;
  if (opt.precision != MTCG_C64 && opt.precision != MTCG_C128)
    throw DataError("unknown precision mode");
  c.elem_bytes = opt.precision == MTCG_C64 ? 8 : 16;
  if (p.n_nodes < 0 || p.n_slots < 0 || p.n_sliced < 0 || p.n_batch_legs < 0)
    throw DataError("negative array length");
  c.n_nodes = p.n_nodes;
  c.n_slots = p.n_slots;
  c.root = p.root;

  // --- check_inputs (multieval.cpp:284-297) --------------------------------
  const PlanIdx ix = index_plan(p);
  const TupleWords tuple_lay = tuple_word_layout(p);
  static thread_local std::vector<uint64_t> tuple_words;  // packed tuples for the device index
  check_tuples(p, &tuple_lay, index_device >= 0 ? &tuple_words : nullptr);
  for (int j = 0; j < p.n_slots; ++j)
    if (p.slot_n_values[j] < 1)
      throw DataError(fmt("slot %lld has an empty value set", j));

  if (opt.eval_mode == MTCG_EVAL_ALL && p.n_sliced > 0)
    throw DataError("plan has sliced legs; use eval_sliced");
  if (opt.eval_mode == MTCG_EVAL_SLICED && p.n_sliced == 0)
    throw DataError("plan has no sliced legs; use eval_all");

  // --- slice_spec (multieval.cpp:332-348) ----------------------------------
  for (int x = 0; x < p.n_sliced; ++x) {
    const uint32_t l = p.sliced[x];
    if (l >= p.n_legs) throw DataError(fmt("sliced leg %lld does not exist", l));
    if (l >= p.n_closed) throw DataError("output legs cannot be sliced");
    if (contains(c.sliced, l)) throw DataError(fmt("leg %lld sliced twice", l));
    c.sliced.push_back(l);
    c.n_slices *= p.leg_dims[l];
    if (c.n_slices > (1ull << 24))
      throw DataError("slice list expands to more than 2^24 slices");
  }
  const int S = p.n_sliced;

  // --- leaf shapes (check_legs, tensor.cpp:31-40) ---------------------------
  std::vector<std::vector<uint32_t>> slot_layout(p.n_slots);  // stored legs
  for (int j = 0; j < p.n_slots; ++j) {
    for (int i = p.slot_leg_begin[j]; i < p.slot_leg_begin[j + 1]; ++i) {
      const uint32_t l = p.slot_legs[i];
      if (l >= p.n_legs) throw DataError("leg id out of range");
      if (contains(slot_layout[j], l))
        throw DataError(fmt("malformed tensor: duplicate leg %lld", l));
      if (p.leg_dims[l] != 2)
        throw DataError(fmt("leg %lld has bond dimension %lld; this engine "
                            "evaluates qubit networks (dimension 2)",
                            l, p.leg_dims[l]));
      slot_layout[j].push_back(l);
    }
    if (slot_layout[j].size() > 32)
      throw DataError("leaf tensor order above 32 is not supported");
  }
  for (uint32_t l : c.sliced)
    if (p.leg_dims[l] != 2)
      throw DataError(fmt("leg %lld has bond dimension %lld; this engine "
                          "evaluates qubit networks (dimension 2)",
                          l, p.leg_dims[l]));

  // leaf blob: every value tensor as given
  c.slot_base.resize(p.n_slots);
  c.slot_item.resize(p.n_slots);
  uint64_t leaf_elems = 0;
  for (int j = 0; j < p.n_slots; ++j) {
    c.slot_base[j] = leaf_elems;
    c.slot_item[j] = uint64_t{1} << slot_layout[j].size();
    leaf_elems += c.slot_item[j] * static_cast<uint64_t>(p.slot_n_values[j]);
  }
  c.leaf_elems = leaf_elems;
  c.leaf_values.assign(p.values, p.values + 2 * leaf_elems);

  timer.mark("validate+leaves");
  // --- tuple index ----------------------------------------------------------
  TupleIndex ti;
  if (index_device < 0 || !build_tuple_index_device(p, ix.postorder, tuple_lay, tuple_words, index_device, ti))
    ti = build_tuple_index(p, ix);
  c.n_requests = p.n_requests;
  c.n_rows = ti.rows;
  c.row_of_request = ti.row_of_request;
  c.row_mult.assign(ti.rows, 0);
  for (uint64_t r : ti.row_of_request) c.row_mult[r] += 1;

  timer.mark("tuple index");
  // --- logical shapes ----------------------------------------------------------
  const int n = p.n_nodes;
  std::vector<std::vector<uint32_t>> legs(n);  // logical legs (sorted for internal)
  for (int node : ix.postorder) {
    if (p.node_slot[node] >= 0) {
      for (uint32_t l : slot_layout[p.node_slot[node]])
        if (!contains(c.sliced, l)) legs[node].push_back(l);
      continue;
    }
    const auto& L = legs[p.node_left[node]];
    const auto& R = legs[p.node_right[node]];
    std::vector<uint32_t> out;
    for (uint32_t l : L)
      if (!contains(R, l)) out.push_back(l);
    for (uint32_t l : R)
      if (!contains(L, l)) out.push_back(l);
    std::sort(out.begin(), out.end());
    // element offsets inside one table entry are 32-bit (SplitTable)
    if (out.size() > 32) throw DataError("intermediate tensor of order above 32 is not supported");
    legs[node] = std::move(out);
  }
  c.out_legs = legs[p.root];
  c.row_elems = uint64_t{1} << c.out_legs.size();
  if (c.out_legs.size() > 30)
    throw DataError("request tensors of order above 30 are not supported");

  // --- stored layouts -------------------------------------------------------------
  // Top-down. Root: ascending (the observable layout). Other internal nodes:
  // [legs kept by the parent, in the parent's layout order][legs the parent
  // closes, ascending] — the parent contraction reads K-contiguous rows (K in
  // the reference's reduction order), and walking those rows in memory order
  // walks the parent's output in address order, so row-parallel epilogues
  // (tensor-core tiles, streaming kernels) write coalesced.
  std::vector<std::vector<uint32_t>> layout(n);
  for (size_t q = ix.postorder.size(); q-- > 0;) {  // parents before children
    const int node = ix.postorder[q];
    if (p.node_slot[node] >= 0) {
      layout[node] = slot_layout[p.node_slot[node]];
      continue;
    }
    const int par = ix.parent[node];
    if (par < 0) {
      layout[node] = legs[node];
      continue;
    }
    const int sib = p.node_left[par] == node ? p.node_right[par] : p.node_left[par];
    std::vector<uint32_t> keep, close;
    for (uint32_t l : layout[par])  // parent's layout order
      if (contains(legs[node], l)) keep.push_back(l);
    for (uint32_t l : legs[node])
      if (contains(legs[sib], l)) close.push_back(l);  // ascending
    layout[node] = keep;
    layout[node].insert(layout[node].end(), close.begin(), close.end());
  }

  // --- schedule order: post-order, larger-footprint child first -------------------
  std::vector<uint64_t> table_elems(n, 0), peak(n, 0);
  for (int node : ix.postorder) {
    if (p.node_slot[node] >= 0) continue;
    table_elems[node] = static_cast<uint64_t>(ti.distinct[node]) << legs[node].size();
  }
  std::vector<char> left_first(n, 1);
  for (int node : ix.postorder) {
    if (p.node_slot[node] >= 0) continue;
    const int l = p.node_left[node], r = p.node_right[node];
    const uint64_t sl = table_elems[l], sr = table_elems[r];
    const uint64_t pl = std::max(peak[l], sl), pr = std::max(peak[r], sr);
    const uint64_t lf = std::max(pl, sl + pr), rf = std::max(pr, sr + pl);
    left_first[node] = lf <= rf;
    peak[node] = std::max(std::min(lf, rf), sl + sr + table_elems[node]);
  }
  std::vector<int> sched;  // internal nodes in execution order
  {
    std::vector<std::pair<int, int>> st{{p.root, 0}};
    while (!st.empty()) {
      auto& [node, ph] = st.back();
      if (p.node_slot[node] >= 0) {
        st.pop_back();
        continue;
      }
      const int first = left_first[node] ? p.node_left[node] : p.node_right[node];
      const int second = left_first[node] ? p.node_right[node] : p.node_left[node];
      if (ph == 0) {
        ph = 1;
        st.push_back({first, 0});
      } else if (ph == 1) {
        ph = 2;
        st.push_back({second, 0});
      } else {
        sched.push_back(node);
        st.pop_back();
      }
    }
  }

  // --- cross-slice reuse (MTCG_FLAG_SLICE_REUSE) ----------------------------------
  // A node is slice-invariant when no leaf of its subtree carries a sliced
  // leg: its tables are the same in every slice (the reference recomputes
  // them per slice, multieval.cpp:465-476). Invariant nodes are scheduled
  // first (a prologue run once per run range) and the invariant tables read
  // by slice-dependent parents are never released. The C ABI drops the flag
  // under an explicit memory cap (the reference's per-slice accounting is the
  // budget there).
  std::vector<char> invariant(n, 0);
  if ((opt.flags & MTCG_FLAG_SLICE_REUSE) && S > 0) {
    for (int node : ix.postorder) {
      if (p.node_slot[node] >= 0) {
        bool any = false;
        for (uint32_t x : slot_layout[p.node_slot[node]]) any |= contains(c.sliced, x);
        invariant[node] = !any;
      } else {
        invariant[node] = invariant[p.node_left[node]] && invariant[p.node_right[node]];
      }
    }
    std::stable_partition(sched.begin(), sched.end(), [&](int node) { return invariant[node] != 0; });
    for (int node : sched) c.n_prologue_ops += invariant[node] ? 1 : 0;
  } else if (request_dependent_slots) {
    // row-chunked evaluation: request-independent nodes first, in the plan's
    // own post-order (independent of this chunk's tuple counts, so every
    // chunk lays the prologue out identically in the first-fit arena)
    if (static_cast<int>(request_dependent_slots->size()) != p.n_slots)
      throw InternalError("request_dependent_slots size");
    for (int node : ix.postorder) {
      if (p.node_slot[node] >= 0)
        invariant[node] = !(*request_dependent_slots)[p.node_slot[node]];
      else
        invariant[node] = invariant[p.node_left[node]] && invariant[p.node_right[node]];
    }
    std::vector<int> pro, body;
    for (int node : ix.postorder)
      if (p.node_slot[node] < 0 && invariant[node]) pro.push_back(node);
    for (int node : sched)
      if (!invariant[node]) body.push_back(node);
    sched = pro;
    sched.insert(sched.end(), body.begin(), body.end());
    c.n_prologue_ops = pro.size();
    c.row_prologue = true;
  }

  // --- static arena: first-fit over the schedule ---------------------------
  const uint64_t align = 256 / c.elem_bytes;
  std::map<uint64_t, uint64_t> free_blocks;  // offset -> length
  uint64_t arena_top = 0;
  std::vector<uint64_t> arena_off(n, 0);
  std::vector<uint64_t> frontier_row_exp(n, ~uint64_t{0});
  const uint64_t fixed_bytes =
      leaf_elems * c.elem_bytes + 2 * c.n_rows * c.row_elems * c.elem_bytes;
  auto alloc = [&](uint64_t elems, int node) -> uint64_t {
    elems = (elems + align - 1) / align * align;
    for (auto it = free_blocks.begin(); it != free_blocks.end(); ++it)
      if (it->second >= elems) {
        const uint64_t off = it->first, len = it->second;
        free_blocks.erase(it);
        if (len > elems) free_blocks[off + elems] = len - elems;
        return off;
      }
    uint64_t off = arena_top;
    // extend: merge with a trailing free block
    if (!free_blocks.empty()) {
      auto last = std::prev(free_blocks.end());
      if (last->first + last->second == arena_top) {
        off = last->first;
        free_blocks.erase(last);
      }
    }
    arena_top = off + elems;
    if (cap_bytes && arena_top * c.elem_bytes + fixed_bytes > cap_bytes)
      throw MemoryCapError(
          "memory cap exceeded at node " + std::to_string(node) + " (" +
              std::to_string(arena_top * c.elem_bytes + fixed_bytes) + " > " +
              std::to_string(cap_bytes) + " bytes)",
          node);
    return off;
  };
  auto release = [&](uint64_t off, uint64_t elems) {
    elems = (elems + align - 1) / align * align;
    auto [it, ok] = free_blocks.emplace(off, elems);
    (void)ok;
    auto nx = std::next(it);
    if (nx != free_blocks.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_blocks.erase(nx);
    }
    if (it != free_blocks.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_blocks.erase(it);
      }
    }
  };
  if (cap_bytes && fixed_bytes > cap_bytes)
    throw MemoryCapError("memory cap exceeded at node " + std::to_string(p.root) +
                             " (" + std::to_string(fixed_bytes) + " > " +
                             std::to_string(cap_bytes) + " bytes)",
                         p.root);

  // Small tables (and small tensor-core scratch) get private, never-reused
  // space above the first-fit region: ops on independent subtrees then share
  // no memory, so the slice graph's dependencies are the data dependencies
  // (the first-fit region alone chains nearly every op through reuse). Not
  // used under a memory cap, where the reference's accounting (live tables,
  // multieval.cpp:38-47) is the whole budget. MTCG_PRIVATE_MB sets the size
  // limit per table; default 0 (off): on cfg2 it shortens the dependency
  // critical path from 9.7 to 8.6 of 10.2 ms, but the multi-stream graph
  // measured no faster (the small ops compete with the large ones for SMs).
  const uint64_t private_mb = std::getenv("MTCG_PRIVATE_MB") ? std::strtoull(std::getenv("MTCG_PRIVATE_MB"), nullptr, 10) : 0;
  const uint64_t private_elems = cap_bytes ? 0 : (private_mb << 20) / c.elem_bytes;
  uint64_t private_top = 0;
  std::vector<char> node_private(n, 0);
  std::vector<size_t> scratch_private;
  timer.mark("shapes+sched");
  // --- ops ------------------------------------------------------------------------
  // smallest log2 N sent to the tensor cores (MTCG_TC_MIN_FB overrides; tuning)
  const int tc_min_fb = std::getenv("MTCG_TC_MIN_FB") ? std::atoi(std::getenv("MTCG_TC_MIN_FB")) : 4;
  c.node_contractions.assign(n, 0);
  // Per-op item arrays and grouping: functions of the tuple index and the
  // plan only, computed for every node up front — over host threads when the
  // batch is large (10^5 requests: ~3.5 ms single-threaded).
  struct OpPrep {
    std::vector<uint32_t> closed, fl, fr, ia, ib, g_order, g_start, tg_start;
    uint32_t g_max = 0, tc_slots = 0;
    bool a_is_left = false, ga_mode = false;
  };
  std::vector<OpPrep> prep(n);
  auto prepare = [&](int node) {
    OpPrep& pr = prep[node];
    const int l = p.node_left[node], r = p.node_right[node];
    const auto& L = legs[l];
    const auto& R = legs[r];
    std::vector<uint32_t>& closed = pr.closed;
    std::vector<uint32_t>& fl = pr.fl;
    std::vector<uint32_t>& fr = pr.fr;
    for (uint32_t x : L) (contains(R, x) ? closed : fl).push_back(x);
    for (uint32_t x : R)
      if (!contains(L, x)) fr.push_back(x);
    std::sort(closed.begin(), closed.end());
    struct {
      bool a_is_left;
      int fb, kc;
      uint32_t nb;
      std::vector<uint32_t> ia, ib;
    } op;
    op.a_is_left = fl.size() >= fr.size();
    // Tensor-core gather mode (see below): the gathered A side has M = 32 / 64
    // rows per item and the B side is shared (>= 8 items per B entry); pick
    // the orientation that satisfies it, else keep A = the side with more
    // free legs (the CUDA-core kernels assume fa >= fb).
    bool ga_mode = false;
    if (c.precision == MTCG_C64 && !(opt.flags & MTCG_FLAG_NO_TENSOR_CORES) && !std::getenv("MTCG_NO_GATHER") &&
        closed.size() >= 4 && ti.distinct[node] >= 1024 && !std::getenv("MTCG_TC_ONLY")) {
      // ... or a long K (>= 512): even one item per 128-row tile (half or a
      // quarter of the rows padding) beats the CUDA-core tile kernels there
      // (cfg3 candidate plans: 2,500 items of 64 x 64 x 4096)
      auto fits = [&](int ca, const std::vector<uint32_t>& fa_, int cb, const std::vector<uint32_t>& fb_) {
        return p.node_slot[ca] < 0 && (fa_.size() == 5 || fa_.size() == 6) && fb_.size() >= 4 && fb_.size() <= 7 &&
               (uint64_t{ti.distinct[cb]} * 8 <= ti.distinct[node] || (closed.size() >= 9 && closed.size() <= 14));
      };
      if (fits(op.a_is_left ? l : r, op.a_is_left ? fl : fr, op.a_is_left ? r : l, op.a_is_left ? fr : fl)) {
        ga_mode = true;
      } else if (fits(op.a_is_left ? r : l, op.a_is_left ? fr : fl, op.a_is_left ? l : r, op.a_is_left ? fl : fr)) {
        ga_mode = true;
        op.a_is_left = !op.a_is_left;
      }
    }
    const int child_a = op.a_is_left ? l : r, child_b = op.a_is_left ? r : l;
    op.fb = static_cast<int>((op.a_is_left ? fr : fl).size());
    op.kc = static_cast<int>(closed.size());
    op.nb = ti.distinct[node];
    // entry of each child per distinct rank of this node; a leaf's rank is
    // the rank of its value index among the rows (ranks == value indices when
    // every value occurs, which build_assignments guarantees; map explicitly).
    {
      const auto& ra = op.a_is_left ? ti.pair_l[node] : ti.pair_r[node];
      const auto& rb = op.a_is_left ? ti.pair_r[node] : ti.pair_l[node];
      const bool a_leaf = p.node_slot[child_a] >= 0, b_leaf = p.node_slot[child_b] >= 0;
      const auto& va = ti.rank_value[child_a];
      const auto& vb = ti.rank_value[child_b];
      op.ia.resize(op.nb);
      op.ib.resize(op.nb);
      for (uint32_t b = 0; b < op.nb; ++b) {
        op.ia[b] = a_leaf ? va[ra[b]] : ra[b];
        op.ib[b] = b_leaf ? vb[rb[b]] : rb[b];
      }
    }
    // Tensor-core path (complex64 only): dense, K-contiguous intermediate A,
    // shapes the 128 x (2N) x (2K) real tiles cover exactly.
    // Ops with intensity MNK / (MK + NK + MN) >= 6 complex MACs per element
    // moved: above that the CUDA-core kernels are FMA-bound while the tensor
    // path (A read once, split in smem) stays near the HBM roofline; below it
    // the streaming kernels win.
    // Items that share their A entry (a distinct A rank feeding several
    // distinct ranks of this node) form groups (CSR by A entry) so each A row
    // streams from HBM once per group: the group is one GEMM whose N is the
    // concatenation of its items' B blocks (N_eff = slots x N, slots = the
    // largest group, padded so 2 N_eff is a multiple of 32 for the tensor
    // path). MTCG_NO_GROUP=1 disables grouping (A/B tuning).
    std::vector<uint32_t>& g_order = pr.g_order;
    std::vector<uint32_t>& g_start = pr.g_start;
    uint32_t& g_max = pr.g_max;
    if (op.nb >= 2 && !std::getenv("MTCG_NO_GROUP")) {
      g_order = order_by_key(op.ia);
      g_start.push_back(0);
      for (uint32_t i = 1; i <= op.nb; ++i)
        if (i == op.nb || op.ia[g_order[i]] != op.ia[g_order[i - 1]]) {
          g_max = std::max(g_max, i - g_start.back());
          g_start.push_back(i);
        }
      if (2 * uint64_t{op.nb} < 3 * (g_start.size() - 1)) {  // < 1.5 items per group
        g_order.clear();
        g_start.clear();
        g_max = 0;
      }
    }
    // Tensor-path groups: every unit is padded to `tc_slots` item blocks, and
    // the epilogue drains the padding too, so large groups are cut into
    // sub-groups of S items with S minimising units x (K + S N) — one A row
    // read per unit plus S item blocks drained per row (S = 1: no grouping).
    // 2 N S must be a multiple of 32 real columns.
    std::vector<uint32_t>& tg_start = pr.tg_start;
    uint32_t& tc_slots = pr.tc_slots;
    if (g_max > 0) {
      const uint32_t q = op.fb < 4 ? 16u >> op.fb : 1u;  // slots per 32 real columns
      const double Kd = std::ldexp(1.0, op.kc), Nd = std::ldexp(1.0, op.fb);
      double best = 0;
      for (uint32_t S = q; S < 2 * std::max(g_max, q); S *= 2) {
        uint64_t units_s = 0;
        for (size_t g = 0; g + 1 < g_start.size(); ++g) units_s += (g_start[g + 1] - g_start[g] + S - 1) / S;
        const double cost = double(units_s) * (Kd + S * Nd);
        if (tc_slots == 0 || cost < best) {
          best = cost;
          tc_slots = S;
        }
      }
      if (tc_slots > 1) {
        tg_start.push_back(0);
        for (size_t g = 0; g + 1 < g_start.size(); ++g)
          for (uint32_t i = g_start[g] + tc_slots; i < g_start[g + 1] + tc_slots; i += tc_slots)
            tg_start.push_back(std::min(i, g_start[g + 1]));
      } else {
        tc_slots = 0;
      }
    }
    pr.a_is_left = op.a_is_left;
    pr.ga_mode = ga_mode;
    pr.ia = std::move(op.ia);
    pr.ib = std::move(op.ib);
  };
  {
    uint64_t items = 0;
    for (int node : sched) items += ti.distinct[node];
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nt = items >= (uint64_t{1} << 17) ? std::min<unsigned>(hw, static_cast<unsigned>(sched.size())) : 1;
    if (nt <= 1) {
      for (int node : sched) prepare(node);
    } else {
      // nodes handed out largest first (one 10^5-item node is most of the work)
      std::vector<int> order(sched.begin(), sched.end());
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ti.distinct[x] > ti.distinct[y]; });
      std::atomic<size_t> next{0};
      std::exception_ptr err;
      std::mutex err_mu;
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&] {
          try {
            for (size_t i; (i = next.fetch_add(1)) < order.size();) prepare(order[i]);
          } catch (...) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!err) err = std::current_exception();
          }
        });
      for (auto& x : th) x.join();
      if (err) std::rethrow_exception(err);
    }
  }
  SectionTimer sec;
  for (int node : sched) {
    sec.start();
    OpPrep& pr = prep[node];
    const int l = p.node_left[node], r = p.node_right[node];
    const std::vector<uint32_t> closed = std::move(pr.closed), fl = std::move(pr.fl), fr = std::move(pr.fr);

    Op op;
    op.node = node;
    op.a_is_left = pr.a_is_left;
    const bool ga_mode = pr.ga_mode;
    op.child_a = op.a_is_left ? l : r;
    op.child_b = op.a_is_left ? r : l;
    const auto& fa_legs = op.a_is_left ? fl : fr;
    const auto& fb_legs = op.a_is_left ? fr : fl;
    op.fa = static_cast<int>(fa_legs.size());
    op.fb = static_cast<int>(fb_legs.size());
    op.kc = static_cast<int>(closed.size());
    op.nb = ti.distinct[node];
    op.root = node == p.root;
    const auto& out_layout = layout[node];

    // operand sources (per-item entries: prep)
    auto setup_operand = [&](int child, bool& is_leaf, uint64_t& base, uint64_t& item) {
      is_leaf = p.node_slot[child] >= 0;
      if (is_leaf) {
        const int slot = p.node_slot[child];
        base = c.slot_base[slot];
        item = c.slot_item[slot];
      } else {
        base = arena_off[child];
        item = uint64_t{1} << legs[child].size();
      }
    };
    setup_operand(op.child_a, op.a_leaf, op.a_base, op.a_item);
    setup_operand(op.child_b, op.b_leaf, op.b_base, op.b_item);
    op.ia = std::move(pr.ia);
    op.ib = std::move(pr.ib);
    sec.lap(0);
    const auto& a_layout = layout[op.child_a];
    const auto& b_layout = layout[op.child_b];
    // m / n bit orders: free legs by increasing address in the output layout
    auto by_out_addr = [&](std::vector<uint32_t> v) {
      std::sort(v.begin(), v.end(), [&](uint32_t x, uint32_t y) {
        return stride_in(out_layout, x) < stride_in(out_layout, y);
      });
      return v;
    };
    op.config = select_config(op.fa, op.fb, op.kc);
    if (op.config == kGenericConfig && c.precision == MTCG_C64 && op.kc >= 6) op.config = kDotConfig;
    std::vector<uint32_t> g_order = std::move(pr.g_order), g_start = std::move(pr.g_start),
                          tg_start = std::move(pr.tg_start);
    const uint32_t g_max = pr.g_max, tc_slots = pr.tc_slots;
    const bool grouped = tc_slots > 0;
    // Tensor-core path (complex64 only): dense, K-contiguous intermediate A,
    // shapes the 128 x (2N) x (2K) real tiles cover exactly.
    // Ops with intensity MNK / (MK + NK + MN) >= 6 complex MACs per element
    // moved: above that the CUDA-core kernels are FMA-bound while the tensor
    // path (A read once, split in smem) stays near the HBM roofline; below it
    // the streaming kernels win. Grouped ops are judged on N_eff and need
    // M >= 4096 (short groups are dominated by per-unit epilogue/B̂ setup).
    const int fb_eff = grouped ? op.fb + static_cast<int>(std::ceil(std::log2(double(tc_slots))))
                               : op.fb;
    const double Md = std::ldexp(1.0, op.fa), Nd = std::ldexp(1.0, fb_eff),
                 Kd = std::ldexp(1.0, op.kc);
    const double intensity = Md * Nd * Kd / (Md * Kd + Nd * Kd + Md * Nd);
    const uint64_t units = grouped ? uint64_t{tg_start.size() - 1} : op.nb;
    const bool tc_ok = c.precision == MTCG_C64 && !(opt.flags & MTCG_FLAG_NO_TENSOR_CORES) &&
                       !op.a_leaf && op.fa >= 7 && fb_eff >= tc_min_fb && op.kc >= 4 &&
                       fb_eff <= 12 && op.kc <= 14 && intensity >= 6.0 && (!grouped || op.fa >= 12) &&
                       (units << (op.fa + fb_eff + op.kc)) >= (uint64_t{1} << 26);
    // MTCG_TC_ONLY=<node>[,<node>...] restricts the tensor path (diagnostics)
    const char* tc_only = std::getenv("MTCG_TC_ONLY");
    bool tc_listed = true;
    if (tc_only) {
      tc_listed = false;
      for (const char* s = tc_only; *s;) {
        char* end = nullptr;
        const long v = std::strtol(s, &end, 10);
        if (end == s) break;
        tc_listed |= v == node;
        s = *end ? end + 1 : end;
      }
    }
    // MTCG_TC_SKIP=<node>[,<node>...] keeps those nodes off the tensor path
    if (const char* tc_skip = std::getenv("MTCG_TC_SKIP")) {
      for (const char* s = tc_skip; *s;) {
        char* end = nullptr;
        const long v = std::strtol(s, &end, 10);
        if (end == s) break;
        if (v == node) tc_listed = false;
        s = *end ? end + 1 : end;
      }
    }
    // Gather mode: M = 32 / 64 rows per item is too short for a 128-row
    // tensor tile, but when many items share few B entries (cfg2 node 349:
    // 9,992 items of 32 x 32 x 128 over 128 B entries) the items of one B
    // entry stack into 128-row tiles against one B̂ (MTCG_NO_GATHER=1 off).
    const bool ga_ok = ga_mode && !(tc_ok && tc_listed);
    if (tc_ok && tc_listed && !ga_mode) {
      op.config = kTcConfig;
      if (grouped) op.grp_max = tc_slots;
    } else if (ga_ok) {
      op.config = kTcConfig;
      const uint32_t per = 128u >> op.fa;  // items per tile
      const std::vector<uint32_t> order = order_by_key(op.ib);
      for (size_t s0 = 0; s0 < order.size();) {
        size_t s1 = s0;
        while (s1 < order.size() && op.ib[order[s1]] == op.ib[order[s0]]) ++s1;
        const uint32_t g = static_cast<uint32_t>(op.ga_groups.size());
        op.ga_groups.push_back(op.ib[order[s0]]);
        for (size_t t0 = s0; t0 < s1; t0 += per) {
          op.ga_tiles.push_back(g);
          for (uint32_t k = 0; k < per; ++k)
            op.ga_tiles.push_back(t0 + k < s1 ? order[t0 + k] : ~0u);
        }
        s0 = s1;
      }
    } else if (g_max > 0 && op.fb <= 4 && op.kc <= 5 && op.fa >= 8 &&
               ((uint64_t{g_max} << (op.fb + op.kc)) * c.elem_bytes) <= kGroupSmemBytes) {
      op.config = kRowsGroupedConfig;
      op.grp_max = g_max;
    }
    if (op.grp_max) {
      op.grp_items = std::move(g_order);
      op.grp_start = op.config == kTcConfig ? std::move(tg_start) : std::move(g_start);
    }
    sec.lap(1);
    // m / n bit orders: free legs by increasing address in the output layout;
    // the tensor-core path walks A rows in A's memory order instead (TMA rows)
    std::vector<uint32_t> m_legs = by_out_addr(fa_legs);
    if (op.config == kTcConfig)
      std::sort(m_legs.begin(), m_legs.end(), [&](uint32_t x, uint32_t y) {
        return stride_in(layout[op.child_a], x) < stride_in(layout[op.child_a], y);
      });
    const std::vector<uint32_t> n_legs = by_out_addr(fb_legs);
    // k bit order: reference reduction order (ascending ids, row-major):
    // bit 0 of k is the highest-id closed leg
    std::vector<uint32_t> k_legs(closed.rbegin(), closed.rend());

    auto strides_of = [&](const std::vector<uint32_t>& space,
                          const std::vector<uint32_t>& lay) {
      std::vector<uint64_t> s;
      for (uint32_t x : space) s.push_back(contains(lay, x) ? stride_in(lay, x) : 0);
      return s;
    };
    // long-K small tiles (cfg3 node 619: 16 x 16 x 16384 per item) stream
    // both operands once instead of through 16 x 16 smem k-steps (decided
    // before the tables: per-element kernels index them by output position)
    if (c.precision == MTCG_C64 && op.config != kTcConfig && op.grp_max == 0 && op.fa >= 2 && op.fa <= 4 &&
        op.fb >= 3 && op.fb <= 4 && op.kc >= 9 && !op.a_leaf && !op.b_leaf && !std::getenv("MTCG_NO_LONGK")) {
      bool kc_a = true, kc_b = true;
      const auto ka = strides_of(k_legs, a_layout), kb = strides_of(k_legs, b_layout);
      for (size_t b = 0; b < ka.size(); ++b) kc_a &= ka[b] == (uint64_t{1} << b);
      for (size_t b = 0; b < kb.size(); ++b) kc_b &= kb[b] == (uint64_t{1} << b);
      if (kc_a && kc_b) op.config = kLongKConfig;
    }
    if (op.config == kGenericConfig || op.config == kDotConfig) {
      // per-output-element kernels: index the stored output directly
      std::vector<uint32_t> o_legs(out_layout.rbegin(), out_layout.rend());
      op.tam.build(strides_of(o_legs, a_layout));   // A offset per out index
      op.tbn.build(strides_of(o_legs, b_layout));   // B offset per out index
      op.tom.build({});
      op.ton.build({});
    } else {
      op.tam.build(strides_of(m_legs, a_layout));
      op.tbn.build(strides_of(n_legs, b_layout));
      op.tom.build(strides_of(m_legs, out_layout));
      op.ton.build(strides_of(n_legs, out_layout));
    }
    op.tak.build(strides_of(k_legs, a_layout));
    op.tbk.build(strides_of(k_legs, b_layout));
    op.store_n_fast = out_layout.empty() || contains(fb_legs, out_layout.back());
    {
      const auto ks = strides_of(k_legs, a_layout);
      op.a_kcontig = !op.a_leaf;
      for (size_t b = 0; b < ks.size(); ++b) op.a_kcontig &= ks[b] == (uint64_t{1} << b);
      const auto kb = strides_of(k_legs, b_layout);
      op.b_kcontig = !op.b_leaf;
      for (size_t b = 0; b < kb.size(); ++b) op.b_kcontig &= kb[b] == (uint64_t{1} << b);
      const auto ns = strides_of(n_legs, out_layout);
      op.o_ncontig = op.config != kGenericConfig && op.config != kDotConfig;
      for (size_t b = 0; b < ns.size(); ++b) op.o_ncontig &= ns[b] == (uint64_t{1} << b);
      const auto ms = strides_of(m_legs, out_layout);
      op.o_mcontig = !ms.empty() && ms[0] == 1;
    }

    sec.lap(2);
    // sliced legs carried by leaf operands: offsets per set bit of the slice
    auto slice_strides = [&](int child, std::vector<uint64_t>& v) {
      if (p.node_slot[child] < 0 || S == 0) return false;
      bool any = false;
      v.assign(S, 0);
      for (int x = 0; x < S; ++x) {
        const uint32_t leg = c.sliced[x];
        if (contains(layout[child], leg)) {
          v[S - 1 - x] = stride_in(layout[child], leg);  // bit S-1-x of idx
          any = true;
        }
      }
      return any;
    };
    const bool sa = slice_strides(op.child_a, op.a_slice_stride);
    const bool sb = slice_strides(op.child_b, op.b_slice_stride);
    if (sa || sb) op.slice_slot = c.n_slice_slots++;

    // exact counts (predicted_cost, tensor.cpp:132-148)
    const uint64_t d_closed = uint64_t{1} << op.kc;
    const uint64_t d_open = uint64_t{1} << (op.fa + op.fb);
    op.mults = d_closed * d_open;
    op.adds = (d_closed - 1) * d_open;
    op.rw = (uint64_t{1} << legs[l].size()) + (uint64_t{1} << legs[r].size()) + d_open;
    c.node_contractions[node] = static_cast<uint64_t>(op.nb) * c.n_slices;
    c.mults += op.mults * op.nb * c.n_slices;
    c.adds += op.adds * op.nb * c.n_slices;
    c.rw += op.rw * op.nb * c.n_slices;
    c.contractions += static_cast<uint64_t>(op.nb) * c.n_slices;
    c.executed_contractions += static_cast<uint64_t>(op.nb) * (invariant[node] ? 1 : c.n_slices);

    sec.lap(3);
    // output storage
    op.out_item = d_open;
    if (op.root) {
      op.out_rows.resize(op.nb);
      const uint32_t* rk = ti.rank[node];
      for (uint64_t row = 0; row < ti.rows; ++row) op.out_rows[rk[row]] = row;
    } else if (op.nb > 0) {
      if (table_elems[node] <= private_elems) {
        node_private[node] = 1;
        arena_off[node] = private_top;
        private_top += (table_elems[node] + align - 1) / align * align;
      } else {
        arena_off[node] = alloc(table_elems[node], node);
      }
      op.out_base = arena_off[node];
      // A frontier table (invariant, read by a dependent parent every slice /
      // chunk) may be a tensor-core A operand quantized once in place after
      // the prologue: its row exponents (one byte per row of the parent's
      // view) get a resident slot here, in the prologue's allocation sequence
      const int par = ix.parent[node];
      if (invariant[node] && par >= 0 && !invariant[par]) {
        const int sib = p.node_left[par] == node ? p.node_right[par] : p.node_left[par];
        int kc = 0;
        for (uint32_t x : legs[node]) kc += contains(legs[sib], x) ? 1 : 0;
        const uint64_t rows = table_elems[node] >> kc;
        frontier_row_exp[node] = alloc((rows + c.elem_bytes - 1) / c.elem_bytes, node);
      }
    }
    if (op.config == kTcConfig && op.nb > 0) {
      // scratch: B̂ hi/lo (2N x 2K floats per item each)
      op.a_entries = ti.distinct[op.child_a];
      const uint64_t units = !op.ga_groups.empty() ? uint64_t{op.ga_groups.size()}
                             : op.grp_max ? uint64_t{op.grp_start.size() - 1} * op.grp_max : op.nb;
      const uint64_t bhat = units << (op.fb + op.kc + 1);
      // B̂ hi / lo (3xFP16 / 3xTF32; the split-integer digit planes use both)
      // + 4 KB of operand-max partials + the split-integer column exponents
      // (one byte per B̂ column pair) and A row exponents (one per A row)
      const uint64_t col_exps = units << op.fb, row_exps = op.a_entries << op.fa;
      // (kc > 5: A rows quantized by a pre-pass, tc_i8_prequant)
      op.a_prequant = invariant[op.child_a] && !invariant[node] && op.kc > 5;
      op.scratch_elems = 2 * bhat + 4096 / c.elem_bytes +
                         (col_exps + (op.a_prequant ? 0 : row_exps) + c.elem_bytes) / c.elem_bytes + 1;
      // (prologue-written, read by every slice: the slot reserved when the
      // frontier table was allocated)
      if (op.a_prequant) {
        if (frontier_row_exp[op.child_a] == ~uint64_t{0}) throw InternalError("frontier row exponents");
        op.row_exp_off = frontier_row_exp[op.child_a];
      }
      if (op.scratch_elems <= private_elems) {
        scratch_private.push_back(c.ops.size());
        op.scratch_off = private_top;
        private_top += (op.scratch_elems + align - 1) / align * align;
      } else {
        op.scratch_off = alloc(op.scratch_elems, node);
        release(op.scratch_off, op.scratch_elems);  // free again once the op is done
      }
    }
    // children are dead once consumed
    // (invariant tables read by a slice-dependent parent live across slices)
    for (int ch : {l, r})
      if (p.node_slot[ch] < 0 && ti.distinct[ch] > 0 && !node_private[ch] &&
          !(invariant[ch] && !invariant[node]))
        release(arena_off[ch], table_elems[ch]);
    c.ops.push_back(std::move(op));
    sec.lap(4);
  }
  {
    static const char* const names[] = {"operands", "kernel choice", "tables", "slice+counts",
                                        "storage"};
    sec.print(names, 5);
  }
  // private tables sit above the first-fit region
  for (Op& op : c.ops) {
    if (!op.a_leaf && node_private[op.child_a]) op.a_base += arena_top;
    if (!op.b_leaf && node_private[op.child_b]) op.b_base += arena_top;
    if (!op.root && node_private[op.node]) op.out_base += arena_top;
  }
  for (size_t i : scratch_private) c.ops[i].scratch_off += arena_top;
  c.arena_elems = arena_top + private_top;
  c.private_elems = private_top;
  // --- fused operand chains ---------------------------------------------------------
  // Runs of consecutive skinny ops (CUDA-core configs, K <= 8, N <= 8) where
  // each op's A is the previous op's table and the items map one-to-one: one
  // kernel keeps the running tensor block in shared memory (Chain). Members
  // are consecutive in the schedule, so the tables they read (the head's A,
  // every step's B) are still intact when the tail launches. Within one
  // slice-reuse segment only.
  if (!std::getenv("MTCG_NO_CHAIN")) {
    std::vector<int> op_of(n, -1);
    for (size_t i = 0; i < c.ops.size(); ++i) op_of[c.ops[i].node] = static_cast<int>(i);
    auto eligible = [&](const Op& op) {
      return !op.root && op.nb > 0 && op.kc <= 3 && op.fb <= 3 && op.config != kTcConfig &&
             op.config != kDotConfig && op.config != kRowsGroupedConfig;
    };
    auto bijective = [&](const Op& op) {
      std::vector<char> seen(op.nb, 0);
      for (uint32_t v : op.ia) {
        if (v >= op.nb || seen[v]) return false;
        seen[v] = 1;
      }
      return true;
    };
    auto linked = [&](size_t i) {  // op i+1 continues op i
      const Op& a = c.ops[i];
      const Op& b = c.ops[i + 1];
      const bool seg = (i < c.n_prologue_ops) == (i + 1 < c.n_prologue_ops) &&
                       // row-chunked plans: a chain's tail table lives in a
                       // region placed after the plan's own arena, which
                       // differs between chunk plans, so the shared prologue
                       // has no chains
                       !(c.row_prologue && i < c.n_prologue_ops);
      return seg && eligible(a) && eligible(b) && !b.a_leaf && op_of[b.child_a] == static_cast<int>(i) &&
             a.nb == b.nb && bijective(b);
    };
    const int q_max = 8;
    size_t i = 0;
    while (i + 1 < c.ops.size()) {
      if (!linked(i) || c.ops[i].a_leaf) {
        ++i;
        continue;
      }
      // extend while the touched legs fit q_max positions: all T0 legs the
      // run closes are loaded up front, each step then closes some touched
      // legs and opens its B's new legs
      const int t0 = c.ops[i].child_a;
      const std::vector<uint32_t>& T = legs[t0];
      auto chain_q = [&](size_t k) {
        std::vector<uint32_t> cur(T), qin;
        for (size_t s = i; s <= k; ++s) {
          const auto& bl = legs[c.ops[s].child_b];
          std::vector<uint32_t> next;
          for (uint32_t x : cur)
            if (!contains(bl, x)) next.push_back(x);
            else if (contains(T, x)) qin.push_back(x);
          for (uint32_t x : bl)
            if (!contains(cur, x)) next.push_back(x);
          cur = next;
        }
        std::vector<uint32_t> active(qin);
        size_t qm = active.size();
        cur = T;
        for (size_t s = i; s <= k; ++s) {
          const auto& bl = legs[c.ops[s].child_b];
          std::vector<uint32_t> next, na;
          for (uint32_t x : cur)
            if (!contains(bl, x)) next.push_back(x);
          for (uint32_t x : active)
            if (!contains(bl, x)) na.push_back(x);
          for (uint32_t x : bl)
            if (!contains(cur, x)) {
              next.push_back(x);
              na.push_back(x);
            }
          cur = next;
          active = na;
          qm = std::max(qm, active.size());
        }
        return static_cast<int>(qm);
      };
      int best_end = -1;
      for (size_t k = i + 1; k < c.ops.size() && linked(k - 1) && k - i < kMaxChainSteps; ++k) {
        if (chain_q(k) > q_max) break;
        best_end = static_cast<int>(k);
      }
      if (best_end < 0) {
        ++i;
        continue;
      }
      const size_t j = static_cast<size_t>(best_end);
      // ---- build the chain over ops [i, j] ----
      Chain ch;
      ch.head = static_cast<int>(i);
      ch.tail = static_cast<int>(j);
      const auto& l0 = layout[t0];
      // Q_in: T0 legs some step closes, by T0 stride ascending
      std::vector<uint32_t> cur(T);
      std::vector<uint32_t> qin;
      {
        std::vector<uint32_t> tmp(T);
        for (size_t s = i; s <= j; ++s) {
          const auto& bl = legs[c.ops[s].child_b];
          std::vector<uint32_t> next;
          for (uint32_t x : tmp)
            if (!contains(bl, x)) next.push_back(x);
            else if (contains(T, x) && !contains(qin, x)) qin.push_back(x);
          for (uint32_t x : bl)
            if (!contains(tmp, x)) next.push_back(x);
          tmp = next;
        }
      }
      std::sort(qin.begin(), qin.end(),
                [&](uint32_t x, uint32_t y) { return stride_in(l0, x) < stride_in(l0, y); });
      std::map<uint32_t, int> pos;  // touched leg -> position
      for (size_t b = 0; b < qin.size(); ++b) pos[qin[b]] = static_cast<int>(b);
      const std::map<uint32_t, int> pos0 = pos;
      int q = static_cast<int>(qin.size());
      std::vector<uint32_t> active(qin);
      for (size_t s = i; s <= j; ++s) {
        const Op& op = c.ops[s];
        const auto& bl = legs[op.child_b];
        const auto& blay = layout[op.child_b];
        std::vector<uint32_t> closed, opened, kept;
        for (uint32_t x : bl) (contains(cur, x) ? closed : opened).push_back(x);
        std::sort(closed.begin(), closed.end());
        std::sort(opened.begin(), opened.end());
        for (uint32_t x : active)
          if (!contains(closed, x)) kept.push_back(x);
        // positions after the step: kept legs stay, opened legs take the
        // lowest free positions (closed ones included — a separate buffer)
        std::map<uint32_t, int> npos;
        std::vector<char> used(64, 0);
        for (uint32_t x : kept) {
          npos[x] = pos[x];
          used[pos[x]] = 1;
        }
        for (uint32_t x : opened) {
          int p_ = 0;
          while (used[p_]) ++p_;
          used[p_] = 1;
          npos[x] = p_;
          q = std::max(q, p_ + 1);
        }
        // output combination o = f + (g << |kept|): f over the kept touched
        // legs (lowest positions first), g over the opened legs
        std::sort(kept.begin(), kept.end(), [&](uint32_t x, uint32_t y) { return pos[x] < pos[y]; });
        std::vector<uint32_t> out_legs(kept);
        out_legs.insert(out_legs.end(), opened.begin(), opened.end());
        ChainStep st;
        st.op = static_cast<int>(s);
        st.kc = static_cast<int>(closed.size());
        st.n_out = 1u << out_legs.size();
        // B tile: (closed combo c, opened combo g) at c * G + g, loaded from
        // the entry at boff[c * G + g]
        const uint32_t G = 1u << opened.size(), F = 1u << kept.size();
        std::vector<uint32_t> in_base(F), out_g(G);  // (kept legs keep their positions)
        for (uint32_t f = 0; f < F; ++f)
          for (size_t x = 0; x < kept.size(); ++x)
            if (f >> x & 1) in_base[f] += 1u << pos[kept[x]];
        for (uint32_t g = 0; g < G; ++g)
          for (size_t x = 0; x < opened.size(); ++x)
            if (g >> x & 1) out_g[g] += 1u << npos[opened[x]];
        // reduction order: ascending closed ids, row-major (bit 0 = highest id)
        std::vector<uint32_t> k_legs(closed.rbegin(), closed.rend());
        const uint32_t K = 1u << k_legs.size();
        std::vector<uint32_t> in_c(K), boff(K * G);
        for (uint32_t cc = 0; cc < K; ++cc) {
          uint32_t coff = 0;
          for (size_t x = 0; x < k_legs.size(); ++x)
            if (cc >> x & 1) {
              in_c[cc] += 1u << pos[k_legs[x]];
              coff += static_cast<uint32_t>(stride_in(blay, k_legs[x]));
            }
          for (uint32_t g = 0; g < G; ++g) {
            uint32_t goff = 0;
            for (size_t x = 0; x < opened.size(); ++x)
              if (g >> x & 1) goff += static_cast<uint32_t>(stride_in(blay, opened[x]));
            boff[cc * G + g] = coff + goff;
          }
        }
        st.g_bits = static_cast<int>(opened.size());
        st.f_bits = static_cast<int>(kept.size());
        for (auto* v : {&in_base, &out_g, &in_c, &boff})
          st.tbl.insert(st.tbl.end(), v->begin(), v->end());
        ch.steps.push_back(std::move(st));
        std::vector<uint32_t> next;
        for (uint32_t x : cur)
          if (!contains(closed, x)) next.push_back(x);
        for (uint32_t x : opened) next.push_back(x);
        cur = next;
        active = out_legs;
        pos = npos;
      }
      ch.q = q;
      // untouched legs: T0's legs outside Q_in == the tail's legs outside active
      const int tl = c.ops[j].node;
      const auto& lt = layout[tl];
      std::vector<uint32_t> U;
      for (uint32_t x : T)
        if (!contains(qin, x)) U.push_back(x);
      bool consistent = U.size() + active.size() == lt.size();
      for (uint32_t x : U) consistent &= contains(lt, x);
      if (!consistent) throw InternalError("operand chain: leg bookkeeping mismatch");
      // A block takes 2^cb combinations of the "inner" untouched legs: the
      // lowest-stride ones of the input AND of the output layout, alternating,
      // so both its loads and its stores run over contiguous memory (the
      // touched legs fill 2^q positions per combination; 2^(cb+q) <= 4096
      // elements per buffer in complex64, 2048 in complex128).
      auto by = [&](const std::vector<uint32_t>& lay) {
        std::vector<uint32_t> v(U);
        std::sort(v.begin(), v.end(), [&](uint32_t x, uint32_t y) { return stride_in(lay, x) < stride_in(lay, y); });
        return v;
      };
      const std::vector<uint32_t> u_in = by(l0), u_out = by(lt);
      const int cb_max = std::max(0, (c.elem_bytes == 8 ? 11 : 10) - q);
      std::vector<uint32_t> inner;
      for (size_t r = 0; static_cast<int>(inner.size()) < std::min<int>(cb_max, static_cast<int>(U.size())); ++r) {
        if (r < u_out.size() && !contains(inner, u_out[r])) inner.push_back(u_out[r]);
        if (static_cast<int>(inner.size()) < cb_max && r < u_in.size() && !contains(inner, u_in[r]))
          inner.push_back(u_in[r]);
      }
      std::vector<uint32_t> outer;
      for (uint32_t x : u_out)
        if (!contains(inner, x)) outer.push_back(x);
      ch.u_bits = static_cast<int>(U.size());
      ch.u_inner_bits = static_cast<int>(inner.size());
      {
        std::vector<uint64_t> si, so;
        for (uint32_t x : outer) {
          si.push_back(stride_in(l0, x));
          so.push_back(stride_in(lt, x));
        }
        ch.tu_in.build(si);
        ch.tu_out.build(so);
      }
      // load / store maps over (inner untouched legs x touched legs), in
      // address order: (shared-memory position, element offset in the block)
      auto block_map = [&](const std::vector<uint32_t>& touched, const std::vector<uint32_t>& lay,
                           const std::map<uint32_t, int>& tpos, std::vector<uint32_t>& out) {
        std::vector<uint32_t> all(inner);
        all.insert(all.end(), touched.begin(), touched.end());
        std::sort(all.begin(), all.end(), [&](uint32_t x, uint32_t y) { return stride_in(lay, x) < stride_in(lay, y); });
        // per bit of the block index: its shared-memory position and its
        // element offset (rows of 2^q + 1 elements: an odd pitch spreads rows
        // over the banks)
        for (uint32_t leg : all) {
          auto it = std::find(inner.begin(), inner.end(), leg);
          out.push_back(it != inner.end() ? ((1u << q) + 1) << static_cast<int>(it - inner.begin())
                                          : 1u << tpos.at(leg));
          out.push_back(static_cast<uint32_t>(stride_in(lay, leg)));
        }
      };
      block_map(qin, l0, pos0, ch.qin);
      block_map(active, lt, pos, ch.qout);
      // entries per final item: back through the one-to-one item maps
      const uint32_t nb = c.ops[j].nb;
      const size_t L = j - i + 1;
      ch.entries.assign((L + 1) * nb, 0);
      for (uint32_t b = 0; b < nb; ++b) {
        uint32_t it = b;
        for (size_t s = j + 1; s-- > i;) {
          ch.entries[(s - i + 1) * nb + b] = c.ops[s].ib[it];
          if (s > i) it = c.ops[s].ia[it];
          else ch.entries[b] = c.ops[s].ia[it];
        }
      }
      const int ci = static_cast<int>(c.chains.size());
      for (size_t s = i; s <= j; ++s) c.ops[s].chain = ci;
      c.ops[j].chain_tail = true;
      if (std::getenv("MTCG_DUMP_OPS")) {
        std::fprintf(stderr, "[mtcg] chain:");
        for (size_t s2 = i; s2 <= j; ++s2) std::fprintf(stderr, " %d", c.ops[s2].node);
        std::fprintf(stderr, "  q %d u_bits %d inner %d items %u\n", ch.q, ch.u_bits, ch.u_inner_bits, nb);
        std::fprintf(stderr, "[mtcg]   ld bit strides:");
        for (size_t e = 0; e < ch.qin.size() / 2; ++e) std::fprintf(stderr, " %u", ch.qin[2 * e + 1]);
        std::fprintf(stderr, "\n[mtcg]   st bit strides:");
        for (size_t e = 0; e < ch.qout.size() / 2; ++e) std::fprintf(stderr, " %u", ch.qout[2 * e + 1]);
        std::fprintf(stderr, "\n");
      }
      c.chains.push_back(std::move(ch));
      i = j + 1;
    }
    // Each tail writes its table into its own region above the arena: in the
    // first-fit arena it could overlap the head's A or a step's B, which the
    // chain kernel still reads while it writes (members write nothing, so
    // nothing else changes). Chains are dropped if that does not fit the cap.
    uint64_t top = c.arena_elems;
    for (const Chain& ch : c.chains) top += (table_elems[c.ops[ch.tail].node] + align - 1) / align * align;
    if (cap_bytes && top * c.elem_bytes + fixed_bytes > cap_bytes) {
      for (Op& op : c.ops) {
        op.chain = -1;
        op.chain_tail = false;
      }
      c.chains.clear();
    }
    top = c.arena_elems;
    for (Chain& ch : c.chains) {
      const int tn = c.ops[ch.tail].node;
      ch.out_base = top;
      c.ops[ch.tail].out_base = top;
      for (Op& o : c.ops) {
        if (!o.a_leaf && o.child_a == tn) o.a_base = top;
        if (!o.b_leaf && o.child_b == tn) o.b_base = top;
      }
      top += (table_elems[tn] + align - 1) / align * align;
    }
    c.arena_elems = top;
  }

  // --- dependencies between ops (arena read/write ranges) ---------------------
  {
    struct Access {
      uint64_t lo, hi;
      int op;
      bool write;
    };
    std::vector<Access> seen;
    std::vector<int> op_of_node(n, -1);
    for (size_t i = 0; i < c.ops.size(); ++i) op_of_node[c.ops[i].node] = static_cast<int>(i);
    for (size_t i = 0; i < c.ops.size(); ++i) {
      Op& op = c.ops[i];
      // fused chains: members launch nothing; the tail performs every
      // member's operand reads
      if (op.chain >= 0 && !op.chain_tail) continue;
      std::vector<std::pair<uint64_t, uint64_t>> reads, writes;
      const size_t first = op.chain >= 0 ? static_cast<size_t>(c.chains[op.chain].head) : i;
      for (size_t m = first; m <= i; ++m) {
        const Op& mo = c.ops[m];
        if (!mo.a_leaf && table_elems[mo.child_a]) reads.push_back({mo.a_base, mo.a_base + table_elems[mo.child_a]});
        if (!mo.b_leaf && table_elems[mo.child_b]) reads.push_back({mo.b_base, mo.b_base + table_elems[mo.child_b]});
      }
      if (!op.root && table_elems[op.node]) writes.push_back({op.out_base, op.out_base + table_elems[op.node]});
      if (op.scratch_elems) writes.push_back({op.scratch_off, op.scratch_off + op.scratch_elems});
      std::vector<int> deps;
      for (const Access& a : seen) {
        bool hit = false;
        for (const auto& r : reads) hit |= a.write && a.lo < r.second && r.first < a.hi;
        for (const auto& w : writes) hit |= a.lo < w.second && w.first < a.hi;
        if (hit && c.ops[a.op].nb > 0) deps.push_back(a.op);
      }
      // operand producers (also covered by their write records; explicit for
      // zero-size tables)
      for (size_t m = first; m <= i; ++m)
        for (int ch : {c.ops[m].child_a, c.ops[m].child_b})
          if (op_of_node[ch] >= 0 && c.ops[op_of_node[ch]].nb > 0) deps.push_back(op_of_node[ch]);
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      op.deps = std::move(deps);
      for (const auto& r : reads) seen.push_back({r.first, r.second, static_cast<int>(i), false});
      for (const auto& w : writes) seen.push_back({w.first, w.second, static_cast<int>(i), true});
    }
  }

  if (p.node_slot[p.root] >= 0) {
    // single-slot network: the root leaf itself is every request's value
    c.has_leaf_root = true;
    LeafRoot& lr = c.leaf_root;
    lr.slot = p.node_slot[p.root];
    lr.item = c.slot_item[lr.slot];
    lr.row_value.resize(ti.rows);
    for (uint64_t row = 0; row < ti.rows; ++row)
      lr.row_value[row] =
          p.tuples[static_cast<uint64_t>(ti.row_tuple_first[row]) * p.n_slots + lr.slot];
    std::vector<uint32_t> o_legs(c.out_legs.rbegin(), c.out_legs.rend());
    std::vector<uint64_t> st;
    for (uint32_t x : o_legs) st.push_back(stride_in(slot_layout[lr.slot], x));
    lr.tout.build(st);
    if (S > 0) {
      lr.slice_stride.assign(S, 0);
      for (int x = 0; x < S; ++x)
        if (contains(slot_layout[lr.slot], c.sliced[x]))
          lr.slice_stride[S - 1 - x] = stride_in(slot_layout[lr.slot], c.sliced[x]);
    }
  }

  timer.mark("ops");
  // --- blobs -----------------------------------------------------------------
  {  // sizes first: one allocation each (growing them cost ~30 ms at 10^6 requests)
    uint64_t tw = 0, iw = 0;
    auto tsz = [&](const SplitTable& t) { tw += t.lo.size() + t.hi.size(); };
    for (const Op& op : c.ops) {
      for (const SplitTable* t : {&op.tam, &op.tak, &op.tbn, &op.tbk, &op.tom, &op.ton}) tsz(*t);
      iw += op.ia.size() + op.ib.size() + op.grp_items.size() + op.grp_start.size() + op.out_rows.size() +
            op.ga_groups.size() + op.ga_tiles.size();
    }
    for (const Chain& ch : c.chains) {
      tsz(ch.tu_in);
      tsz(ch.tu_out);
      iw += ch.qin.size() + ch.qout.size() + ch.entries.size();
      for (const ChainStep& st : ch.steps) iw += st.tbl.size();
    }
    if (c.has_leaf_root) {
      tsz(c.leaf_root.tout);
      iw += c.leaf_root.row_value.size();
    }
    c.table_blob.reserve(c.table_blob.size() + tw);
    c.index_blob.reserve(c.index_blob.size() + iw);
  }
  auto put_table = [&](SplitTable& t) {
    t.dev_off = c.table_blob.size();
    c.table_blob.insert(c.table_blob.end(), t.lo.begin(), t.lo.end());
    c.table_blob.insert(c.table_blob.end(), t.hi.begin(), t.hi.end());
  };
  auto put_index = [&](const std::vector<uint32_t>& v) {
    const uint64_t off = c.index_blob.size();
    c.index_blob.insert(c.index_blob.end(), v.begin(), v.end());
    return off;
  };
  for (Op& op : c.ops) {
    for (SplitTable* t : {&op.tam, &op.tak, &op.tbn, &op.tbk, &op.tom, &op.ton})
      put_table(*t);
    op.ia_off = put_index(op.ia);
    op.ib_off = put_index(op.ib);
    op.grp_items_off = put_index(op.grp_items);
    op.grp_start_off = put_index(op.grp_start);
    op.out_rows_off = put_index(op.out_rows);
    op.ga_groups_off = put_index(op.ga_groups);
    op.ga_tiles_off = put_index(op.ga_tiles);
  }
  for (Chain& ch : c.chains) {
    put_table(ch.tu_in);
    put_table(ch.tu_out);
    ch.qin_off = put_index(ch.qin);
    ch.qout_off = put_index(ch.qout);
    ch.entries_off = put_index(ch.entries);
    for (ChainStep& st : ch.steps) st.tbl_off = put_index(st.tbl);
  }
  if (c.has_leaf_root) {
    put_table(c.leaf_root.tout);
    c.leaf_root.rows_off = put_index(c.leaf_root.row_value);
  }
  timer.mark("blobs");
  if (std::getenv("MTCG_DUMP_OPS")) {
    for (const Op& op : c.ops) {
      std::vector<uint32_t> a(op.ia), b(op.ib);
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      const auto da = std::unique(a.begin(), a.end()) - a.begin();
      const auto db = std::unique(b.begin(), b.end()) - b.begin();
      std::fprintf(stderr,
                   "[mtcg] op node %d M2^%d N2^%d K2^%d batch %u distinct_a %ld distinct_b %ld cfg %d"
                   " slots %u kcontig %d ncontig %d mcontig %d%s\n",
                   op.node, op.fa, op.fb, op.kc, op.nb, (long)da, (long)db, op.config, op.grp_max,
                   op.a_kcontig, op.o_ncontig, op.o_mcontig, op.root ? " root" : "");
      std::fprintf(stderr, "[mtcg]   deps");
      for (int d : op.deps) std::fprintf(stderr, " %d", c.ops[d].node);
      std::fprintf(stderr, "\n");
      // per-bit strides (elements) of the op's index spaces
      auto bit_strides = [](const char* name, const SplitTable& t) {
        std::fprintf(stderr, "[mtcg]   %s:", name);
        for (int b = 0; b < t.bits; ++b) {
          const uint64_t v = b < t.lo_bits ? t.lo[uint64_t{1} << b] : t.hi[uint64_t{1} << (b - t.lo_bits)];
          std::fprintf(stderr, " %llu", static_cast<unsigned long long>(v));
        }
        std::fprintf(stderr, "\n");
      };
      bit_strides("A m", op.tam);
      bit_strides("A k", op.tak);
      bit_strides("B n", op.tbn);
      bit_strides("B k", op.tbk);
      bit_strides("out m", op.tom);
      bit_strides("out n", op.ton);
    }
  }
  return c;
}

}  // namespace mtcg
