// Simulated annealing over contraction trees (plan producer for the
// 53-qubit workloads; see plans/sycamore_plan.py). The paper's local search
// (PAPER.md:846-953): rotations (a*b)*c -> (a*c)*b / (c*b)*a of any subtree,
// objective
//     f = log2(C + α RW) + beta_mem * max(0, log2(table_max / M_max))
// with the multi-amplitude cost C = S * Σ_nodes k_T
// 2^|legs L ∪ legs R|, RW = S * Σ_nodes k_T (|L| + |R| + |T|) and
// memo table k_T 2^|legs T| (k_T: distinct output-bit tuples of the
// subtree over the k requests, estimated as 2^q (1 - e^(-k/2^q)) for q
// output qubits; S = 2^sliced). With memo streaming (requests in chunks of
// B, mtcg_options.row_chunk) a request-dependent node is evaluated per chunk
// for that chunk's distinct tuples and its table holds one chunk's. A rotation changes one node's legs, so a move
// is evaluated in O(1): the two affected nodes' costs are swapped in and the
// total is recomputed exactly from scratch every few thousand moves (the
// reference's incremental long-double p-norm drifts). Every
// `slice_every` moves a slicing move adds (or swaps) a sliced leg chosen
// among the legs of the largest tables.
//
// stdin: n_leaves n_legs k chunk alpha (memo streaming chunk, 0: none;
//        alpha: complex MACs per element of traffic, the paper's C + αRW)
//        per leaf: q count leg...
//        n_merges, then n_merges lines "a b" (ids: leaves 0..n-1, merge i -> n+i)
//        steps beta0 beta1 log2_max_table beta_mem slice_every max_slices seed
//        n_fixed_sliced leg...
// stdout: n_merges lines "a b", then "slice: leg..."
//   g++ -O3 -march=native -o treesa plans/treesa.cpp
#include <algorithm>
#include <bitset>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <random>
#include <vector>

constexpr int kMaxLegs = 1024;
using Legs = std::bitset<kMaxLegs>;

struct Node {
  int left = -1, right = -1, parent = -1;
  Legs legs;
  int q = 0;
};

struct Tree {
  std::vector<Node> nodes;  // leaves first
  int n_leaves = 0, root = -1;
  double k = 1;
  double chunk = 0;  // memo streaming: requests per chunk (0: all at once)
  Legs sliced;

  static double distinct(int q, double n) {
    if (n <= 1 || q == 0) return 1.0;
    if (q >= 62) return n;
    const double m = std::ldexp(1.0, q);
    return n < 40 * m ? m * -std::expm1(-n / m) : m;
  }
  double chunk_size() const { return chunk > 0 && chunk < k ? chunk : k; }
  // evaluations of a node with q output qubits: once when request-
  // independent, else per chunk the chunk's distinct tuples
  double evals(int q) const {
    if (q == 0) return 1.0;
    const double b = chunk_size();
    return std::ceil(k / b) * distinct(q, b);
  }
  // cost of internal node v (per slice), and its memo table (one chunk)
  double alpha = 0;  // complex MACs one element of memory traffic is worth (the paper's C + αRW)
  double node_cost(int v) const {
    const Node& n = nodes[v];
    const Legs l = nodes[n.left].legs & ~sliced, r = nodes[n.right].legs & ~sliced;
    const double macs = std::ldexp(1.0, static_cast<int>((l | r).count()));
    const double rw = alpha > 0 ? std::ldexp(1.0, static_cast<int>(l.count())) +
                                      std::ldexp(1.0, static_cast<int>(r.count())) +
                                      std::ldexp(1.0, static_cast<int>((l ^ r).count()))
                                : 0.0;
    // cc > 1: MACs of contractions the tensor-core path cannot take (fewer
    // than 128 free rows on the larger side, fewer than 16 on the other, or
    // K < 16) cost cc times more (the CUDA-core kernels' rate)
    double factor = 1.0;
    if (cc > 1.0) {
      const int kk = static_cast<int>((l & r).count());
      const int fl = static_cast<int>(l.count()) - kk, fr = static_cast<int>(r.count()) - kk;
      const int mm = std::max(fl, fr), nn = std::min(fl, fr);
      if (mm < 7 || nn < 4 || kk < 4) factor = cc;
    }
    return evals(n.q) * (macs * factor + alpha * rw);
  }
  double cc = 1.0;  // CUDA-core MAC cost multiplier (see node_cost)
  double node_table(int v) const {
    return distinct(nodes[v].q, chunk_size()) * std::ldexp(1.0, static_cast<int>((nodes[v].legs & ~sliced).count()));
  }
  void refresh(int v) {
    Node& n = nodes[v];
    n.legs = nodes[n.left].legs ^ nodes[n.right].legs;
    n.q = nodes[n.left].q + nodes[n.right].q;
  }
  void refresh_all(int v) {
    if (v < n_leaves) return;
    refresh_all(nodes[v].left);
    refresh_all(nodes[v].right);
    refresh(v);
  }
  double total() const {
    double t = 0;
    for (size_t v = n_leaves; v < nodes.size(); ++v) t += node_cost(static_cast<int>(v));
    return t;
  }
  double table_max() const {
    double t = 0;
    for (size_t v = n_leaves; v < nodes.size(); ++v) t = std::max(t, node_table(static_cast<int>(v)));
    return t;
  }
};

int main() {
  std::ios::sync_with_stdio(false);
  Tree T;
  int n_legs;
  double k;
  double chunk, alpha;
  std::cin >> T.n_leaves >> n_legs >> k >> chunk >> alpha;
  T.k = k;
  T.chunk = chunk;
  T.alpha = alpha;
  if (const char* e = std::getenv("TREESA_CC")) T.cc = std::atof(e);  // CUDA-core MAC multiplier
  T.nodes.resize(T.n_leaves);
  for (int i = 0; i < T.n_leaves; ++i) {
    int q, c;
    std::cin >> q >> c;
    T.nodes[i].q = q;
    for (int j = 0; j < c; ++j) {
      int l;
      std::cin >> l;
      T.nodes[i].legs.set(l);
    }
  }
  int nm;
  std::cin >> nm;
  for (int i = 0; i < nm; ++i) {
    int a, b;
    std::cin >> a >> b;
    Node n;
    n.left = a;
    n.right = b;
    T.nodes.push_back(n);
    const int v = static_cast<int>(T.nodes.size()) - 1;
    T.nodes[a].parent = v;
    T.nodes[b].parent = v;
  }
  T.root = static_cast<int>(T.nodes.size()) - 1;
  long long steps;
  double beta0, beta1, log2_max_table, beta_mem;
  long long slice_every;
  int max_slices;
  unsigned seed;
  std::cin >> steps >> beta0 >> beta1 >> log2_max_table >> beta_mem >> slice_every >> max_slices >> seed;
  int nf;
  std::cin >> nf;
  for (int i = 0; i < nf; ++i) {
    int l;
    std::cin >> l;
    T.sliced.set(l);
  }
  T.refresh_all(T.root);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const double max_table = std::ldexp(1.0, static_cast<int>(log2_max_table)) *
                           std::exp2(log2_max_table - std::floor(log2_max_table));
  auto objective = [&](double cost, double tmax) {
    return std::log2(cost * std::ldexp(1.0, static_cast<int>(T.sliced.count()))) +
           beta_mem * std::max(0.0, std::log2(tmax / max_table));
  };
  double cost = T.total();
  double tmax = T.table_max();
  double cur = objective(cost, tmax);
  std::vector<Node> best_nodes = T.nodes;
  Legs best_sliced = T.sliced;
  double best = cur;
  std::vector<int> internal;
  for (size_t v = T.n_leaves; v < T.nodes.size(); ++v) internal.push_back(static_cast<int>(v));

  for (long long step = 0; step < steps; ++step) {
    const double beta = beta0 * std::pow(beta1 / beta0, static_cast<double>(step) / std::max(1LL, steps - 1));
    if (slice_every > 0 && step % slice_every == slice_every - 1 &&
        (static_cast<int>(T.sliced.count()) < max_slices || tmax > max_table)) {
      // slicing move: candidate legs of the largest tables; add the one that
      // minimises the objective (or, at the slice budget, swap the least
      // useful sliced leg out)
      std::vector<std::pair<double, int>> tabs;
      for (int v : internal) tabs.push_back({T.node_table(v), v});
      std::sort(tabs.rbegin(), tabs.rend());
      Legs cand;
      for (size_t i = 0; i < std::min<size_t>(tabs.size(), 8); ++i) cand |= T.nodes[tabs[i].second].legs;
      cand &= ~T.sliced;
      int best_leg = -1;
      double best_val = 1e300;
      for (int l = 0; l < kMaxLegs; ++l) {
        if (!cand[l]) continue;
        T.sliced.set(l);
        const double v = objective(T.total(), T.table_max());
        T.sliced.reset(l);
        if (v < best_val) best_val = v, best_leg = l;
      }
      if (best_leg >= 0) {
        if (static_cast<int>(T.sliced.count()) >= max_slices) {
          // drop the sliced leg whose removal hurts least, then add
          int drop = -1;
          double dv = 1e300;
          for (int l = 0; l < kMaxLegs; ++l) {
            if (!T.sliced[l]) continue;
            T.sliced.reset(l);
            T.sliced.set(best_leg);
            const double v = objective(T.total(), T.table_max());
            T.sliced.reset(best_leg);
            T.sliced.set(l);
            if (v < dv) dv = v, drop = l;
          }
          if (drop >= 0 && dv < cur) {
            T.sliced.reset(drop);
            T.sliced.set(best_leg);
          }
        } else if (best_val < cur || tmax > max_table) {
          T.sliced.set(best_leg);
        }
        cost = T.total();
        tmax = T.table_max();
        cur = objective(cost, tmax);
      }
      continue;
    }
    // rotation at a random internal node v with an internal child u
    const int v = internal[rng() % internal.size()];
    Node& nv = T.nodes[v];
    const bool use_left = (rng() & 1) != 0;
    int u = use_left ? nv.left : nv.right;
    int c = use_left ? nv.right : nv.left;
    if (u < T.n_leaves) {
      std::swap(u, c);
      if (u < T.n_leaves) continue;
    }
    Node& nu = T.nodes[u];
    const bool keep_left = (rng() & 1) != 0;  // (a*b)*c -> (a*c)*b  or  (b*c)*a
    const int stay = keep_left ? nu.left : nu.right;
    const int move = keep_left ? nu.right : nu.left;
    const double old_u = T.node_cost(u), old_v = T.node_cost(v);
    // apply
    const Node su = nu, sv = nv;
    nu.left = stay;
    nu.right = c;
    T.nodes[c].parent = u;
    nv.left = u;
    nv.right = move;
    T.nodes[move].parent = v;
    T.refresh(u);
    const double new_u = T.node_cost(u), new_v = T.node_cost(v);
    const double new_cost = cost - old_u - old_v + new_u + new_v;
    const double new_tab_u = T.node_table(u);
    const double new_tmax = std::max(tmax, new_tab_u);  // (max may also drop; refreshed periodically)
    const double val = objective(new_cost, new_tmax);
    if (val <= cur || U(rng) < std::exp(-beta * (val - cur))) {
      cost = new_cost;
      tmax = new_tmax;
      cur = val;
      if ((step & 4095) == 0) {  // exact refresh: no drift
        cost = T.total();
        tmax = T.table_max();
        cur = objective(cost, tmax);
      }
      if (cur < best) {
        cost = T.total();
        tmax = T.table_max();
        cur = objective(cost, tmax);
        if (cur < best) {
          best = cur;
          best_nodes = T.nodes;
          best_sliced = T.sliced;
        }
      }
    } else {
      // revert
      T.nodes[move].parent = u;
      T.nodes[c].parent = v;
      nu = su;
      nv = sv;
    }
  }
  T.nodes = best_nodes;
  T.sliced = best_sliced;
  std::fprintf(stderr, "treesa: best objective %.3f, cost %.4e MACs x %zu slices, max table %.4e\n", best,
               T.total(), static_cast<size_t>(1) << T.sliced.count(), T.table_max());
  // emit merges in post-order
  std::vector<int> id(T.nodes.size(), -1);
  for (int i = 0; i < T.n_leaves; ++i) id[i] = i;
  int next = T.n_leaves;
  std::vector<std::pair<int, int>> out;
  std::vector<std::pair<int, bool>> st{{T.root, false}};
  while (!st.empty()) {
    auto [v, done] = st.back();
    st.pop_back();
    if (v < T.n_leaves) continue;
    if (!done) {
      st.push_back({v, true});
      st.push_back({T.nodes[v].right, false});
      st.push_back({T.nodes[v].left, false});
    } else {
      out.push_back({id[T.nodes[v].left], id[T.nodes[v].right]});
      id[v] = next++;
    }
  }
  for (auto [a, b] : out) std::printf("%d %d\n", a, b);
  std::printf("slice:");
  for (int l = 0; l < kMaxLegs; ++l)
    if (T.sliced[l]) std::printf(" %d", l);
  std::printf("\n");
  return 0;
}
