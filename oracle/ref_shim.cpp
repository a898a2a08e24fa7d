// ORACLE TEST INFRASTRUCTURE — not product code.
//
// C-ABI glue over the UNMODIFIED reference library (`mtc`, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It only
// forwards to the reference's public API so Python tests, golden-vector
// generators and the bench's CPU baseline can drive the reference itself:
//
//   inputs   parse_circuit / to_diagram / build_assignments / parse_plan
//            (proj/src/circuit.cpp:113, diagram.cpp:164, diagram.cpp:229,
//             plan.cpp:176)
//   engine   eval_all / eval_sliced / eval_naive / emulate
//            (proj/include/mtc/multieval.hpp:53-75)
//   costs    CostedPlan exact mode totals (proj/include/mtc/plan.hpp:136-214)
//   plans    anneal (proj/include/mtc/optimizer.hpp:52-53)
//   XEB      linear_xeb (proj/include/mtc/xeb.hpp:38)
//   tests    grid_circuit / random_circuit / random_bitstrings / StateVector
//            (proj/tests/support/gen.hpp, oracle.hpp)
//
// Nothing here is on the product path and nothing here is shipped.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mtc/circuit.hpp"
#include "mtc/diagram.hpp"
#include "mtc/errors.hpp"
#include "mtc/formats.hpp"
#include "mtc/multieval.hpp"
#include "mtc/optimizer.hpp"
#include "mtc/plan.hpp"
#include "mtc/rng.hpp"
#include "mtc/tensor.hpp"
#include "mtc/xeb.hpp"
#include "support/gen.hpp"
#include "support/oracle.hpp"

using namespace mtc;

namespace {

thread_local std::string g_err;

struct Problem {
  Circuit circuit;
  NetworkDiagram d;
  std::vector<std::string> bits;
  std::vector<LegId> batch;
  AssignmentSet as;
  Plan plan;
  bool has_plan = false;
};

std::vector<std::string> split_lines(const char* text) {
  std::vector<std::string> out;
  if (!text) return out;
  std::istringstream ss(text);
  std::string line;
  while (std::getline(ss, line)) {
    while (!line.empty() && (line.back() == '\r' || line.back() == ' '))
      line.pop_back();
    if (!line.empty()) out.push_back(line);
  }
  return out;
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

int classify(const std::exception_ptr& e, int* cap_node) {
  try {
    std::rethrow_exception(e);
  } catch (const MemoryCapError& x) {
    g_err = x.what();
    if (cap_node) *cap_node = x.node();
    return 3;
  } catch (const ParseError& x) {
    g_err = x.what();
    return 4;
  } catch (const DataError& x) {
    g_err = x.what();
    return 2;
  } catch (const std::exception& x) {
    g_err = x.what();
    return 1;
  }
  return 1;
}

void copy_values(const std::vector<Tensor>& values, double* out) {
  std::size_t o = 0;
  for (const Tensor& t : values)
    for (const Complex& c : t.data()) {
      out[o++] = c.real();
      out[o++] = c.imag();
    }
}

// Per-slice leaves, exactly as run_slice does (proj/src/multieval.cpp:352-367,
// :465-476): every value-set tensor is projected on each sliced leg it carries,
// in plan.sliced order, at the mixed-radix values of `idx` (last leg fastest,
// :322-329).
AssignmentSet slice_assignments(const Problem& p, std::uint64_t idx) {
  AssignmentSet as = p.as;
  const auto& legs = p.plan.sliced;
  std::vector<std::uint32_t> vals(legs.size());
  for (std::size_t j = legs.size(); j-- > 0;) {
    std::uint32_t dim = p.d.leg_dims[legs[j]];
    vals[j] = static_cast<std::uint32_t>(idx % dim);
    idx /= dim;
  }
  for (auto& vs : as.value_sets)
    for (Tensor& t : vs)
      for (std::size_t x = 0; x < legs.size(); ++x)
        if (t.has_leg(legs[x])) t = project_leg(t, legs[x], vals[x]);
  return as;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// ---- problem construction -------------------------------------------------

void* ref_problem_new(const char* circuit_text, int fuse,
                      const char* bitstrings_nl, const char* plan_text) {
  try {
    auto* p = new Problem;
    p->circuit = parse_circuit(std::string(circuit_text));
    p->d = to_diagram(p->circuit, fuse != 0);
    p->bits = split_lines(bitstrings_nl);
    if (!p->bits.empty())
      for (std::size_t q = 0; q < p->bits.front().size(); ++q)
        if (p->bits.front()[q] == '*')
          p->batch.push_back(p->d.open_legs.at(q));
    p->as = build_assignments(p->d, p->bits, p->batch);
    if (plan_text && *plan_text) {
      p->plan = parse_plan(std::string(plan_text));
      p->has_plan = true;
    }
    return p;
  } catch (...) {
    classify(std::current_exception(), nullptr);
    return nullptr;
  }
}

void ref_problem_free(void* h) { delete static_cast<Problem*>(h); }

int ref_set_plan(void* h, const char* plan_text) {
  auto* p = static_cast<Problem*>(h);
  try {
    p->plan = parse_plan(std::string(plan_text));
    p->has_plan = true;
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

char* ref_plan_text(void* h) {
  return dup_string(format_plan(static_cast<Problem*>(h)->plan));
}

int ref_n_qubits(void* h) { return static_cast<Problem*>(h)->d.n_qubits; }
std::uint32_t ref_n_closed(void* h) {
  return static_cast<Problem*>(h)->d.n_closed;
}
std::uint32_t ref_n_legs(void* h) {
  return static_cast<std::uint32_t>(static_cast<Problem*>(h)->d.leg_count());
}
int ref_n_slots(void* h) {
  return static_cast<int>(static_cast<Problem*>(h)->d.slot_count());
}

// Unprojected slot tensor of the diagram.
int ref_slot_tensor(void* h, int j, std::uint32_t* legs, double* data) {
  const Tensor& t = static_cast<Problem*>(h)->d.slot_tensors.at(j);
  if (legs)
    for (std::size_t i = 0; i < t.order(); ++i) legs[i] = t.legs()[i].id;
  if (data) copy_values({t}, data);
  return static_cast<int>(t.order());
}

int ref_slot_n_values(void* h, int j) {
  return static_cast<int>(static_cast<Problem*>(h)->as.value_sets.at(j).size());
}

// Legs of slot j's value tensors (all share one leg list) and their data.
int ref_slot_values(void* h, int j, std::uint32_t* legs, double* data) {
  const auto& vs = static_cast<Problem*>(h)->as.value_sets.at(j);
  const Tensor& t0 = vs.front();
  if (legs)
    for (std::size_t i = 0; i < t0.order(); ++i) legs[i] = t0.legs()[i].id;
  if (data) copy_values(vs, data);
  return static_cast<int>(t0.order());
}

std::uint64_t ref_n_requests(void* h) {
  return static_cast<Problem*>(h)->as.request_count();
}

void ref_tuples(void* h, std::uint32_t* out) {
  const auto& as = static_cast<Problem*>(h)->as;
  std::size_t o = 0;
  for (const auto& t : as.tuples)
    for (std::uint32_t v : t) out[o++] = v;
}

int ref_batch_legs(void* h, std::uint32_t* out) {
  const auto& b = static_cast<Problem*>(h)->as.batch_legs;
  if (out) std::copy(b.begin(), b.end(), out);
  return static_cast<int>(b.size());
}

int ref_plan_nodes(void* h, int* left, int* right, int* slot) {
  const Plan& pl = static_cast<Problem*>(h)->plan;
  for (std::size_t i = 0; i < pl.nodes.size(); ++i) {
    if (left) left[i] = pl.nodes[i].left;
    if (right) right[i] = pl.nodes[i].right;
    if (slot) slot[i] = pl.nodes[i].slot;
  }
  return static_cast<int>(pl.nodes.size());
}

int ref_plan_root(void* h) { return static_cast<Problem*>(h)->plan.root; }

int ref_plan_sliced(void* h, std::uint32_t* out) {
  const auto& s = static_cast<Problem*>(h)->plan.sliced;
  if (out) std::copy(s.begin(), s.end(), out);
  return static_cast<int>(s.size());
}

// ---- engine -----------------------------------------------------------------

// mode: 0 eval_all, 1 eval_sliced, 2 eval_naive, 3 auto (the CLI's choice,
// proj/tools/main.cpp:159-160). out_values: request-major complex pairs.
int ref_eval(void* h, int mode, int workers, std::uint64_t cap,
             double* out_values, std::uint64_t* node_contractions,
             std::uint64_t* counters, std::uint64_t* peak, int* cap_node) {
  auto* p = static_cast<Problem*>(h);
  try {
    EvalOptions opts;
    opts.memory_cap_bytes = cap;
    opts.workers = workers;
    EvalResult r;
    if (mode == 3) mode = p->plan.sliced.empty() ? 0 : 1;
    if (mode == 0)
      r = eval_all(p->plan, p->d, p->as, opts);
    else if (mode == 1)
      r = eval_sliced(p->plan, p->d, p->as, opts);
    else
      r = eval_naive(p->plan, p->d, p->as, opts);
    if (out_values) copy_values(r.values, out_values);
    if (node_contractions)
      std::copy(r.node_contractions.begin(), r.node_contractions.end(),
                node_contractions);
    if (counters) {
      counters[0] = r.counters.mults;
      counters[1] = r.counters.adds;
      counters[2] = r.counters.rw;
    }
    if (peak) *peak = r.peak_bytes;
    return 0;
  } catch (...) {
    return classify(std::current_exception(), cap_node);
  }
}

// One slice through the public API: the projected assignment set evaluated by
// eval_all on the plan without its slice list. Bit-identical to the slice's
// per-row values inside eval_sliced.
int ref_eval_slice(void* h, std::uint64_t idx, double* out_values) {
  auto* p = static_cast<Problem*>(h);
  try {
    AssignmentSet as = slice_assignments(*p, idx);
    Plan pl = p->plan;
    pl.sliced.clear();
    EvalResult r = eval_all(pl, p->d, as);
    if (out_values) copy_values(r.values, out_values);
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// `n` slices [first, first+n) on `threads` std::threads, each a full
// single-threaded eval_all (the reference's per-slice executor). Used as the
// bench's CPU baseline sample. Returns 0 or an error class.
int ref_eval_slices_parallel(void* h, std::uint64_t first, std::uint64_t n,
                             int threads) {
  auto* p = static_cast<Problem*>(h);
  std::vector<std::thread> pool;
  std::vector<int> status(threads, 0);
  for (int w = 0; w < threads; ++w)
    pool.emplace_back([&, w]() {
      for (std::uint64_t i = w; i < n; i += threads)
        if (ref_eval_slice(p, first + i, nullptr) != 0) status[w] = 1;
    });
  for (auto& t : pool) t.join();
  for (int s : status)
    if (s) return 1;
  return 0;
}

int ref_emulate(void* h, std::uint64_t cap, std::uint64_t* counters,
                std::uint64_t* peak, std::uint64_t* node_contractions) {
  auto* p = static_cast<Problem*>(h);
  try {
    EvalOptions opts;
    opts.memory_cap_bytes = cap;
    EmulateResult em = emulate(p->plan, p->d, p->as, opts);
    counters[0] = em.counters.mults;
    counters[1] = em.counters.adds;
    counters[2] = em.counters.rw;
    *peak = em.peak_bytes;
    if (node_contractions)
      std::copy(em.node_contractions.begin(), em.node_contractions.end(),
                node_contractions);
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// CostedPlan in exact mode: totals as (hi, lo) u64 pairs, plus per-node k_t.
int ref_exact_totals(void* h, std::uint64_t* mults, std::uint64_t* adds,
                     std::uint64_t* rw, std::uint64_t* node_kt,
                     std::uint64_t* node_size) {
  auto* p = static_cast<Problem*>(h);
  try {
    CostConfig cfg;
    cfg.k = std::max<std::uint64_t>(p->as.request_count(), 1);
    CostedPlan exact(p->plan, p->d, cfg, exact_value_counts(p->as), &p->as);
    auto split = [](u128 v, std::uint64_t* o) {
      o[0] = static_cast<std::uint64_t>(v >> 64);
      o[1] = static_cast<std::uint64_t>(v);
    };
    split(exact.total_mults(), mults);
    split(exact.total_adds(), adds);
    split(exact.total_rw(), rw);
    for (std::size_t n = 0; n < exact.node_count(); ++n) {
      if (node_kt) node_kt[n] = exact.node(static_cast<int>(n)).k_t;
      if (node_size) node_size[n] = exact.node(static_cast<int>(n)).size;
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// ---- generators ---------------------------------------------------------------

char* ref_grid_circuit(int rows, int cols, int layers, std::uint64_t seed) {
  return dup_string(format_circuit(test::grid_circuit(rows, cols, layers, seed)));
}

char* ref_random_circuit(std::uint64_t seed, int n_qubits, int n_gates) {
  Rng rng(seed);
  return dup_string(format_circuit(test::random_circuit(rng, n_qubits, n_gates)));
}

char* ref_random_bitstrings(std::uint64_t seed, int n_qubits, int count) {
  Rng rng(seed);
  std::string out;
  for (const std::string& s : test::random_bitstrings(rng, n_qubits, count))
    out += s + "\n";
  return dup_string(out);
}

char* ref_left_deep_plan(int n_slots) {
  return dup_string(format_plan(left_deep_plan(n_slots)));
}

// Simulated annealing with bound-mode value counts (the `mtc optimize` path,
// proj/tools/main.cpp:123-143). Returns the plan text or nullptr.
char* ref_anneal(void* h, std::uint64_t k, std::uint64_t m_max, double alpha,
                 double beta, double p_norm, std::uint64_t steps,
                 std::uint64_t slice_interval, std::uint64_t seed,
                 std::uint32_t chains, double* objective_out) {
  auto* p = static_cast<Problem*>(h);
  try {
    CostConfig cfg;
    cfg.k = k;
    cfg.m_max = m_max;
    cfg.alpha = alpha;
    cfg.beta = beta;
    cfg.p = p_norm;
    ValueCounts counts = bound_value_counts(p->d, p->batch, k);
    SearchConfig sc;
    sc.steps = steps;
    sc.slice_interval = slice_interval;
    sc.seed = seed;
    sc.chains = chains;
    AnnealResult a = anneal(p->d, counts, cfg, sc);
    if (objective_out) *objective_out = a.objective;
    return dup_string(format_plan(a.plan));
  } catch (...) {
    classify(std::current_exception(), nullptr);
    return nullptr;
  }
}

// Adds `n` sliced legs to the current plan, one at a time, each the sliceable
// leg that minimises the bound-mode objective after slicing (criterion 0: the
// memory estimate, as slicing_move does, proj/src/optimizer.cpp:53-77;
// criterion 1: total cost C(T,k)). Uses only CostedPlan's public API.
int ref_add_slices_greedy(void* h, int n, std::uint64_t k, std::uint64_t m_max,
                          int criterion) {
  auto* p = static_cast<Problem*>(h);
  try {
    CostConfig cfg;
    cfg.k = k;
    cfg.m_max = m_max;
    ValueCounts counts = bound_value_counts(p->d, p->batch, k);
    CostedPlan cp(p->plan, p->d, cfg, counts);
    for (int s = 0; s < n; ++s) {
      bool found = false;
      LegId best_leg = 0;
      long double best = 0;
      for (LegId l = 0; l < cp.leg_count(); ++l) {
        if (!cp.leg_sliceable(l)) continue;
        CostedPlan probe = cp;
        probe.add_slice(l);
        long double v = criterion == 0
                            ? static_cast<long double>(probe.memory_estimate_bytes())
                            : static_cast<long double>(probe.total_cost());
        if (!found || v < best) {
          best = v;
          best_leg = l;
          found = true;
        }
      }
      if (!found) break;
      cp.add_slice(best_leg);
    }
    p->plan = cp.plan();
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// Bounded-sample timing of the reference engine's hot loop on this problem.
//
// For every internal plan node the reference's own contract_pair
// (tensor.cpp:150-253, ~94% of eval time) is run on random operands with
// the node's real leg lists (slice-projected leaves, contraction_result_legs
// intermediates, every shared leg closed as multieval.cpp:97 does). Nodes
// costing more than `budget` complex MACs are sampled on a sub-block: free
// legs of the larger operand are projected away (project_leg) until the
// contraction fits — contract_pair's cost per output element is d_closed
// multiply-adds whatever d_open is, so time scales linearly by the
// projected-away factor. Returns the single-thread-equivalent time of the
// whole evaluation, Σ_n distinct[n] · S · t_n, plus the sampling wall time.
// Nodes are sampled concurrently on `threads` std::threads (the per-core
// rate under a loaded socket, as eval_sliced's workers see it).
int ref_sample_eval_time(void* h, std::uint64_t budget, int threads,
                         double* est_seconds_1thread, double* sample_wall,
                         double* sampled_fraction) {
  auto* p = static_cast<Problem*>(h);
  try {
    TupleIndex ti = build_tuple_index(p->plan, p->as);
    PlanIndex ix = index_plan(p->plan, p->d.slot_count());
    std::uint64_t slices = 1;
    for (LegId l : p->plan.sliced) slices *= p->d.leg_dims[l];
    const std::size_t n = p->plan.nodes.size();
    std::vector<std::vector<Leg>> legs(n);
    std::vector<int> work;
    for (int node : ix.postorder) {
      const Plan::Node& nd = p->plan.nodes[node];
      if (nd.leaf()) {
        for (const Leg& l : p->as.value_sets[nd.slot].front().legs())
          if (std::find(p->plan.sliced.begin(), p->plan.sliced.end(), l.id) ==
              p->plan.sliced.end())
            legs[node].push_back(l);
        continue;
      }
      std::vector<LegId> closed;
      for (const Leg& a : legs[nd.left])
        for (const Leg& b : legs[nd.right])
          if (a.id == b.id) closed.push_back(a.id);
      legs[node] = contraction_result_legs(legs[nd.left], legs[nd.right], closed);
      if (ti.distinct[node] > 0) work.push_back(node);
    }
    std::vector<double> node_time(n, 0.0);
    std::vector<double> node_frac(n, 1.0);
    std::atomic<std::size_t> next{0};
    auto worker = [&](int w) {
      Rng rng(0x5eed + w);
      for (std::size_t i = next++; i < work.size(); i = next++) {
        const int node = work[i];
        const Plan::Node& nd = p->plan.nodes[node];
        std::vector<Leg> la = legs[nd.left], lb = legs[nd.right];
        std::vector<LegId> closed;
        for (const Leg& a : la)
          for (const Leg& b : lb)
            if (a.id == b.id) closed.push_back(a.id);
        auto is_closed = [&](LegId id) {
          return std::find(closed.begin(), closed.end(), id) != closed.end();
        };
        auto size_of = [](const std::vector<Leg>& v) {
          std::uint64_t s = 1;
          for (const Leg& l : v) s *= l.dim;
          return s;
        };
        PairCost full = predicted_cost(la, lb, closed);
        PairCost pc = full;
        double scale = 1.0;
        while (pc.mults > budget) {
          std::vector<Leg>& big = size_of(la) >= size_of(lb) ? la : lb;
          auto it = std::find_if(big.begin(), big.end(),
                                 [&](const Leg& l) { return !is_closed(l.id); });
          if (it == big.end()) break;
          scale *= it->dim;
          big.erase(it);
          pc = predicted_cost(la, lb, closed);
        }
        auto random_tensor = [&](const std::vector<Leg>& v) {
          std::vector<Complex> data(size_of(v));
          for (Complex& c : data) c = {rng.uniform_real01() - 0.5, rng.uniform_real01() - 0.5};
          return Tensor(v, std::move(data));
        };
        Tensor a = random_tensor(la), b = random_tensor(lb);
        double best = 1e300;
        for (int rep = 0; rep < 2; ++rep) {
          auto t0 = std::chrono::steady_clock::now();
          Tensor r = contract_pair(a, b, closed);
          double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          best = std::min(best, dt);
          if (dt > 0.05) break;  // large samples: one timing is enough
        }
        node_time[node] = best * scale;
        node_frac[node] = 1.0 / scale;
      }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < std::max(1, threads); ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
    *sample_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double total = 0.0, full_mults = 0.0, sampled_mults = 0.0;
    for (int node : work) {
      total += static_cast<double>(ti.distinct[node]) * slices * node_time[node];
      const Plan::Node& nd = p->plan.nodes[node];
      std::vector<LegId> closed;
      for (const Leg& a : legs[nd.left])
        for (const Leg& b : legs[nd.right])
          if (a.id == b.id) closed.push_back(a.id);
      const double m = static_cast<double>(predicted_cost(legs[nd.left], legs[nd.right], closed).mults);
      full_mults += m;
      sampled_mults += m * node_frac[node];
    }
    *est_seconds_1thread = total;
    if (sampled_fraction) *sampled_fraction = full_mults > 0 ? sampled_mults / full_mults : 1.0;
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// Brute-force state vector (proj/tests/support/oracle.cpp:98-148).
int ref_statevector(const char* circuit_text, const char* bitstrings_nl,
                    double* out) {
  try {
    Circuit c = parse_circuit(std::string(circuit_text));
    test::StateVector sv(c.n_qubits);
    sv.run(c);
    std::size_t o = 0;
    for (const std::string& b : split_lines(bitstrings_nl)) {
      Complex a = sv.amplitude(b);
      out[o++] = a.real();
      out[o++] = a.imag();
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

// ---- request ingestion (formats.cpp:42-83) ---------------------------------

int ref_read_samples(const char* text, std::uint64_t len, int order, char* out, std::uint64_t cap,
                     std::uint64_t* n_rows, int* n_qubits) {
  try {
    std::istringstream in(std::string(text, len));
    const std::vector<std::string> v =
        read_samples(in, order ? BitOrder::kQubit0Last : BitOrder::kQubit0First);
    std::uint64_t o = 0;
    for (const std::string& r : v) {
      if (o + r.size() > cap) throw std::runtime_error("capacity");
      std::memcpy(out + o, r.data(), r.size());
      o += r.size();
    }
    *n_rows = v.size();
    *n_qubits = v.empty() ? 0 : static_cast<int>(v.front().size());
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

int ref_format_amplitude_row(const char* bits, double re, double im, int order, char* out, std::uint64_t cap) {
  const std::string r = format_amplitude_row(std::string(bits), {re, im},
                                             order ? BitOrder::kQubit0Last : BitOrder::kQubit0First);
  if (r.size() + 1 > cap) return 1;
  std::memcpy(out, r.c_str(), r.size() + 1);
  return 0;
}

int ref_linear_xeb(int n, const double* probs, std::uint64_t count,
                   double* out) {
  try {
    *out = linear_xeb(n, std::vector<double>(probs, probs + count));
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

int ref_xeb_from_amplitudes(int n, const double* amps, std::uint64_t count,
                            double* out) {
  try {
    std::vector<std::complex<double>> a(count);
    for (std::uint64_t i = 0; i < count; ++i) a[i] = {amps[2 * i], amps[2 * i + 1]};
    *out = linear_xeb(n, probs_from_amplitudes(a));
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr);
  }
}

}  // extern "C"
