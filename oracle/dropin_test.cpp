// ORACLE TEST INFRASTRUCTURE — the reference's own types and tests, with the
// hot path swapped for the device engine through include/mtcg_mtc.hpp.
//
// Built by `make -C oracle dropin` against the reference headers and objects
// (oracle/_ref/), linked to the in-tree libmtcg.so; run on a GPU box by
// tests/test_gpu_dropin.py. Each criterion mirrors a reference test and
// prints one PASS/FAIL line (the acceptance_main.cpp convention):
//   1  worked example (multieval_test.cpp:78-116): amplitudes, node counts,
//      exact counters — complex128 device path bit-identical to eval_all
//   2  eval_all vs device on 100 random circuits/plans (multieval_test.cpp:
//      118-141 pattern): bit-identical in C128, 1e-4 relative in C64
//   3  sliced == reference eval_sliced, bit-identical (multieval_test.cpp:251-283)
//   4  batch legs (multieval_test.cpp:186-227)
//   5  memory cap -> mtc::MemoryCapError (multieval_test.cpp:333-349)
//   6  DataError on a sliced plan through eval_all (multieval_test.cpp:295-298)
//   7  linear_xeb equals the reference's on cfg-style probabilities
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mtc/multieval.hpp"
#include "mtc/xeb.hpp"
#include "mtcg_mtc.hpp"
#include "support/gen.hpp"

using namespace mtc;

namespace {

int g_fail = 0;

void report(int n, const char* name, bool pass, const std::string& detail) {
  std::printf("%s  criterion %d: %s  [%s]\n", pass ? "PASS" : "FAIL", n, name, detail.c_str());
  std::fflush(stdout);
  if (!pass) ++g_fail;
}

bool bit_equal(const EvalResult& a, const EvalResult& b) {
  if (a.values.size() != b.values.size()) return false;
  for (std::size_t i = 0; i < a.values.size(); ++i) {
    if (!(a.values[i].legs() == b.values[i].legs())) return false;
    for (std::size_t e = 0; e < a.values[i].data().size(); ++e)
      if (a.values[i].data()[e] != b.values[i].data()[e]) return false;
  }
  return a.node_contractions == b.node_contractions && a.counters == b.counters;
}

double max_rel(const EvalResult& got, const EvalResult& want, int n_qubits) {
  const double floor = std::pow(2.0, -n_qubits / 2.0);
  double worst = 0;
  for (std::size_t i = 0; i < want.values.size(); ++i)
    for (std::size_t e = 0; e < want.values[i].data().size(); ++e) {
      const Complex w = want.values[i].data()[e], g = got.values[i].data()[e];
      worst = std::max(worst, std::abs(g - w) / std::max(std::abs(w), floor));
    }
  return worst;
}

Plan random_plan(Rng& rng, std::size_t n_slots) {
  Plan p;
  std::vector<int> roots;
  for (std::size_t s = 0; s < n_slots; ++s) {
    p.nodes.push_back({-1, -1, static_cast<int>(s)});
    roots.push_back(static_cast<int>(s));
  }
  while (roots.size() > 1) {
    std::size_t i = rng.uniform_index(roots.size());
    int a = roots[i];
    roots.erase(roots.begin() + i);
    std::size_t j = rng.uniform_index(roots.size());
    int b = roots[j];
    roots.erase(roots.begin() + j);
    p.nodes.push_back({a, b, -1});
    roots.push_back(static_cast<int>(p.nodes.size()) - 1);
  }
  p.root = roots[0];
  return p;
}

}  // namespace

int main() {
  using gpu::Precision;
  {  // 1
    NetworkDiagram d = to_diagram(test::ghz_like_circuit(), false);
    Plan plan = parse_plan(test::kGhzPlanText);
    AssignmentSet as = build_assignments(d, {"000", "100", "111"}, {});
    EvalResult ref = eval_all(plan, d, as);
    EvalResult dev = gpu::eval_all(plan, d, as, {}, Precision::C128);
    EvalResult dev64 = gpu::eval_all(plan, d, as);
    bool pass = bit_equal(dev, ref) && max_rel(dev64, ref, 3) <= 1e-6;
    std::uint64_t total = 0;
    for (auto x : dev.node_contractions) total += x;
    pass = pass && total == 13;
    report(1, "worked example through the device engine", pass,
           "bit-identical (c128), 13 contractions, |amp| " +
               std::to_string(std::abs(dev.values[0].data()[0])));
  }
  {  // 2
    Rng rng(4711);
    bool pass = true;
    double worst = 0;
    for (int rep = 0; rep < 100 && pass; ++rep) {
      int n = 2 + static_cast<int>(rng.uniform_index(6));
      Circuit c = test::random_circuit(rng, n, 18);
      NetworkDiagram d = to_diagram(c, rep % 2 == 0);
      Plan plan = random_plan(rng, d.slot_count());
      int k = 1 + static_cast<int>(rng.uniform_index(10));
      AssignmentSet as = build_assignments(d, test::random_bitstrings(rng, n, k), {});
      EvalResult ref = eval_all(plan, d, as);
      pass = pass && bit_equal(gpu::eval_all(plan, d, as, {}, Precision::C128), ref);
      double e = max_rel(gpu::eval_all(plan, d, as), ref, n);
      worst = std::max(worst, e);
      pass = pass && e <= 1e-4;
    }
    report(2, "eval_all == device on 100 random instances", pass,
           "c128 bit-identical, c64 worst rel " + std::to_string(worst));
  }
  {  // 3
    Rng rng(1212);
    bool pass = true;
    for (int rep = 0; rep < 12 && pass; ++rep) {
      int n = 2 + static_cast<int>(rng.uniform_index(4));
      Circuit c = test::random_circuit(rng, n, 14);
      NetworkDiagram d = to_diagram(c, false);
      Plan plan = random_plan(rng, d.slot_count());
      AssignmentSet as = build_assignments(d, test::random_bitstrings(rng, n, 4), {});
      int n_slices = 1 + static_cast<int>(rng.uniform_index(3));
      for (int s = 0; s < n_slices; ++s) {
        LegId leg;
        do {
          leg = static_cast<LegId>(rng.uniform_index(d.n_closed));
        } while (std::find(plan.sliced.begin(), plan.sliced.end(), leg) != plan.sliced.end());
        plan.sliced.push_back(leg);
      }
      pass = bit_equal(gpu::eval_sliced(plan, d, as, {}, Precision::C128), eval_sliced(plan, d, as));
    }
    report(3, "eval_sliced == device (slice enumeration and fold)", pass, "12 instances, c128");
  }
  {  // 4
    Circuit c = parse_circuit(std::string("3\n0 h 0\n0 h 2\n1 cx 0 1\n2 fs 1 2 0.7 0.3\n"));
    NetworkDiagram d = to_diagram(c, false);
    Plan plan = left_deep_plan(d.slot_count());
    LegId q1 = d.open_legs[1];
    AssignmentSet as = build_assignments(d, {"0*0", "1*1"}, {q1});
    bool pass = bit_equal(gpu::eval_all(plan, d, as, {}, Precision::C128), eval_all(plan, d, as));
    report(4, "batch legs", pass, "values over the '*' leg, legs and data");
  }
  {  // 5
    Rng rng(77);
    Circuit c = test::random_circuit(rng, 5, 20);
    NetworkDiagram d = to_diagram(c, false);
    Plan plan = left_deep_plan(d.slot_count());
    AssignmentSet as = build_assignments(d, test::random_bitstrings(rng, 5, 3), {});
    EvalOptions tight;
    tight.memory_cap_bytes = 256;
    bool pass = false;
    std::string what;
    try {
      gpu::eval_all(plan, d, as, tight);
    } catch (const MemoryCapError& e) {
      what = e.what();
      pass = what.find("memory cap exceeded") != std::string::npos && e.node() >= 0;
    }
    report(5, "memory cap raises MemoryCapError with the node", pass, what);
  }
  {  // 6
    Circuit c = parse_circuit(std::string("1\n0 h 0\n"));
    NetworkDiagram d = to_diagram(c, false);
    Plan plan = parse_plan("0 1\nslice: 0\n");
    AssignmentSet as = build_assignments(d, {"0"}, {});
    bool pass = false;
    try {
      gpu::eval_all(plan, d, as);
    } catch (const DataError& e) {
      pass = std::string(e.what()) == "plan has sliced legs; use eval_sliced";
    }
    EvalResult r = gpu::eval_sliced(plan, d, as, {}, Precision::C128);
    pass = pass && std::abs(r.values[0].data()[0] - Complex{1 / std::sqrt(2.0), 0}) < 1e-12;
    report(6, "DataError semantics and the sliced H golden", pass, "");
  }
  {  // 7
    Circuit c = test::grid_circuit(3, 4, 8, 12345);
    NetworkDiagram d = to_diagram(c, true);
    Rng rng(99);
    auto bits = test::random_bitstrings(rng, 12, 1000);
    AssignmentSet as = build_assignments(d, bits, {});
    Plan plan = left_deep_plan(d.slot_count());
    std::vector<std::complex<double>> amps;
    for (const Tensor& t : gpu::eval_all(plan, d, as, {}, Precision::C128).values)
      amps.push_back(t.data()[0]);
    std::vector<double> probs = probs_from_amplitudes(amps);
    double a = linear_xeb(12, probs), b = gpu::linear_xeb(12, probs);
    report(7, "linear_xeb on the device", std::abs(a - b) <= 1e-12 * std::max(1.0, std::abs(a)),
           std::to_string(a) + " vs " + std::to_string(b));
  }
  {  // 8: workers -> GPUs (multieval_test.cpp:251-283: workers=4 bit-identical
     // to workers=1); a 4-device handle over GPU 0 listed four times when the
     // box has one GPU (the same per-device schedule, copies for NCCL)
    std::vector<int> devs = gpu::Device::all_visible();
    while (devs.size() < 4) devs.push_back(0);
    gpu::Device multi(devs);
    Rng rng(4711);
    bool pass = true;
    for (int rep = 0; rep < 8 && pass; ++rep) {
      int n = 2 + static_cast<int>(rng.uniform_index(4));
      Circuit c = test::random_circuit(rng, n, 16);
      NetworkDiagram d = to_diagram(c, false);
      Plan plan = random_plan(rng, d.slot_count());
      AssignmentSet as = build_assignments(d, test::random_bitstrings(rng, n, 5), {});
      for (int s = 0; s < 3; ++s) {
        LegId leg;
        do {
          leg = static_cast<LegId>(rng.uniform_index(d.n_closed));
        } while (std::find(plan.sliced.begin(), plan.sliced.end(), leg) != plan.sliced.end());
        plan.sliced.push_back(leg);
      }
      EvalOptions w1, w4;
      w1.workers = 1;
      w4.workers = 4;
      const EvalResult ref = eval_sliced(plan, d, as, w4);
      pass = bit_equal(gpu::eval_sliced(plan, d, as, w1, Precision::C128, multi), ref) &&
             bit_equal(gpu::eval_sliced(plan, d, as, w4, Precision::C128, multi), ref);
    }
    report(8, "eval_sliced workers=4 on 4 devices == workers=1 == reference", pass,
           std::to_string(multi.count()) + " devices, 8 instances x 8 slices, c128");
  }
  if (g_fail) {
    std::printf("%d criterion(s) failed\n", g_fail);
    return 1;
  }
  std::printf("all drop-in criteria passed\n");
  return 0;
}
