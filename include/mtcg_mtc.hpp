// mtcg_mtc.hpp — header-only drop-in for the reference's hot path.
//
// A maintainer of the reference (`mtc`, /root/reference/proj) adds this header
// and links libmtcg.so; then
//
//     mtc::gpu::eval_all(plan, d, as, opts)      // multieval.hpp:62-63
//     mtc::gpu::eval_sliced(plan, d, as, opts)   // multieval.hpp:69-70
//     mtc::gpu::linear_xeb(n, probs)             // xeb.hpp:38
//
// have the reference's signatures, return the reference's EvalResult and
// throw the reference's DataError / MemoryCapError (errors.hpp:26-55), so a
// caller such as cmd_amplitudes (tools/main.cpp:159-160) switches with a
// namespace change. The C ABI underneath is include/mtcg.h.
#ifndef MTCG_MTC_HPP
#define MTCG_MTC_HPP

#include <algorithm>
#include <complex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mtc/diagram.hpp"
#include "mtc/errors.hpp"
#include "mtc/multieval.hpp"
#include "mtc/plan.hpp"
#include "mtcg.h"

namespace mtc::gpu {

// Device precision: complex64 (default, 1e-4) or bit-exact complex128.
enum class Precision { C64 = MTCG_C64, C128 = MTCG_C128 };

// One GPU, or several GPUs of the node (eval_sliced spreads slices over
// min(EvalOptions.workers, GPUs) of them — the GPU analogue of the reference's
// worker threads, with the same guarantee: values bit-identical for every
// count, multieval.hpp:26-29, 64-68).
class Device {
 public:
  explicit Device(int device = 0, std::uint64_t hbm_cap = 0) : Device(std::vector<int>{device}, hbm_cap) {}
  explicit Device(const std::vector<int>& devices, std::uint64_t hbm_cap_per_gpu = 0) {
    char err[512] = {0};
    if (mtcg_create_multi(devices.data(), static_cast<int>(devices.size()), hbm_cap_per_gpu, &h_, err,
                          sizeof err) != MTCG_OK)
      throw std::runtime_error(std::string("mtcg_create_multi: ") + err);
  }
  ~Device() { mtcg_destroy(h_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  mtcg_handle* handle() const { return h_; }
  int count() const { return mtcg_device_count(h_); }

  // every visible GPU (device 0 the root)
  static Device& default_device() {
    static Device d(all_visible());
    return d;
  }
  static std::vector<int> all_visible() {
    std::vector<int> v(static_cast<std::size_t>(std::max(1, mtcg_visible_devices())));
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = static_cast<int>(i);
    return v;
  }

 private:
  mtcg_handle* h_ = nullptr;
};

namespace detail {

[[noreturn]] inline void rethrow(mtcg_status st, const char* err, int node) {
  if (st == MTCG_ERR_DATA) throw DataError(err);
  if (st == MTCG_ERR_MEMORY_CAP) throw MemoryCapError(err, node);
  throw std::logic_error(std::string("mtcg: ") + err);
}

inline EvalResult eval(const Plan& plan, const NetworkDiagram& d, const AssignmentSet& as,
                       const EvalOptions& opts, mtcg_eval_mode mode, Precision precision,
                       Device& dev) {
  // Plan (plan.hpp:33-45)
  std::vector<int32_t> left, right, slot;
  for (const Plan::Node& n : plan.nodes) {
    left.push_back(n.left);
    right.push_back(n.right);
    slot.push_back(n.slot);
  }
  std::vector<uint32_t> sliced(plan.sliced.begin(), plan.sliced.end());
  // AssignmentSet (diagram.hpp:61-68): one leg list per slot
  std::vector<int32_t> n_values, leg_begin{0};
  std::vector<uint32_t> legs;
  std::vector<double> values;
  for (const auto& vs : as.value_sets) {
    n_values.push_back(static_cast<int32_t>(vs.size()));
    for (const Leg& l : vs.front().legs()) legs.push_back(l.id);
    leg_begin.push_back(static_cast<int32_t>(legs.size()));
    for (const Tensor& t : vs)
      for (const Complex& c : t.data()) {
        values.push_back(c.real());
        values.push_back(c.imag());
      }
  }
  std::vector<uint32_t> tuples;
  for (const auto& t : as.tuples) tuples.insert(tuples.end(), t.begin(), t.end());
  std::vector<uint32_t> batch(as.batch_legs.begin(), as.batch_legs.end());

  mtcg_problem p{};
  p.n_nodes = static_cast<int32_t>(plan.nodes.size());
  p.node_left = left.data();
  p.node_right = right.data();
  p.node_slot = slot.data();
  p.root = plan.root;
  p.n_sliced = static_cast<int32_t>(sliced.size());
  p.sliced = sliced.data();
  p.n_legs = static_cast<uint32_t>(d.leg_count());
  p.n_closed = d.n_closed;
  p.leg_dims = d.leg_dims.data();
  p.n_slots = static_cast<int32_t>(as.value_sets.size());
  p.slot_n_values = n_values.data();
  p.slot_leg_begin = leg_begin.data();
  p.slot_legs = legs.data();
  p.values = values.data();
  p.n_requests = as.request_count();
  p.tuples = tuples.data();
  p.n_batch_legs = static_cast<int32_t>(batch.size());
  p.batch_legs = batch.data();

  mtcg_options o{};
  o.eval_mode = mode;
  o.precision = static_cast<int32_t>(precision);
  o.memory_cap_bytes = opts.memory_cap_bytes;
  o.workers = opts.workers;

  const std::size_t w = std::size_t{1} << batch.size();
  std::vector<double> out(2 * as.request_count() * w);
  EvalResult res;
  res.node_contractions.assign(plan.nodes.size(), 0);
  mtcg_result r{};
  r.values = out.data();
  r.values_capacity = as.request_count() * w;
  r.node_contractions = res.node_contractions.data();
  char err[1024] = {0};
  const mtcg_status st = mtcg_eval(dev.handle(), &p, &o, &r, err, sizeof err);
  if (st != MTCG_OK) rethrow(st, err, r.cap_node);

  std::vector<Leg> out_legs;
  for (int i = 0; i < r.n_out_legs; ++i) out_legs.push_back({r.out_legs[i], 2});
  res.values.reserve(as.request_count());
  for (std::size_t i = 0; i < as.request_count(); ++i) {
    std::vector<Complex> data(w);
    for (std::size_t e = 0; e < w; ++e)
      data[e] = {out[2 * (i * w + e)], out[2 * (i * w + e) + 1]};
    res.values.emplace_back(out_legs, std::move(data));
  }
  res.counters.mults = r.mults;
  res.counters.adds = r.adds;
  res.counters.rw = r.rw;
  res.peak_bytes = r.hbm_peak_bytes;
  return res;
}

}  // namespace detail

inline EvalResult eval_all(const Plan& plan, const NetworkDiagram& d, const AssignmentSet& as,
                           const EvalOptions& opts = {}, Precision precision = Precision::C64,
                           Device& dev = Device::default_device()) {
  return detail::eval(plan, d, as, opts, MTCG_EVAL_ALL, precision, dev);
}

inline EvalResult eval_sliced(const Plan& plan, const NetworkDiagram& d,
                              const AssignmentSet& as, const EvalOptions& opts = {},
                              Precision precision = Precision::C64,
                              Device& dev = Device::default_device()) {
  return detail::eval(plan, d, as, opts, MTCG_EVAL_SLICED, precision, dev);
}

inline double linear_xeb(int n, const std::vector<double>& probs,
                         Device& dev = Device::default_device()) {
  double f = 0.0;
  char err[512] = {0};
  const mtcg_status st =
      mtcg_linear_xeb(dev.handle(), n, probs.data(), probs.size(), &f, err, sizeof err);
  if (st != MTCG_OK) detail::rethrow(st, err, -1);
  return f;
}

}  // namespace mtc::gpu

#endif  // MTCG_MTC_HPP
