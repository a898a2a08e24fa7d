// The C ABI (include/mtcg.h): exception-free wrappers that map the engine's
// errors onto mtcg_status, as the reference CLI maps its exceptions onto exit
// codes (proj/tools/main.cpp:365-386).
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <memory>

#include "device.hpp"
#include "configs.hpp"
#include "planner.hpp"

using namespace mtcg;

struct mtcg_handle {
  Engine* engine = nullptr;
  uint64_t cap = 0;
};

struct mtcg_plan {
  std::unique_ptr<DevicePlan> dp;
};

namespace {

void set_err(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg);
  }
}

template <class F>
mtcg_status guarded(char* err, size_t errlen, int32_t* cap_node, F&& f) {
  if (cap_node) *cap_node = -1;
  try {
    f();
    return MTCG_OK;
  } catch (const MemoryCapError& e) {
    if (cap_node) *cap_node = e.node;
    set_err(err, errlen, e.what());
    return MTCG_ERR_MEMORY_CAP;
  } catch (const DataError& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_DATA;
  } catch (const CudaError& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    set_err(err, errlen, "host allocation failed");
    return MTCG_ERR_MEMORY_CAP;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_INTERNAL;
  }
}

mtcg_options default_options() {
  mtcg_options o;
  std::memset(&o, 0, sizeof o);
  o.eval_mode = MTCG_EVAL_AUTO;
  o.precision = MTCG_C64;
  o.workers = 1;
  return o;
}

void check_problem_pointers(const mtcg_problem* p) {
  if (!p) throw DataError("null problem");
  if ((p->n_nodes > 0 && (!p->node_left || !p->node_right || !p->node_slot)) ||
      (p->n_sliced > 0 && !p->sliced) || (p->n_legs > 0 && !p->leg_dims) ||
      (p->n_slots > 0 && (!p->slot_n_values || !p->slot_leg_begin)) ||
      (p->n_requests > 0 && p->n_slots > 0 && !p->tuples) ||
      (p->n_batch_legs > 0 && !p->batch_legs))
    throw DataError("null array in problem");
}

// Slice reuse keeps invariant tables resident across slices, outside the
// reference's per-slice accounting: it is dropped under an explicit cap
// (options or handle), where MemoryCapError must follow the reference.
mtcg_options effective_options(const mtcg_handle* h, mtcg_options o) {
  if (o.memory_cap_bytes || h->cap) o.flags &= ~MTCG_FLAG_SLICE_REUSE;
  return o;
}

uint64_t device_cap(const mtcg_handle* h, const mtcg_options& o) {
  if (o.memory_cap_bytes) return o.memory_cap_bytes;
  if (h->cap) return h->cap;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 0;
  free_b += engine_arena_bytes(h->engine);  // the cached arena is reusable
  return free_b > (256ull << 20) ? free_b - (256ull << 20) : free_b;
}

void fill_info(const Compiled& c, mtcg_plan_info* info) {
  std::memset(info, 0, sizeof *info);
  info->n_requests = c.n_requests;
  info->n_rows = c.n_rows;
  info->row_elems = c.row_elems;
  info->n_slices = c.n_slices;
  info->mults = c.mults;
  info->adds = c.adds;
  info->rw = c.rw;
  info->contractions = c.contractions;
  info->hbm_arena_bytes = c.arena_bytes();
  info->hbm_resident_bytes = c.resident_bytes();
  info->precision = c.precision;
  info->prologue_ops = c.n_prologue_ops;
  info->executed_contractions = c.executed_contractions;
  info->fused_chains = c.chains.size();
  info->fused_ops = 0;
  for (const Chain& ch : c.chains) info->fused_ops += static_cast<uint64_t>(ch.tail - ch.head + 1);
  int k = 0;
  for (const Op& op : c.ops)
    if (op.nb && (op.chain < 0 || op.chain_tail)) ++k;
  if (c.has_leaf_root && c.n_rows) ++k;
  info->n_kernels_per_slice = k;
}

void fetch_into(mtcg_plan* plan, const void* d_acc, void* stream, mtcg_result* res) {
  DevicePlan& dp = *plan->dp;
  const Compiled& c = dp.c;
  const uint64_t need = c.n_requests * c.row_elems;
  if (res->values && res->values_capacity < need)
    throw DataError("values buffer too small: need " + std::to_string(need) + " complex");
  const uint64_t n_elem = c.n_rows * c.row_elems;
  if (res->values && need) {
    std::vector<double> by_row(2 * n_elem);
    if (c.precision == MTCG_C64) {
      std::vector<float> tmp(2 * n_elem);
      copy_to_host(dp.engine, tmp.data(), d_acc, tmp.size() * sizeof(float), stream);
      for (size_t i = 0; i < tmp.size(); ++i) by_row[i] = tmp[i];
    } else {
      copy_to_host(dp.engine, by_row.data(), d_acc, by_row.size() * sizeof(double), stream);
    }
    // fan_out (multieval.cpp:374-380)
    for (uint64_t i = 0; i < c.n_requests; ++i)
      std::memcpy(res->values + 2 * i * c.row_elems,
                  by_row.data() + 2 * c.row_of_request[i] * c.row_elems,
                  sizeof(double) * 2 * c.row_elems);
  }
  if (res->node_contractions)
    std::memcpy(res->node_contractions, c.node_contractions.data(),
                sizeof(uint64_t) * c.node_contractions.size());
  res->mults = c.mults;
  res->adds = c.adds;
  res->rw = c.rw;
  res->hbm_peak_bytes = c.arena_bytes() + c.resident_bytes() + n_elem * c.elem_bytes;
  res->cap_node = -1;
  res->n_out_legs = static_cast<int32_t>(c.out_legs.size());
  for (size_t i = 0; i < c.out_legs.size() && i < 64; ++i) res->out_legs[i] = c.out_legs[i];
}

}  // namespace

extern "C" {

int mtcg_version(void) { return MTCG_ABI_VERSION; }

mtcg_status mtcg_create(int device, uint64_t hbm_cap_bytes, mtcg_handle** out, char* err,
                        size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!out) throw DataError("null output handle");
    auto h = std::make_unique<mtcg_handle>();
    h->engine = engine_create(device);
    h->cap = hbm_cap_bytes;
    *out = h.release();
  });
}

void mtcg_destroy(mtcg_handle* h) {
  if (!h) return;
  engine_destroy(h->engine);
  delete h;
}

mtcg_status mtcg_emulate(const mtcg_problem* p, const mtcg_options* opt, uint64_t cap_bytes,
                         mtcg_plan_info* info, uint64_t* node_contractions, int32_t* cap_node,
                         char* err, size_t errlen) {
  return guarded(err, errlen, cap_node, [&] {
    check_problem_pointers(p);
    const mtcg_options o = opt ? *opt : default_options();
    Compiled c = compile_problem(*p, o, cap_bytes);
    if (info) fill_info(c, info);
    if (node_contractions)
      std::memcpy(node_contractions, c.node_contractions.data(),
                  sizeof(uint64_t) * c.node_contractions.size());
  });
}

mtcg_status mtcg_compile(mtcg_handle* h, const mtcg_problem* p, const mtcg_options* opt,
                         mtcg_plan** out, int32_t* cap_node, char* err, size_t errlen) {
  return guarded(err, errlen, cap_node, [&] {
    if (!h || !out) throw DataError("null handle");
    check_problem_pointers(p);
    const mtcg_options o = effective_options(h, opt ? *opt : default_options());
    Compiled c = compile_problem(*p, o, device_cap(h, o));
    auto plan = std::make_unique<mtcg_plan>();
    plan->dp = upload_plan(h->engine, std::move(c));
    *out = plan.release();
  });
}

void mtcg_plan_destroy(mtcg_plan* plan) { delete plan; }

mtcg_status mtcg_plan_get_info(const mtcg_plan* plan, mtcg_plan_info* info) {
  if (!plan || !info) return MTCG_ERR_ARGUMENT;
  fill_info(plan->dp->c, info);
  return MTCG_OK;
}

mtcg_status mtcg_run(mtcg_plan* plan, uint64_t slice_begin, uint64_t slice_end, void* d_acc,
                     int accumulate, void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan) throw DataError("null plan");
    const Compiled& c = plan->dp->c;
    if (slice_begin > slice_end || slice_end > c.n_slices)
      throw DataError("slice range outside [0, " + std::to_string(c.n_slices) + ")");
    if (!d_acc && c.n_rows) throw DataError("null accumulator");
    run_slices(*plan->dp, slice_begin, slice_end, d_acc, accumulate != 0, stream);
  });
}

mtcg_status mtcg_fetch(mtcg_plan* plan, const void* d_acc, void* stream, mtcg_result* res,
                       char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan || !res) throw DataError("null argument");
    fetch_into(plan, d_acc, stream, res);
  });
}

mtcg_status mtcg_xeb_device(mtcg_plan* plan, const void* d_acc, int n_qubits, void* stream,
                            double* out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan || !out) throw DataError("null argument");
    const Compiled& c = plan->dp->c;
    if (c.n_requests == 0) throw DataError("linear_xeb needs at least one sample");
    if (n_qubits < 0 || n_qubits > 1022) throw DataError("qubit count out of range");
    *out = xeb_device(*plan->dp, d_acc, n_qubits, stream);
  });
}

mtcg_status mtcg_eval(mtcg_handle* h, const mtcg_problem* p, const mtcg_options* opt,
                      mtcg_result* res, char* err, size_t errlen) {
  int32_t cap_node = -1;
  mtcg_status st = guarded(err, errlen, &cap_node, [&] {
    if (!h || !res) throw DataError("null argument");
    check_problem_pointers(p);
    const mtcg_options o = effective_options(h, opt ? *opt : default_options());
    Compiled c = compile_problem(*p, o, device_cap(h, o));
    mtcg_plan plan;
    plan.dp = upload_plan(h->engine, std::move(c));
    const Compiled& cc = plan.dp->c;
    void* d_acc = device_alloc(h->engine, cc.n_rows * cc.row_elems * cc.elem_bytes);
    try {
      run_slices(*plan.dp, 0, cc.n_slices, d_acc, false, nullptr);
      fetch_into(&plan, d_acc, nullptr, res);
    } catch (...) {
      device_free(h->engine, d_acc);
      throw;
    }
    device_free(h->engine, d_acc);
  });
  if (res) res->cap_node = cap_node;
  return st;
}

mtcg_status mtcg_linear_xeb(mtcg_handle* h, int n_qubits, const double* probs, uint64_t count,
                            double* out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!h || !out) throw DataError("null argument");
    if (count == 0) throw DataError("linear_xeb needs at least one sample");
    if (n_qubits < 0 || n_qubits > 1022) throw DataError("qubit count out of range");
    *out = xeb_probs(h->engine, probs, count, n_qubits, false);
  });
}

mtcg_status mtcg_linear_xeb_amplitudes(mtcg_handle* h, int n_qubits, const double* amps,
                                       uint64_t count, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!h || !out) throw DataError("null argument");
    if (count == 0) throw DataError("linear_xeb needs at least one sample");
    if (n_qubits < 0 || n_qubits > 1022) throw DataError("qubit count out of range");
    *out = xeb_probs(h->engine, amps, count, n_qubits, true);
  });
}

int32_t mtcg_plan_op_count(const mtcg_plan* plan) {
  return plan ? static_cast<int32_t>(plan->dp->c.ops.size()) : 0;
}

mtcg_status mtcg_plan_op_info(const mtcg_plan* plan, int32_t i, mtcg_op_info* info) {
  if (!plan || !info || i < 0 || i >= static_cast<int32_t>(plan->dp->c.ops.size()))
    return MTCG_ERR_ARGUMENT;
  const Compiled& c = plan->dp->c;
  const Op& op = c.ops[i];
  info->node = op.node;
  info->kernel = op.chain >= 0 ? kChainConfig : op.config;
  info->fa = op.fa;
  info->fb = op.fb;
  info->kc = op.kc;
  info->batch = op.nb;
  info->mults = op.mults * op.nb;
  info->bytes = op.rw * op.nb * static_cast<uint64_t>(c.elem_bytes);
  auto distinct = [](std::vector<uint32_t> v) {
    std::sort(v.begin(), v.end());
    return static_cast<uint64_t>(std::unique(v.begin(), v.end()) - v.begin());
  };
  const Chain* ch = op.chain >= 0 ? &c.chains[op.chain] : nullptr;
  const bool reads_a = !ch || ch->head == i, writes_out = !ch || ch->tail == i;
  uint64_t elems = distinct(op.ib) * (op.b_item >> op.b_slice_stride.size());
  if (reads_a) elems += distinct(op.ia) * (op.a_item >> op.a_slice_stride.size());
  if (writes_out) elems += static_cast<uint64_t>(op.nb) * op.out_item;
  info->compulsory_bytes = elems * static_cast<uint64_t>(c.elem_bytes);
  return MTCG_OK;
}

mtcg_status mtcg_time_ops(mtcg_plan* plan, uint64_t slice, void* d_acc, int accumulate,
                          void* stream, float* op_ms, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan || !op_ms) throw DataError("null argument");
    if (slice >= plan->dp->c.n_slices) throw DataError("slice out of range");
    time_ops(*plan->dp, slice, d_acc, accumulate != 0, stream, op_ms);
  });
}

uint64_t mtcg_launch_count(const mtcg_handle* h) { return h ? engine_launches(h->engine) : 0; }

}  // extern "C"
