// The C ABI (include/mtcg.h): exception-free wrappers that map the engine's
// errors onto mtcg_status, as the reference CLI maps its exceptions onto exit
// codes (proj/tools/main.cpp:365-386).
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>

#include <dlfcn.h>
#include <nccl.h>

#include <numeric>
#include <set>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "device.hpp"
#include "configs.hpp"
#include "planner.hpp"
#include "ingest.hpp"

using namespace mtcg;

struct mtcg_handle {
  Engine* engine = nullptr;          // root: engines[0]
  std::vector<Engine*> engines;      // one per listed device (repeats allowed)
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;     // distinct devices: one NCCL rank each
  uint64_t cap = 0;
};

struct mtcg_plan {
  std::unique_ptr<DevicePlan> dp;  // the schedule; chunk 0 of a chunked plan
  // memo streaming (mtcg_options.row_chunk): one schedule per request chunk
  // sharing the request-independent prologue; the caller's accumulator holds
  // the chunks' rows back to back
  struct Chunked {
    std::vector<std::unique_ptr<DevicePlan>> rest;  // chunks 1..
    std::vector<uint64_t> row_off;                  // first accumulator row per chunk
    std::vector<uint64_t> req_off;                  // first request (in `order`) per chunk
    std::vector<uint64_t> order;                    // requests in lexicographic tuple order
    uint64_t rows = 0;                              // accumulator rows, all chunks
    std::unique_ptr<Compiled> whole;                // the whole evaluation's counts
    DevicePlan& chunk(size_t c, mtcg_plan& pl) { return c == 0 ? *pl.dp : *rest[c - 1]; }
    size_t n() const { return rest.size() + 1; }
  };
  std::unique_ptr<Chunked> chunked;
};

namespace {

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_err(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg);
  }
}

// NVTX ranges around the ABI entry points (visible in Nsight Systems /
// Compute timelines; no-ops without a profiler attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

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
  } catch (const ParseError& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_PARSE;
  } catch (const CudaError& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_CUDA;
  } catch (const NcclError& e) {
    set_err(err, errlen, e.what());
    return MTCG_ERR_NCCL;
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

// GPU the tuple index is built on (-1: the host builder). Below 2^15
// requests the host builder is as fast (k = 10^4: 4.9 vs 4.3 ms) and leaves
// the GPU to the previous evaluation's kernels.
int index_device(const mtcg_handle* h, const mtcg_problem& p, const mtcg_options& o) {
  if (o.flags & MTCG_FLAG_HOST_INDEX) return -1;
  if (!(o.flags & MTCG_FLAG_DEVICE_INDEX) && p.n_requests < (uint64_t{1} << 15)) return -1;
  return engine_device(h->engine);
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

// ---- NCCL (loaded on first use: the process may already hold torch's
// libnccl.so.2, which dlopen then shares) -------------------------------------
struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw NcclError(std::string("libnccl.so.2 not loadable: ") + dlerror());
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) throw NcclError(std::string("NCCL symbol missing: ") + name);
      return f;
    };
    r.init_all = reinterpret_cast<decltype(r.init_all)>(sym("ncclCommInitAll"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(sym("ncclCommDestroy"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(sym("ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(sym("ncclGroupEnd"));
    r.send = reinterpret_cast<decltype(r.send)>(sym("ncclSend"));
    r.recv = reinterpret_cast<decltype(r.recv)>(sym("ncclRecv"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(sym("ncclGetErrorString"));
    return r;
  }();
  return n;
}

#define NCK(x)                                                                     \
  do {                                                                             \
    ncclResult_t r__ = (x);                                                        \
    if (r__ != ncclSuccess) throw NcclError(std::string(#x) + ": " + nccl().error_string(r__)); \
  } while (0)

#define CCK(x)                                                                     \
  do {                                                                             \
    cudaError_t e__ = (x);                                                         \
    if (e__ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// Device buffer owned for one call.
struct DevBuf {
  Engine* e = nullptr;
  void* p = nullptr;
  DevBuf(Engine* eng, uint64_t bytes) : e(eng), p(bytes ? device_alloc(eng, bytes) : nullptr) {}
  ~DevBuf() {
    if (p) device_free(e, p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// eval_sliced over several devices: rounds of R slices per device in
// contiguous blocks (device g: [base + g R, base + (g + 1) R)), each slice's
// root values gathered to the root in slice order, folded there in slice
// order (bit-identical to one device). One host thread issues every device's
// asynchronous work; NCCL send/recv pairs (one group per round) or device
// copies (repeated devices) carry the values; device streams order reuse of
// the per-device and root buffers across rounds.
// Fewer slices than devices (SURVEY §8e fallback): the requests, in
// lexicographic tuple order, are split into one contiguous block per device;
// each device evaluates its block over every slice with its own memo (the
// request-independent subtrees repeat per device) and the rows come back to
// the host by request — no cross-device sum, so every value is the one the
// owning device computes alone (complex128: the reference's bits for any
// device count). Counts and node_contractions are the whole evaluation's.
void eval_multi_rows(mtcg_handle* h, const mtcg_problem* p, const mtcg_options& o, int n_use, mtcg_result* res) {
  const uint64_t K = p->n_requests;
  const int ns = p->n_slots;
  mtcg_options oc = o;
  oc.row_chunk = 0;
  oc.flags &= ~MTCG_FLAG_SLICE_REUSE;
  const Compiled whole = compile_problem(*p, oc, 0, nullptr, -1);  // exact counts, validation
  const uint64_t need = K * whole.row_elems;
  if (res->values && res->values_capacity < need)
    throw DataError("values buffer too small: need " + std::to_string(need) + " complex");
  std::vector<uint64_t> order(K);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
    return std::lexicographical_compare(p->tuples + a * ns, p->tuples + (a + 1) * ns, p->tuples + b * ns,
                                        p->tuples + (b + 1) * ns);
  });
  struct Part {
    uint64_t r0 = 0, r1 = 0;
    std::vector<uint32_t> tuples;
    std::unique_ptr<mtcg_plan> plan;
    std::unique_ptr<DevBuf> acc;
  };
  std::vector<Part> parts(n_use);
  // compile + enqueue every device's block, then collect
  for (int g = 0; g < n_use; ++g) {
    Part& pt = parts[g];
    pt.r0 = K * g / n_use;
    pt.r1 = K * (g + 1) / n_use;
    if (pt.r1 <= pt.r0) continue;
    pt.tuples.resize((pt.r1 - pt.r0) * ns);
    for (uint64_t r = pt.r0; r < pt.r1; ++r)
      std::memcpy(pt.tuples.data() + (r - pt.r0) * ns, p->tuples + order[r] * ns, sizeof(uint32_t) * ns);
    mtcg_problem q = *p;
    q.n_requests = pt.r1 - pt.r0;
    q.tuples = pt.tuples.data();
    CCK(cudaSetDevice(h->devices[g]));
    pt.plan = std::make_unique<mtcg_plan>();
    pt.plan->dp = upload_plan(h->engines[g], compile_problem(q, oc, device_cap(h, oc), nullptr, -1));
    const Compiled& cg = pt.plan->dp->c;
    pt.acc = std::make_unique<DevBuf>(h->engines[g], cg.n_rows * cg.row_elems * cg.elem_bytes);
    run_slices(*pt.plan->dp, 0, cg.n_slices, pt.acc->p, false, nullptr);
  }
  std::vector<double> vals;
  uint64_t peak = 0;
  for (int g = 0; g < n_use; ++g) {
    Part& pt = parts[g];
    if (!pt.plan) continue;
    CCK(cudaSetDevice(h->devices[g]));
    const uint64_t n = pt.r1 - pt.r0;
    vals.assign(2 * n * whole.row_elems, 0.0);
    mtcg_result sub;
    std::memset(&sub, 0, sizeof sub);
    sub.values = vals.data();
    sub.values_capacity = n * whole.row_elems;
    fetch_into(pt.plan.get(), pt.acc->p, nullptr, &sub);
    peak = std::max<uint64_t>(peak, sub.hbm_peak_bytes);
    if (res->values)
      for (uint64_t i = 0; i < n; ++i)
        std::memcpy(res->values + 2 * order[pt.r0 + i] * whole.row_elems, vals.data() + 2 * i * whole.row_elems,
                    sizeof(double) * 2 * whole.row_elems);
  }
  CCK(cudaSetDevice(h->devices[0]));
  if (res->node_contractions)
    std::memcpy(res->node_contractions, whole.node_contractions.data(),
                sizeof(uint64_t) * whole.node_contractions.size());
  res->mults = whole.mults;
  res->adds = whole.adds;
  res->rw = whole.rw;
  res->hbm_peak_bytes = peak;
  res->cap_node = -1;
  res->n_out_legs = static_cast<int32_t>(whole.out_legs.size());
  for (size_t i = 0; i < whole.out_legs.size() && i < 64; ++i) res->out_legs[i] = whole.out_legs[i];
}

void eval_multi(mtcg_handle* h, const mtcg_problem* p, const mtcg_options& o, int n_use, mtcg_result* res) {
  Compiled c = compile_problem(*p, o, device_cap(h, o), nullptr, index_device(h, *p, o));
  std::vector<std::unique_ptr<DevicePlan>> plans;
  for (int g = 0; g < n_use; ++g) {
    Compiled cg = c;  // host copy per device
    plans.push_back(upload_plan(h->engines[g], std::move(cg)));
  }
  const Compiled& cc = plans[0]->c;
  const uint64_t S = cc.n_slices, ne = cc.n_rows * cc.row_elems, eb = cc.elem_bytes;
  const uint64_t slice_bytes = ne * eb;
  // slices per device per round: all at once when the per-slice values fit
  // in 512 MB per device
  uint64_t R = (S + n_use - 1) / n_use;
  if (slice_bytes) R = std::max<uint64_t>(1, std::min<uint64_t>(R, (512ull << 20) / slice_bytes));
  const bool use_nccl = !h->comms.empty() && static_cast<int>(h->comms.size()) >= n_use;
  Engine* root = h->engines[0];
  DevBuf acc(root, slice_bytes);
  DevBuf gather(root, static_cast<uint64_t>(n_use) * R * slice_bytes);
  std::vector<std::unique_ptr<DevBuf>> stage, parts;
  for (int g = 0; g < n_use; ++g) {
    stage.push_back(std::make_unique<DevBuf>(h->engines[g], slice_bytes));
    // the root writes its per-slice values straight into the gather buffer
    parts.push_back(std::make_unique<DevBuf>(h->engines[g], g == 0 ? 0 : R * slice_bytes));
  }
  std::vector<cudaEvent_t> ev_done(n_use, nullptr);
  cudaEvent_t ev_fold = nullptr;
  auto cleanup = [&] {
    for (int g = 0; g < n_use; ++g)
      if (ev_done[g]) {
        cudaSetDevice(h->devices[g]);
        cudaEventDestroy(ev_done[g]);
      }
    if (ev_fold) {
      cudaSetDevice(h->devices[0]);
      cudaEventDestroy(ev_fold);
    }
  };
  try {
    for (int g = 0; g < n_use; ++g) {
      CCK(cudaSetDevice(h->devices[g]));
      CCK(cudaEventCreateWithFlags(&ev_done[g], cudaEventDisableTiming));
    }
    CCK(cudaSetDevice(h->devices[0]));
    CCK(cudaEventCreateWithFlags(&ev_fold, cudaEventDisableTiming));
    auto dstream = [&](int g) { return static_cast<cudaStream_t>(engine_stream(h->engines[g])); };
    uint8_t* gbuf = static_cast<uint8_t*>(gather.p);
    for (uint64_t base = 0, round = 0; base < S; base += static_cast<uint64_t>(n_use) * R, ++round) {
      std::vector<uint64_t> cnt(n_use, 0);
      for (int g = 0; g < n_use; ++g) {
        const uint64_t lo = base + g * R, hi = std::min(S, lo + R);
        if (lo >= hi) continue;
        cnt[g] = hi - lo;
        CCK(cudaSetDevice(h->devices[g]));
        void* out = g == 0 ? static_cast<void*>(gbuf) : parts[g]->p;
        run_slices(*plans[g], lo, hi, stage[g]->p, false, nullptr, out);
      }
      if (use_nccl) {
        const ncclDataType_t t = cc.precision == MTCG_C64 ? ncclFloat32 : ncclFloat64;
        NCK(nccl().group_start());
        for (int g = 1; g < n_use; ++g) {
          if (!cnt[g]) continue;
          const size_t count = cnt[g] * ne * 2;
          NCK(nccl().recv(gbuf + g * R * slice_bytes, count, t, g, h->comms[0], dstream(0)));
          NCK(nccl().send(parts[g]->p, count, t, 0, h->comms[g], dstream(g)));
        }
        NCK(nccl().group_end());
      } else {
        for (int g = 1; g < n_use; ++g) {
          if (!cnt[g]) continue;
          CCK(cudaSetDevice(h->devices[g]));
          // the root's gather slots are free once the previous round's fold ran
          if (round > 0) CCK(cudaStreamWaitEvent(dstream(g), ev_fold, 0));
          CCK(cudaMemcpyPeerAsync(gbuf + g * R * slice_bytes, h->devices[0], parts[g]->p, h->devices[g],
                                  cnt[g] * slice_bytes, dstream(g)));
          CCK(cudaEventRecord(ev_done[g], dstream(g)));
          CCK(cudaSetDevice(h->devices[0]));
          CCK(cudaStreamWaitEvent(dstream(0), ev_done[g], 0));
        }
      }
      uint64_t total = 0;
      for (uint64_t x : cnt) total += x;
      fold_slices(root, cc.precision, gbuf, total, ne, acc.p, round > 0, nullptr);
      CCK(cudaSetDevice(h->devices[0]));
      CCK(cudaEventRecord(ev_fold, dstream(0)));
    }
    for (int g = 0; g < n_use; ++g) {
      CCK(cudaSetDevice(h->devices[g]));
      CCK(cudaStreamSynchronize(dstream(g)));
    }
    CCK(cudaSetDevice(h->devices[0]));
    mtcg_plan plan;
    plan.dp = std::move(plans[0]);
    fetch_into(&plan, acc.p, nullptr, res);
    plans[0] = std::move(plan.dp);
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

// mtcg_eval with options.row_chunk: memo streaming. The requests, in
// lexicographic tuple order (the reference walks rows in lexicographic order
// with a one-entry left cache and per-node right dictionaries dropped at last
// use, multieval.cpp:199-274), are cut into chunks of row_chunk; each chunk is
// compiled as its own schedule whose request-independent subtrees form a
// prologue laid out identically in every chunk (planner: request_dependent_
// slots). Per slice the first chunk runs the prologue, then every chunk runs
// its own ops against the resident prologue tables: the memo tables hold one
// chunk's distinct tuples, the request-independent work is not repeated.
// Values are each row's own slice sums, folded in slice order as without
// chunking; counters and node_contractions are the whole evaluation's.
std::unique_ptr<mtcg_plan> compile_chunked(mtcg_handle* h, const mtcg_problem* p, const mtcg_options& o) {
  const uint64_t K = p->n_requests, B = o.row_chunk;
  const int ns = p->n_slots;
  std::vector<char> dep(ns, 0);
  for (int j = 0; j < ns; ++j) dep[j] = p->slot_n_values[j] > 1;
  mtcg_options oc = o;
  oc.row_chunk = 0;
  oc.flags &= ~MTCG_FLAG_SLICE_REUSE;
  auto plan = std::make_unique<mtcg_plan>();
  plan->chunked = std::make_unique<mtcg_plan::Chunked>();
  auto& ch = *plan->chunked;
  // the whole evaluation's exact counts (host only; no device schedule kept)
  ch.whole = std::make_unique<Compiled>(compile_problem(*p, oc, 0, nullptr, index_device(h, *p, oc)));
  ch.order.resize(K);
  std::iota(ch.order.begin(), ch.order.end(), 0);
  std::stable_sort(ch.order.begin(), ch.order.end(), [&](uint64_t a, uint64_t b) {
    return std::lexicographical_compare(p->tuples + a * ns, p->tuples + (a + 1) * ns, p->tuples + b * ns,
                                        p->tuples + (b + 1) * ns);
  });
  const uint64_t n_chunks = (K + B - 1) / B;
  std::vector<uint32_t> tuples;
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const uint64_t r0 = c * B, r1 = std::min(K, r0 + B);
    tuples.resize((r1 - r0) * ns);
    for (uint64_t r = r0; r < r1; ++r)
      std::memcpy(tuples.data() + (r - r0) * ns, p->tuples + ch.order[r] * ns, sizeof(uint32_t) * ns);
    mtcg_problem q = *p;
    q.n_requests = r1 - r0;
    q.tuples = tuples.data();
    auto dp = upload_plan(h->engine, compile_problem(q, oc, device_cap(h, oc), &dep, index_device(h, q, oc)));
    ch.req_off.push_back(r0);
    ch.row_off.push_back(ch.rows);
    ch.rows += dp->c.n_rows;
    if (c == 0)
      plan->dp = std::move(dp);
    else
      ch.rest.push_back(std::move(dp));
  }
  // the shared arena at its largest before any run
  for (size_t c = 0; c < ch.n(); ++c) ensure_arena(ch.chunk(c, *plan));
  return plan;
}

void run_chunked(mtcg_plan& plan, uint64_t s0, uint64_t s1, void* d_acc, bool accumulate, void* stream) {
  auto& ch = *plan.chunked;
  for (size_t c = 0; c < ch.n(); ++c) ensure_arena(ch.chunk(c, plan));
  const Compiled& c0 = plan.dp->c;
  const uint64_t row_bytes = c0.row_elems * static_cast<uint64_t>(c0.elem_bytes);
  for (uint64_t s = s0; s < s1; ++s)
    for (size_t c = 0; c < ch.n(); ++c)
      run_slice_chunk(ch.chunk(c, plan), s, static_cast<uint8_t*>(d_acc) + ch.row_off[c] * row_bytes,
                      accumulate || s > s0, c == 0, stream);
}

void fetch_chunked(mtcg_plan& plan, const void* d_acc, void* stream, mtcg_result* res) {
  auto& ch = *plan.chunked;
  const Compiled& whole = *ch.whole;
  const uint64_t K = whole.n_requests, w = whole.row_elems;
  if (res->values && res->values_capacity < K * w)
    throw DataError("values buffer too small: need " + std::to_string(K * w) + " complex");
  const uint64_t row_bytes = w * static_cast<uint64_t>(whole.elem_bytes);
  for (size_t c = 0; c < ch.n(); ++c) {
    DevicePlan& dp = ch.chunk(c, plan);
    const uint64_t cnt = dp.c.n_requests;
    std::vector<double> vals(2 * cnt * w);
    mtcg_result sub{};
    sub.values = vals.data();
    sub.values_capacity = cnt * w;
    mtcg_plan one;
    one.dp.reset(&dp);  // borrowed for fetch_into
    try {
      fetch_into(&one, static_cast<const uint8_t*>(d_acc) + ch.row_off[c] * row_bytes, stream, &sub);
    } catch (...) {
      one.dp.release();
      throw;
    }
    one.dp.release();
    if (res->values)
      for (uint64_t i = 0; i < cnt; ++i)
        std::memcpy(res->values + 2 * ch.order[ch.req_off[c] + i] * w, vals.data() + 2 * i * w,
                    sizeof(double) * 2 * w);
    if (c == 0) {
      res->n_out_legs = sub.n_out_legs;
      std::memcpy(res->out_legs, sub.out_legs, sizeof(res->out_legs));
    }
  }
  if (res->node_contractions)
    std::memcpy(res->node_contractions, whole.node_contractions.data(),
                sizeof(uint64_t) * whole.node_contractions.size());
  res->mults = whole.mults;
  res->adds = whole.adds;
  res->rw = whole.rw;
  uint64_t peak = 0;
  for (size_t c = 0; c < ch.n(); ++c)
    peak = std::max(peak, ch.chunk(c, plan).c.arena_bytes() + ch.chunk(c, plan).c.resident_bytes());
  res->hbm_peak_bytes = peak + ch.rows * row_bytes;
  res->cap_node = -1;
}

void eval_chunked(mtcg_handle* h, const mtcg_problem* p, const mtcg_options& o, mtcg_result* res) {
  std::unique_ptr<mtcg_plan> plan = compile_chunked(h, p, o);
  const uint64_t row_bytes = plan->dp->c.row_elems * static_cast<uint64_t>(plan->dp->c.elem_bytes);
  DevBuf acc(h->engine, plan->chunked->rows * row_bytes);
  run_chunked(*plan, 0, plan->chunked->whole->n_slices, acc.p, false, nullptr);
  fetch_chunked(*plan, acc.p, nullptr, res);
}

}  // namespace

extern "C" {

int mtcg_version(void) { return MTCG_ABI_VERSION; }

mtcg_status mtcg_create(int device, uint64_t hbm_cap_bytes, mtcg_handle** out, char* err,
                        size_t errlen) {
  return mtcg_create_multi(&device, 1, hbm_cap_bytes, out, err, errlen);
}

mtcg_status mtcg_create_multi(const int* devices, int n_devices, uint64_t hbm_cap_bytes_per_gpu,
                              mtcg_handle** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!out) throw DataError("null output handle");
    if (!devices || n_devices < 1) throw DataError("no devices");
    int visible = 0;
    CCK(cudaGetDeviceCount(&visible));
    for (int i = 0; i < n_devices; ++i)
      if (devices[i] < 0 || devices[i] >= visible)
        throw DataError("device " + std::to_string(devices[i]) + " not visible (" + std::to_string(visible) +
                        " devices)");
    auto h = std::make_unique<mtcg_handle>();
    h->cap = hbm_cap_bytes_per_gpu;
    h->devices.assign(devices, devices + n_devices);
    try {
      for (int d : h->devices) h->engines.push_back(engine_create(d));
      h->engine = h->engines[0];
      const std::set<int> distinct(h->devices.begin(), h->devices.end());
      if (n_devices > 1 && static_cast<int>(distinct.size()) == n_devices) {
        h->comms.assign(n_devices, nullptr);
        NCK(nccl().init_all(h->comms.data(), n_devices, h->devices.data()));
      }
    } catch (...) {
      for (ncclComm_t c : h->comms)
        if (c) nccl().destroy(c);
      for (Engine* e : h->engines) engine_destroy(e);
      throw;
    }
    *out = h.release();
  });
}

int32_t mtcg_device_count(const mtcg_handle* h) { return h ? static_cast<int32_t>(h->engines.size()) : 0; }

int32_t mtcg_visible_devices(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

void mtcg_destroy(mtcg_handle* h) {
  if (!h) return;
  for (ncclComm_t c : h->comms)
    if (c) nccl().destroy(c);
  for (Engine* e : h->engines) engine_destroy(e);
  delete h;
}

mtcg_status mtcg_read_samples(const char* text, uint64_t len, int32_t bit_order, char* out,
                              uint64_t out_capacity, uint64_t* n_rows, int32_t* n_qubits, char* err,
                              size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if ((!text && len) || !n_rows || !n_qubits) throw DataError("null argument");
    SampleMatrix m = read_samples(text, len, bit_order);
    if (m.chars.size() > out_capacity || (!out && !m.chars.empty())) throw DataError("sample output capacity");
    if (!m.chars.empty()) std::memcpy(out, m.chars.data(), m.chars.size());
    *n_rows = m.n_rows;
    *n_qubits = m.n_qubits;
  });
}

mtcg_status mtcg_assign(const char* samples, uint64_t n_rows, int32_t n_qubits, int32_t n_slots,
                        const int32_t* slot_qubit_begin, const int32_t* slot_qubits, uint32_t* tuples,
                        int32_t* slot_n_values, uint64_t* value_key_begin, uint32_t* value_keys,
                        uint64_t keys_capacity, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if ((!samples && n_rows) || n_slots < 0 || n_qubits < 0 || !slot_qubit_begin ||
        (!slot_qubits && slot_qubit_begin[n_slots] > 0) || (!tuples && n_rows && n_slots) || !slot_n_values ||
        !value_key_begin)
      throw DataError("null argument");
    Assignment a = assign(samples, n_rows, n_qubits, n_slots, slot_qubit_begin, slot_qubits, tuples);
    if (a.value_keys.size() > keys_capacity || !value_keys) throw DataError("value key capacity");
    std::memcpy(slot_n_values, a.slot_n_values.data(), a.slot_n_values.size() * 4);
    std::memcpy(value_key_begin, a.value_key_begin.data(), a.value_key_begin.size() * 8);
    std::memcpy(value_keys, a.value_keys.data(), a.value_keys.size() * 4);
  });
}

mtcg_status mtcg_write_amplitudes(const char* path, const char* samples, uint64_t n_rows, int32_t n_qubits,
                                  int32_t bit_order, const double* values, int32_t w, uint64_t* written,
                                  char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!path || (!samples && n_rows) || (!values && n_rows) || w < 0 || w > 30) throw DataError("bad argument");
    const std::string text = format_amplitudes(samples, n_rows, n_qubits, bit_order, values, w);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw DataError(std::string("cannot open output file: ") + path);
    const size_t put = text.empty() ? 0 : std::fwrite(text.data(), 1, text.size(), f);
    const bool ok = std::fclose(f) == 0 && put == text.size();
    if (!ok) throw DataError(std::string("cannot write output file: ") + path);
    if (written) *written = text.size();
  });
}

mtcg_status mtcg_tuple_index_check(mtcg_handle* h, const mtcg_problem* p, int32_t* equal, uint64_t* rows,
                                   double* host_ms, double* device_ms, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!h) throw DataError("null handle");
    check_problem_pointers(p);
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    const TupleIndex a = tuple_index(*p, -1);
    auto t1 = clk::now();
    const TupleIndex b = tuple_index(*p, engine_device(h->engine));
    auto t2 = clk::now();
    bool eq = a.rows == b.rows && a.row_of_request == b.row_of_request &&
              a.row_tuple_first == b.row_tuple_first && a.distinct == b.distinct &&
              a.rank_value == b.rank_value && a.pair_l == b.pair_l && a.pair_r == b.pair_r;
    if (eq && a.rows) {
      const uint32_t* ra = a.rank[p->root];
      const uint32_t* rb = b.rank[p->root];
      eq = ra && rb && std::equal(ra, ra + a.rows, rb);
    }
    if (equal) *equal = eq;
    if (rows) *rows = a.rows;
    if (host_ms) *host_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (device_ms) *device_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  });
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
  NvtxRange nv("mtcg_compile");
  return guarded(err, errlen, cap_node, [&] {
    if (!h || !out) throw DataError("null handle");
    check_problem_pointers(p);
    const mtcg_options o = effective_options(h, opt ? *opt : default_options());
    if (o.row_chunk && o.row_chunk < p->n_requests) {
      *out = compile_chunked(h, p, o).release();
      return;
    }
    Compiled c = compile_problem(*p, o, device_cap(h, o), nullptr, index_device(h, *p, o));
    auto plan = std::make_unique<mtcg_plan>();
    plan->dp = upload_plan(h->engine, std::move(c));
    *out = plan.release();
  });
}

void mtcg_plan_destroy(mtcg_plan* plan) { delete plan; }

mtcg_status mtcg_plan_get_info(const mtcg_plan* plan, mtcg_plan_info* info) {
  if (!plan || !info) return MTCG_ERR_ARGUMENT;
  if (plan->chunked) {
    fill_info(*plan->chunked->whole, info);
    info->n_rows = plan->chunked->rows;  // the accumulator: every chunk's rows
    uint64_t arena = 0, resident = 0;
    for (size_t c = 0; c < plan->chunked->n(); ++c) {
      const Compiled& cc = plan->chunked->chunk(c, *const_cast<mtcg_plan*>(plan)).c;
      arena = std::max(arena, cc.arena_bytes());
      resident += cc.resident_bytes();
    }
    info->hbm_arena_bytes = arena;
    info->hbm_resident_bytes = resident;
    info->prologue_ops = plan->dp->c.n_prologue_ops;
    return MTCG_OK;
  }
  fill_info(plan->dp->c, info);
  return MTCG_OK;
}

mtcg_status mtcg_run(mtcg_plan* plan, uint64_t slice_begin, uint64_t slice_end, void* d_acc,
                     int accumulate, void* stream, char* err, size_t errlen) {
  NvtxRange nv("mtcg_run");
  return guarded(err, errlen, nullptr, [&] {
    if (!plan) throw DataError("null plan");
    const Compiled& c = plan->dp->c;
    if (slice_begin > slice_end || slice_end > c.n_slices)
      throw DataError("slice range outside [0, " + std::to_string(c.n_slices) + ")");
    if (!d_acc && c.n_rows) throw DataError("null accumulator");
    if (plan->chunked) {
      run_chunked(*plan, slice_begin, slice_end, d_acc, accumulate != 0, stream);
      return;
    }
    run_slices(*plan->dp, slice_begin, slice_end, d_acc, accumulate != 0, stream);
  });
}

mtcg_status mtcg_run_slices_out(mtcg_plan* plan, uint64_t slice_begin, uint64_t slice_end, void* d_out,
                                void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan) throw DataError("null plan");
    DevicePlan& dp = *plan->dp;
    const Compiled& c = dp.c;
    if (slice_begin > slice_end || slice_end > c.n_slices)
      throw DataError("slice range outside [0, " + std::to_string(c.n_slices) + ")");
    if (!d_out && c.n_rows && slice_end > slice_begin) throw DataError("null output buffer");
    if (plan->chunked) throw DataError("per-slice outputs of a row-chunked plan are not supported");
    if (!dp.d_stage) dp.d_stage = device_alloc(dp.engine, c.n_rows * c.row_elems * c.elem_bytes);
    run_slices(dp, slice_begin, slice_end, dp.d_stage, false, stream, d_out);
  });
}

mtcg_status mtcg_fold(mtcg_plan* plan, const void* d_parts, uint64_t n_parts, void* d_acc, int accumulate,
                      void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!plan) throw DataError("null plan");
    const Compiled& c = plan->dp->c;
    if (n_parts && (!d_parts || !d_acc)) throw DataError("null buffer");
    const uint64_t rows = plan->chunked ? plan->chunked->rows : c.n_rows;
    fold_slices(plan->dp->engine, c.precision, d_parts, n_parts, rows * c.row_elems, d_acc, accumulate != 0,
                stream);
  });
}

mtcg_status mtcg_fetch(mtcg_plan* plan, const void* d_acc, void* stream, mtcg_result* res,
                       char* err, size_t errlen) {
  NvtxRange nv("mtcg_fetch");
  return guarded(err, errlen, nullptr, [&] {
    if (!plan || !res) throw DataError("null argument");
    if (plan->chunked) {
      fetch_chunked(*plan, d_acc, stream, res);
      return;
    }
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
    if (plan->chunked) {  // over the fetched amplitudes (compensated device reduction)
      const Compiled& w = *plan->chunked->whole;
      std::vector<double> vals(2 * w.n_requests * w.row_elems);
      mtcg_result r{};
      r.values = vals.data();
      r.values_capacity = w.n_requests * w.row_elems;
      fetch_chunked(*plan, d_acc, stream, &r);
      *out = xeb_probs(plan->dp->engine, vals.data(), w.n_requests * w.row_elems, n_qubits, true);
      return;
    }
    *out = xeb_device(*plan->dp, d_acc, n_qubits, stream);
  });
}

mtcg_status mtcg_eval(mtcg_handle* h, const mtcg_problem* p, const mtcg_options* opt,
                      mtcg_result* res, char* err, size_t errlen) {
  NvtxRange nv("mtcg_eval");
  int32_t cap_node = -1;
  mtcg_status st = guarded(err, errlen, &cap_node, [&] {
    if (!h || !res) throw DataError("null argument");
    check_problem_pointers(p);
    const mtcg_options o = effective_options(h, opt ? *opt : default_options());
    const int n_dev = static_cast<int>(h->engines.size());
    const int n_use = o.workers > 0 ? std::min(n_dev, static_cast<int>(o.workers)) : n_dev;
    if (n_use > 1) {
      if (o.row_chunk) throw DataError("row_chunk with several devices is not supported");
      const uint64_t S = p->n_sliced >= 0 && p->n_sliced < 63 ? uint64_t{1} << p->n_sliced : ~uint64_t{0};
      if (S < static_cast<uint64_t>(n_use) && p->n_requests >= static_cast<uint64_t>(n_use))
        eval_multi_rows(h, p, o, n_use, res);  // fewer slices than GPUs: split the requests
      else
        eval_multi(h, p, o, n_use, res);
      return;
    }
    if (o.row_chunk && o.row_chunk < p->n_requests) {
      eval_chunked(h, p, o, res);
      return;
    }
    Compiled c = compile_problem(*p, o, device_cap(h, o), nullptr, index_device(h, *p, o));
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
