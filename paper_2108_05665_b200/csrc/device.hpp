// Device executor for a Compiled schedule (sm_100a).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "planner.hpp"

namespace mtcg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Engine;  // one per handle (device + stream + counters)

struct DevicePlan {
  Compiled c;
  Engine* engine = nullptr;
  void* d_leaves = nullptr;
  void* d_arena = nullptr;
  uint32_t* d_tables = nullptr;
  uint32_t* d_index = nullptr;
  uint32_t* d_row_mult = nullptr;
  double* d_xeb_part = nullptr;         // fused-XEB block partials (device)
  void* d_blob = nullptr;               // one allocation behind the pointers above
  uint64_t blob_bytes = 0;
  // slice parameters in device memory: per-bit projection strides of sliced
  // leaf operands (-1: operand not sliced) and the current {slice, accumulate}
  uint64_t* d_sstr = nullptr;
  uint32_t* d_cur = nullptr;
  std::vector<int64_t> a_str_off, b_str_off;  // per op, into d_sstr
  int64_t lr_str_off = -1;                    // leaf root
  int s_bits = 0;
  // One instantiated CUDA graph of a whole slice's launches per accumulator
  // (slice parameters are read from d_cur, so the graph serves every slice):
  // a slice is one tiny set-slice kernel plus one graph launch.
  struct GraphEntry {
    void* exec = nullptr;   // cudaGraphExec_t
    uint64_t kernels = 0;   // device launches replayed per graph launch
    void* exec_pro = nullptr;  // slice-reuse prologue (invariant ops), once per run
    uint64_t kernels_pro = 0;
  };
  std::map<void*, GraphEntry> graphs;
  // Concurrent capture: independent ops (disjoint subtrees) are issued on
  // several streams joined by per-op events, so the captured slice graph is
  // a DAG and small ops run side by side.
  std::vector<void*> aux_streams;  // cudaStream_t
  std::vector<void*> op_events;    // cudaEvent_t per op
  std::vector<void*> join_events;  // cudaEvent_t per aux stream, + fork
  void* d_stage = nullptr;         // per-slice output staging (mtcg_run_slices_out)
  ~DevicePlan();
};

Engine* engine_create(int device);
void engine_destroy(Engine* e);
uint64_t engine_launches(const Engine* e);
uint64_t engine_arena_bytes(const Engine* e);  // cached intermediate arena
void* engine_stream(Engine* e);

std::unique_ptr<DevicePlan> upload_plan(Engine* e, Compiled&& c);

// Runs slices [s0, s1) accumulating into d_acc (rows x row_elems elements of
// the plan precision). accumulate=false: the first slice overwrites.
// d_out_slices != null: no fold — each slice's root values (d_acc is then
// staging) are copied to d_out_slices + (s - s0) * rows * row_elems.
void run_slices(DevicePlan& dp, uint64_t s0, uint64_t s1, void* d_acc,
                bool accumulate, void* stream, void* d_out_slices = nullptr);

// One slice of a row-chunked plan (Compiled::row_prologue): the request-
// independent prologue when with_prologue (the slice's first chunk), then the
// chunk's own ops; accumulates into d_acc like run_slices.
void run_slice_chunk(DevicePlan& dp, uint64_t s, void* d_acc, bool accumulate, bool with_prologue,
                     void* stream);
// Sizes the handle's shared arena for this plan (all chunk plans of one
// evaluation share it: resolve every plan before the first run).
void ensure_arena(DevicePlan& dp);

// acc = (accumulate ? acc : parts[0]) + parts[1] + ... in part order (the
// reference's slice fold); parts: n_parts x n_elem complex of `precision`.
void fold_slices(Engine* e, int precision, const void* d_parts, uint64_t n_parts, uint64_t n_elem,
                 void* d_acc, bool accumulate, void* stream);
int engine_device(const Engine* e);

// Same as run_slices for one slice, with an event pair around each op;
// op_ms[i] receives op i's device time (ops with batch 0 get 0).
void time_ops(DevicePlan& dp, uint64_t slice, void* d_acc, bool accumulate, void* stream,
              float* op_ms);

// Fused |amp|^2 -> linear XEB over all requests (row multiplicities).
double xeb_device(DevicePlan& dp, const void* d_acc, int n_qubits, void* stream);

// linear_xeb over host probabilities / amplitudes (device reduction).
double xeb_probs(Engine* e, const double* probs, uint64_t count, int n_qubits,
                 bool amplitudes);

// Device buffer helpers for the one-shot path.
void* device_alloc(Engine* e, uint64_t bytes);
void device_free(Engine* e, void* p);
void copy_to_host(Engine* e, void* dst, const void* src, uint64_t bytes, void* stream);

}  // namespace mtcg
