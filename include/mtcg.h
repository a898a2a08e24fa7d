/*
 * mtcg.h — C ABI of the B200-native multi-tensor contraction engine.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2108.05665 `mtc`):
 *
 *   mtcg_eval          replaces  EvalResult eval_all(const Plan&,
 *                                  const NetworkDiagram&, const AssignmentSet&,
 *                                  const EvalOptions&)      multieval.hpp:62-63
 *                          and   EvalResult eval_sliced(...) multieval.hpp:69-70
 *                     (the CLI's choice `plan.sliced.empty() ? eval_all :
 *                      eval_sliced` is MTCG_EVAL_AUTO, tools/main.cpp:159-160)
 *   mtcg_linear_xeb    replaces  double linear_xeb(int n,
 *                                  const std::vector<double>& probs)  xeb.hpp:38
 *   mtcg_linear_xeb_amplitudes
 *                      replaces  linear_xeb(n, probs_from_amplitudes(amps))
 *                                                            xeb.hpp:38,42-43
 *
 * (paths relative to /root/reference/proj/include/mtc and proj/tools.)
 *
 * The staged API (mtcg_compile / mtcg_run / mtcg_fetch / mtcg_xeb_device)
 * splits mtcg_eval so callers can keep the compiled problem resident in HBM,
 * shard slice ranges over one process per GPU and combine the per-rank
 * partial amplitudes with one NCCL collective.
 *
 * Conventions
 *  - No function throws. Every call returns an mtcg_status; on failure a
 *    NUL-terminated message is written to err[0..errlen) when err != NULL.
 *    Status codes mirror the reference's exception classes:
 *      MTCG_ERR_DATA        mtc::DataError     (CLI exit 2)
 *      MTCG_ERR_MEMORY_CAP  mtc::MemoryCapError (CLI exit 3); the offending
 *                           plan node is returned in mtcg_result.cap_node /
 *                           the cap_node out-parameter
 *      MTCG_ERR_INTERNAL    std::logic_error    (CLI exit 1)
 *  - All input arrays are borrowed for the duration of the call and copied
 *    to the device; the caller owns every output buffer. No device pointer
 *    owned by the library escapes; device pointers passed IN (mtcg_run's
 *    accumulator) belong to the caller.
 *  - Calls on one handle are not reentrant; separate handles are
 *    independent.
 *  - Complex numbers cross the boundary as interleaved (re, im) doubles, the
 *    layout of std::complex<double> (tensor.hpp:26).
 */
#ifndef MTCG_H
#define MTCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTCG_ABI_VERSION 2

typedef enum mtcg_status {
  MTCG_OK = 0,
  MTCG_ERR_INTERNAL = 1,
  MTCG_ERR_DATA = 2,
  MTCG_ERR_MEMORY_CAP = 3,
  MTCG_ERR_CUDA = 5,
  MTCG_ERR_ARGUMENT = 6,
  MTCG_ERR_NCCL = 7,
  MTCG_ERR_PARSE = 8
} mtcg_status;

/* Arithmetic of the device path.
 *  MTCG_C64   complex64 (fp32 pairs) — the production mode; amplitudes agree
 *             with the complex128 reference within 1e-4 relative.
 *  MTCG_C128  complex128 with every multiply/add individually rounded
 *             (no FMA contraction) and closed legs summed in the reference's
 *             ascending-id row-major order (tensor.cpp:186-245): per-slice
 *             values are bit-identical to the reference, and so is the
 *             slice fold on one device. */
typedef enum mtcg_precision { MTCG_C64 = 0, MTCG_C128 = 1 } mtcg_precision;

typedef enum mtcg_eval_mode {
  MTCG_EVAL_AUTO = 0,   /* sliced plan ? eval_sliced : eval_all */
  MTCG_EVAL_ALL = 1,    /* eval_all: rejects sliced plans (DataError) */
  MTCG_EVAL_SLICED = 2  /* eval_sliced: rejects unsliced plans (DataError) */
} mtcg_eval_mode;

/* The engine's inputs, as POD arrays. Field groups mirror the reference
 * types the engine reads; nothing else of them is needed. */
typedef struct mtcg_problem {
  /* Plan (plan.hpp:33-45): binary tree over slots + sliced legs. Leaves have
   * slot >= 0 and left = right = -1; internal nodes have slot = -1. */
  int32_t n_nodes;
  const int32_t* node_left;
  const int32_t* node_right;
  const int32_t* node_slot;
  int32_t root;
  int32_t n_sliced;
  const uint32_t* sliced; /* in plan order: slice enumeration is mixed radix
                             with the LAST listed leg fastest
                             (multieval.cpp:322-329) */
  /* NetworkDiagram (diagram.hpp:32-45): legs [0, n_closed) are closed, legs
   * [n_closed, n_legs) open (the open leg of qubit q is n_closed + q). */
  uint32_t n_legs;
  uint32_t n_closed;
  const uint32_t* leg_dims; /* [n_legs]; this engine supports dim 2 */
  int32_t n_slots;
  /* AssignmentSet (diagram.hpp:61-68). Slot j has slot_n_values[j] value
   * tensors sharing one leg list slot_legs[slot_leg_begin[j] ..
   * slot_leg_begin[j+1]) (listed order = row-major order). `values` holds
   * all of them, slot-major then value-major, each row-major. */
  const int32_t* slot_n_values;   /* [n_slots] */
  const int32_t* slot_leg_begin;  /* [n_slots + 1] */
  const uint32_t* slot_legs;
  const double* values;           /* complex128 interleaved */
  uint64_t n_requests;
  const uint32_t* tuples;         /* [n_requests][n_slots] value indices */
  int32_t n_batch_legs;           /* '*' legs kept open, ascending */
  const uint32_t* batch_legs;
} mtcg_problem;

typedef struct mtcg_options {
  int32_t eval_mode;          /* mtcg_eval_mode */
  int32_t precision;          /* mtcg_precision */
  uint64_t memory_cap_bytes;  /* device arena cap; 0 = the handle's cap */
  int32_t workers;            /* EvalOptions.workers: on a multi-device
                                 handle, the GPUs mtcg_eval uses (0 = all);
                                 results never depend on it,
                                 multieval.hpp:66-68 */
  int32_t flags;              /* MTCG_FLAG_* */
  uint64_t row_chunk;         /* memo streaming (the reference's bounded
                                 left/right caches, multieval.cpp:213-274):
                                 mtcg_eval takes the requests, in
                                 lexicographic tuple order, in chunks of this
                                 many; the request-independent subtrees run
                                 once per slice for all chunks and the memo
                                 tables hold one chunk's distinct tuples.
                                 0 = all requests at once */
} mtcg_options;

/* mtcg_options.flags */
#define MTCG_FLAG_NO_TENSOR_CORES 1 /* dense ops on the CUDA-core kernels */
#define MTCG_FLAG_SLICE_REUSE 2     /* evaluate slice-invariant subtrees (no
                                       sliced leg among their leaves) once per
                                       run instead of once per slice; values
                                       are unchanged, counters stay the
                                       reference's (per-slice) counts. Ignored
                                       under a memory cap. */
#define MTCG_FLAG_HOST_INDEX 4      /* build the tuple index (plan.cpp:292-333)
                                       on the host CPU */
#define MTCG_FLAG_DEVICE_INDEX 8    /* build it with radix sorts on the
                                       handle's GPU (same rows, ranks and
                                       pairs). Neither flag: the GPU from
                                       2^15 requests up, else the host.
                                       mtcg_emulate always uses the host. */

/* eval outputs. `values` is a caller buffer of values_capacity complex
 * elements receiving, request-major, each request's tensor (order-0, or
 * order-w over the batch legs ascending — tools/main.cpp:167-178). */
typedef struct mtcg_result {
  double* values;
  uint64_t values_capacity;      /* complex elements available */
  uint64_t* node_contractions;   /* [n_nodes] or NULL: contractions performed
                                    per plan node, summed over slices */
  uint64_t mults, adds, rw;      /* OpCounters (tensor.hpp:36-51), exact */
  uint64_t hbm_peak_bytes;       /* device arena high-water mark (the GPU
                                    schedule's; not the reference's
                                    Session peak) */
  int32_t cap_node;              /* node of a MEMORY_CAP failure, else -1 */
  int32_t n_out_legs;            /* legs of each value tensor */
  uint32_t out_legs[64];
} mtcg_result;

typedef struct mtcg_handle mtcg_handle;
typedef struct mtcg_plan mtcg_plan;

/* Static facts about a compiled problem. */
typedef struct mtcg_plan_info {
  uint64_t n_requests;
  uint64_t n_rows;              /* distinct request tuples */
  uint64_t row_elems;           /* 2^w: elements per request tensor */
  uint64_t n_slices;            /* Π dims(sliced legs); 1 when unsliced */
  uint64_t mults, adds, rw;     /* per full evaluation (all slices) */
  uint64_t contractions;        /* Σ node contractions, all slices */
  uint64_t hbm_arena_bytes;     /* device bytes of the per-slice schedule */
  uint64_t hbm_resident_bytes;  /* leaves + index arrays kept on device */
  int32_t precision;
  int32_t n_kernels_per_slice;  /* device launches per slice */
  uint64_t prologue_ops;        /* MTCG_FLAG_SLICE_REUSE: slice-invariant ops
                                   run once per run range (0 without) */
  uint64_t executed_contractions; /* contractions one run over all slices
                                     executes (= contractions without reuse) */
  uint64_t fused_chains;        /* runs of skinny ops evaluated by one kernel */
  uint64_t fused_ops;           /* ops inside those runs */
} mtcg_plan_info;

int mtcg_version(void);

/* Creates an engine bound to CUDA device `device`. hbm_cap_bytes caps the
 * device arena of every compiled plan (0 = free device memory). */
mtcg_status mtcg_create(int device, uint64_t hbm_cap_bytes,
                        mtcg_handle** out, char* err, size_t errlen);
/* An engine over several GPUs of one node: devices[0] is the
 * root, which holds results and runs the XEB. mtcg_eval distributes the
 * slices over the first min(options.workers, n_devices) devices
 * (options.workers = 0: all) — the GPU analogue of EvalOptions.workers,
 * multieval.hpp:26-29 — in contiguous blocks, gathers every slice's root
 * values to the root over NVLink (NCCL point-to-point on a communicator
 * created here) and folds them there in slice order: results are
 * bit-identical for every device count, like the reference's for every
 * worker count (multieval.hpp:64-68). A device may repeat (ranks sharing one
 * GPU: the same arithmetic, device-to-device copies instead of NCCL). The
 * staged API below runs on the root device. */
mtcg_status mtcg_create_multi(const int* devices, int n_devices,
                              uint64_t hbm_cap_bytes_per_gpu, mtcg_handle** out,
                              char* err, size_t errlen);
int32_t mtcg_device_count(const mtcg_handle* h);
int32_t mtcg_visible_devices(void);  /* CUDA devices this process sees */
void mtcg_destroy(mtcg_handle* h);

/* One-shot evaluation: compile + run all slices + fetch. The drop-in for
 * eval_all / eval_sliced. */
mtcg_status mtcg_eval(mtcg_handle* h, const mtcg_problem* p,
                      const mtcg_options* opt, mtcg_result* res, char* err,
                      size_t errlen);

/* linear_xeb (xeb.cpp:43-50): (2^n / k) * Σ probs − 1, compensated sum;
 * DataError on empty input, n outside [0, 1022] or a negative probability. */
mtcg_status mtcg_linear_xeb(mtcg_handle* h, int n_qubits, const double* probs,
                            uint64_t count, double* out, char* err,
                            size_t errlen);
/* The same over |amp|^2 of complex amplitudes (probs_from_amplitudes,
 * xeb.cpp:67-73), fused on the device. */
mtcg_status mtcg_linear_xeb_amplitudes(mtcg_handle* h, int n_qubits,
                                       const double* amps, uint64_t count,
                                       double* out, char* err, size_t errlen);

/* ---- staged API -------------------------------------------------------- */

/* Validates the problem exactly as eval_all/eval_sliced do, builds the
 * tuple index (plan.cpp:292-333) and the device schedule, and uploads the
 * leaves. The device arena is sized here (MEMORY_CAP → cap_node). */
mtcg_status mtcg_compile(mtcg_handle* h, const mtcg_problem* p,
                         const mtcg_options* opt, mtcg_plan** out,
                         int32_t* cap_node, char* err, size_t errlen);
void mtcg_plan_destroy(mtcg_plan* plan);
mtcg_status mtcg_plan_get_info(const mtcg_plan* plan, mtcg_plan_info* info);

/* Runs slices [slice_begin, slice_end) on `stream` (a cudaStream_t, NULL =
 * the handle's stream) and accumulates the root values, by row, into the
 * caller's device buffer `d_acc` (n_rows * row_elems complex of the plan's
 * precision: float2 for C64, double2 for C128). accumulate = 0 overwrites
 * with the first slice of the range. Slices are folded in increasing slice
 * index (multieval.cpp:498-513). Asynchronous with respect to the host. */
mtcg_status mtcg_run(mtcg_plan* plan, uint64_t slice_begin,
                     uint64_t slice_end, void* d_acc, int accumulate,
                     void* stream, char* err, size_t errlen);

/* Per-slice values instead of a fold: runs slices [slice_begin, slice_end)
 * and writes slice s's root values (n_rows * row_elems complex, plan
 * precision) to d_out + (s - slice_begin) * n_rows * row_elems — the
 * per-rank half of a deterministic multi-GPU evaluation (gather, then
 * mtcg_fold on one rank). Asynchronous with respect to the host. */
mtcg_status mtcg_run_slices_out(mtcg_plan* plan, uint64_t slice_begin,
                                uint64_t slice_end, void* d_out, void* stream,
                                char* err, size_t errlen);
/* d_acc = (accumulate ? d_acc : parts[0]) + parts[1] + ... + parts[n-1],
 * one rounded add per part in order: the reference's slice fold
 * (multieval.cpp:498-513). parts: n_parts consecutive n_rows * row_elems
 * blocks on the plan's device. */
mtcg_status mtcg_fold(mtcg_plan* plan, const void* d_parts, uint64_t n_parts,
                      void* d_acc, int accumulate, void* stream, char* err,
                      size_t errlen);

/* Copies a device accumulator back and fans rows out to requests
 * (multieval.cpp:374-380), filling res->values / out_legs / counters for the
 * slices [0, n_slices) (node_contractions, mults, adds, rw are the full
 * evaluation's). Synchronises `stream`. */
mtcg_status mtcg_fetch(mtcg_plan* plan, const void* d_acc, void* stream,
                       mtcg_result* res, char* err, size_t errlen);

/* Fused |amp|^2 -> linear XEB over every request (duplicates included, each
 * batch element an amplitude, as the CLI's TSV feeds `mtc xeb`) straight from
 * a device accumulator. Synchronises `stream`. */
mtcg_status mtcg_xeb_device(mtcg_plan* plan, const void* d_acc,
                            int n_qubits, void* stream, double* out,
                            char* err, size_t errlen);

/* Shape-only replay (the reference's `emulate`, multieval.hpp:72-75): runs
 * every validation of mtcg_eval and the full schedule construction on the
 * host — no device needed — and reports the exact counts (info->mults, adds,
 * rw, contractions; node_contractions [n_nodes] or NULL) and the device
 * arena the evaluation would use. cap_bytes = 0: no cap. */
mtcg_status mtcg_emulate(const mtcg_problem* p, const mtcg_options* opt,
                         uint64_t cap_bytes, mtcg_plan_info* info,
                         uint64_t* node_contractions, int32_t* cap_node,
                         char* err, size_t errlen);

/* Tuple index check (build_tuple_index, plan.cpp:292-333): builds the index
 * of `p` with the host builder and on the handle's GPU, compares rows,
 * row_of_request, the row representatives, every node's distinct count,
 * (rank_left, rank_right) pairs, leaf value lists and the root's ranks;
 * *equal = 1 when all match. *rows = the distinct request tuples, host_ms /
 * device_ms = the two builders' wall times (either pointer may be NULL). */
mtcg_status mtcg_tuple_index_check(mtcg_handle* h, const mtcg_problem* p,
                                   int32_t* equal, uint64_t* rows,
                                   double* host_ms, double* device_ms,
                                   char* err, size_t errlen);

/* ---- paper-scale request ingestion (host, multithreaded) -------------------
 * read_samples (formats.cpp:42-69): parses a samples text of `len` bytes —
 * one string over {0,1,*} per line, '#' comments, blank lines skipped, one
 * length and one '*' pattern — into `out` [n_rows][n_qubits] canonical
 * characters (qubit 0 first; bit_order 1 = the text has qubit 0 last).
 * out_capacity >= len always suffices. MTCG_ERR_PARSE carries the
 * reference's message ("line N: ..."). */
mtcg_status mtcg_read_samples(const char* text, uint64_t len, int32_t bit_order,
                              char* out, uint64_t out_capacity,
                              uint64_t* n_rows, int32_t* n_qubits,
                              char* err, size_t errlen);

/* build_assignments' ranking (diagram.cpp:229-297): slot j's fixed bits are
 * the sample characters at qubits slot_qubits[slot_qubit_begin[j] ..
 * slot_qubit_begin[j+1]) (its open legs in slot_open_legs order) that are not
 * batch positions (the '*' columns of sample 0; every sample must agree).
 * Outputs: tuples [n_rows][n_slots] (mtcg_problem.tuples), slot_n_values
 * [n_slots], and the distinct fixed-bit tuples of every slot ascending —
 * packed with the first fixed bit most significant — in value_keys
 * [value_key_begin[j] .. value_key_begin[j+1]) (value_key_begin [n_slots+1];
 * a slot without fixed bits has the one key 0: its unprojected tensor).
 * keys_capacity >= n_slots * min(n_rows, 2^max fixed bits) suffices. The
 * value tensors are the slot tensors projected on those bits (project_leg,
 * tensor.cpp:255-282). */
mtcg_status mtcg_assign(const char* samples, uint64_t n_rows, int32_t n_qubits,
                        int32_t n_slots, const int32_t* slot_qubit_begin,
                        const int32_t* slot_qubits, uint32_t* tuples,
                        int32_t* slot_n_values, uint64_t* value_key_begin,
                        uint32_t* value_keys, uint64_t keys_capacity,
                        char* err, size_t errlen);

/* Amplitude TSV (format_amplitude_row, formats.cpp:78-83): one row
 * "bits<TAB>%.16e<TAB>%.16e" per request and batch value, '*' positions
 * expanded in row-major order of the batch legs (tools/main.cpp:161-179);
 * values [n_rows][2^w] complex doubles (mtcg_result.values). Writes `path`;
 * *written = bytes. */
mtcg_status mtcg_write_amplitudes(const char* path, const char* samples,
                                  uint64_t n_rows, int32_t n_qubits,
                                  int32_t bit_order, const double* values,
                                  int32_t w, uint64_t* written, char* err,
                                  size_t errlen);

/* Per-op introspection of a compiled schedule (one op = one batched launch
 * per slice). */
typedef struct mtcg_op_info {
  int32_t node;          /* plan node */
  int32_t kernel;        /* tile configuration (0 = per-element kernel) */
  int32_t fa, fb, kc;    /* log2 of M, N, K */
  uint32_t batch;        /* distinct evaluations of the node per slice */
  uint64_t mults;        /* algorithmic complex MACs per slice */
  uint64_t bytes;        /* algorithmic HBM bytes per slice: |A|+|B|+|out|
                            per item x element size (predicted_cost rw) */
  uint64_t compulsory_bytes; /* bytes this launch cannot avoid: every distinct
                            A and B entry read once (slice-projected leaves at
                            their projected size) + every output written once;
                            fused-chain members count only what reaches HBM */
} mtcg_op_info;
int32_t mtcg_plan_op_count(const mtcg_plan* plan);
mtcg_status mtcg_plan_op_info(const mtcg_plan* plan, int32_t i, mtcg_op_info* info);

/* Runs slice `slice` once with a CUDA event pair around every op launch
 * (on `stream`) and writes each op's device time in milliseconds to
 * op_ms[mtcg_plan_op_count]. Accumulates into d_acc like mtcg_run. */
mtcg_status mtcg_time_ops(mtcg_plan* plan, uint64_t slice, void* d_acc,
                          int accumulate, void* stream, float* op_ms,
                          char* err, size_t errlen);

/* Count of device kernel launches issued by this process through the
 * library since mtcg_create (evidence for the bench's gpu_launches). */
uint64_t mtcg_launch_count(const mtcg_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* MTCG_H */
