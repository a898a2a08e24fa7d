// Host-side compilation of one multi-tensor evaluation into a static device
// schedule. Pure C++ (no CUDA): validation, tuple index, per-node shapes and
// layouts, the batched contraction op list, the static HBM arena plan and the
// exact operation counts. Citations are to /root/reference/proj.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mtcg.h"

namespace mtcg {

// Exceptions mirror the reference's classes (errors.hpp:26-55); the C ABI
// maps them to mtcg_status codes.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// ParseError (errors.hpp:26-36): "line N: what" when the line is known
struct ParseError : std::runtime_error {
  ParseError(const std::string& what, uint64_t line)
      : std::runtime_error(line ? "line " + std::to_string(line) + ": " + what : what) {}
};
struct MemoryCapError : std::runtime_error {
  MemoryCapError(const std::string& w, int node) : std::runtime_error(w), node(node) {}
  int node;
};
struct InternalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Offset table for one bit-permuted index space: offset(x) = lo[x & lo_mask]
// + hi[x >> lo_bits], element units. Bits of x map to legs; each leg
// contributes bit * stride (bond dimension 2 everywhere).
struct SplitTable {
  int bits = 0;
  int lo_bits = 0;
  std::vector<uint32_t> lo, hi;
  uint64_t dev_off = 0;  // word offset of lo in the plan's table blob
  void build(const std::vector<uint64_t>& strides);  // strides[bit], LSB first
};

// One batched pairwise contraction: node `node` for every distinct rank of it
// (plan.hpp:103-111 `distinct`), out[b] = Σ_c A[ia[b]] B[ib[b]].
struct Op {
  int node = -1;
  int child_a = -1, child_b = -1;  // plan nodes feeding the A (m) / B (n) side
  bool a_is_left = true;
  uint32_t nb = 0;                 // batch = distinct[node]
  int fa = 0, fb = 0, kc = 0;      // log2 M, N, K
  // operand sources: table base (arena offset or leaf blob offset, elements)
  bool a_leaf = false, b_leaf = false;
  uint64_t a_base = 0, b_base = 0;          // element offsets
  uint64_t a_item = 0, b_item = 0;          // elements per stored entry
  std::vector<uint32_t> ia, ib;             // per item entry index
  uint64_t ia_off = 0, ib_off = 0;          // word offsets in the index blob
  SplitTable tam, tak, tbn, tbk, tom, ton;  // A(m), A(k), B(n), B(k), out(m), out(n)
  // slice projection of leaf operands: element offset added per set bit of
  // the slice index (bit j = sliced leg n_sliced-1-j, multieval.cpp:322-329)
  std::vector<uint64_t> a_slice_stride, b_slice_stride;
  int slice_slot = -1;             // index into the per-slice offset array
  // output
  bool root = false;
  uint64_t out_base = 0;           // arena element offset (non-root)
  uint64_t out_item = 0;           // elements per output entry
  bool store_n_fast = true;        // epilogue lane order
  std::vector<uint32_t> out_rows;  // root: item -> accumulator row
  uint64_t out_rows_off = 0;
  // grouped rows kernel: items sharing one A entry, CSR by A entry
  std::vector<uint32_t> grp_items;  // item ids ordered by A entry
  std::vector<uint32_t> grp_start;  // n_groups + 1 offsets into grp_items
  uint32_t grp_max = 0;             // largest group
  uint64_t grp_items_off = 0, grp_start_off = 0;
  int config = 0;                  // kernel tile configuration
  uint64_t a_entries = 0;          // tensor-core path: entries in A's table
  uint64_t scratch_off = 0;        // tensor-core path: arena scratch (elements)
  uint64_t scratch_elems = 0;
  // tensor-core split-integer path, slice reuse: the A table is slice-
  // invariant and its rows are quantized once by the prologue (K > 32
  // complex); the row exponents then live at row_exp_off (never released)
  bool a_prequant = false;
  uint64_t row_exp_off = 0;
  bool a_kcontig = false;          // A rows are K-contiguous (tak(k) == k)
  bool b_kcontig = false;          // B rows are K-contiguous (tbk(k) == k)
  bool o_ncontig = false;          // output n index is contiguous (ton(n) == n)
  bool o_mcontig = false;          // output m bit 0 has stride 1
  // ops this op must wait for when independent ops run concurrently: the
  // producers of its operands and every earlier op that used the arena
  // ranges it writes (the first-fit arena reuses memory in schedule order)
  std::vector<int> deps;
  // exact algorithmic counts per slice (tensor.cpp:132-148)
  uint64_t mults = 0, adds = 0, rw = 0;
  // fused operand chain (Compiled::chains) this op belongs to, -1: none. The
  // chain's last op launches the fused kernel; the others launch nothing.
  int chain = -1;
  bool chain_tail = false;
  // Tensor-core gather mode (small M, shared B): items grouped by B entry;
  // each 128-row tile stacks 128 / M items of one group (TMA gathers their A
  // entries). ga_groups: B entry per group; ga_tiles: per tile the group and
  // its 128 / M items (~0u pads a group's last tile).
  std::vector<uint32_t> ga_groups, ga_tiles;
  uint64_t ga_groups_off = 0, ga_tiles_off = 0;
};

// A run of consecutive skinny ops along one operand chain (each op's A is the
// previous op's output, items map one-to-one) evaluated by one kernel: a block
// of the first op's A is loaded into shared memory once, every step contracts
// it in place with its small B in the reference's order, and only the last
// op's table is written. Intermediate tables never reach HBM.
//   The legs the chain touches (A legs some step closes, legs a B opens) live
//   in shared-memory positions [0, 2^q) per untouched-leg combination u;
//   closed legs free their positions for the legs opened after them.
constexpr int kMaxChainSteps = 8;
constexpr int kMaxChainTable = 256 + 8 + 8 + 64;  // words of one step's tables (q <= 8, K, G <= 8)
struct ChainStep {
  int op = -1;                 // op index (B operand, ib, slice strides)
  int kc = 0;
  int g_bits = 0;              // legs the step's B opens
  int f_bits = 0;              // touched legs the step keeps
  uint32_t n_out = 0;          // combos of the active touched legs after the step
  // in_base[2^f] | out_g[2^g] | in_c[2^kc] | boff[2^(kc + g)]: row positions
  // of the kept-leg combination f (the same in the input and output rows),
  // of the opened-leg combination g, of the closed combination c, and the B
  // tile's element offsets (c * 2^g + g) in the B entry
  std::vector<uint32_t> tbl;
  uint64_t tbl_off = 0;        // word offset in the index blob
};
struct Chain {
  int head = -1, tail = -1;    // op indices, consecutive
  int q = 0;                   // log2 positions per inner combination
  int u_bits = 0;              // untouched legs
  int u_inner_bits = 0;        // of which inside one block (the rest index blocks)
  SplitTable tu_in, tu_out;    // outer combination -> element offset in the head's A / tail's output
  // block load / store maps: the block's elements are indexed by bits over
  // (inner untouched legs + touched legs) in address order; per bit, the
  // (shared-memory position, element offset) it adds
  std::vector<uint32_t> qin, qout;
  uint64_t qin_off = 0, qout_off = 0;
  uint64_t out_base = 0;       // tail output: its own arena region (never reused)
  std::vector<ChainStep> steps;
  // per final item: the head's A entry, then each step's B entry ([steps+1][nb])
  std::vector<uint32_t> entries;
  uint64_t entries_off = 0;
};

// A plan whose root is a leaf (single-slot network): copy/accumulate the
// projected leaf tensors into the accumulator.
struct LeafRoot {
  int slot = -1;
  std::vector<uint32_t> row_value;   // row -> value index
  uint64_t item = 0;                 // stored elements per value
  SplitTable tout;                   // out index -> offset in the value
  std::vector<uint64_t> slice_stride;
  uint64_t rows_off = 0;
};

struct Compiled {
  // inputs (copied)
  int precision = MTCG_C64;
  int n_nodes = 0, n_slots = 0, root = -1;
  std::vector<uint32_t> sliced;
  uint64_t n_slices = 1;
  uint64_t n_requests = 0, n_rows = 0;
  uint64_t row_elems = 1;
  std::vector<uint32_t> out_legs;      // legs of every request tensor
  std::vector<uint64_t> row_of_request;
  std::vector<uint32_t> row_mult;      // requests per row (XEB weights)
  // leaves: all value sets, stored as given (incl. sliced legs)
  std::vector<uint64_t> slot_base;     // element offset of slot j's values
  std::vector<uint64_t> slot_item;     // elements per value tensor
  uint64_t leaf_elems = 0;
  std::vector<double> leaf_values;     // complex128 interleaved (host copy)
  // schedule
  std::vector<Op> ops;
  std::vector<Chain> chains;           // fused operand chains (MTCG_NO_CHAIN=1: none)
  bool has_leaf_root = false;
  LeafRoot leaf_root;
  std::vector<uint32_t> table_blob;    // all SplitTables
  std::vector<uint32_t> index_blob;    // ia/ib/out_rows arrays
  uint64_t arena_elems = 0;            // per-slice intermediate arena
  int elem_bytes = 8;
  // counts (whole evaluation)
  std::vector<uint64_t> node_contractions;
  uint64_t mults = 0, adds = 0, rw = 0, contractions = 0;
  int n_slice_slots = 0;               // ops/leaf root needing slice offsets

  uint64_t private_elems = 0;          // of arena_elems: never-reused small tables
  // MTCG_FLAG_SLICE_REUSE: ops[0, n_prologue_ops) are the slice-invariant
  // nodes, run once per run range; their tables feeding slice-dependent
  // parents stay resident in the arena across slices
  size_t n_prologue_ops = 0;
  // row-chunked evaluation: the prologue is the request-independent part,
  // run once per slice (by the first chunk) rather than once per run range
  bool row_prologue = false;
  uint64_t executed_contractions = 0;  // per run range of S slices: see slice_contractions()
  uint64_t arena_bytes() const { return arena_elems * elem_bytes; }
  uint64_t resident_bytes() const {
    return leaf_elems * elem_bytes + 4 * (table_blob.size() + index_blob.size());
  }
};

// build_tuple_index (plan.cpp:292-333) output. Rows are the distinct request
// tuples in lexicographic order; a node's dense ranks order its distinct
// restrictions by (rank_left, rank_right).
struct TupleIndex {
  uint64_t rows = 0;
  std::vector<uint32_t> row_tuple_first;  // request index representing row
  std::vector<uint64_t> row_of_request;
  // rank of every row per node (host builder: every node; device builder:
  // the root only, in root_rank)
  std::vector<uint32_t*> rank;                    // [node] -> [row]
  std::vector<uint32_t> root_rank;
  std::vector<std::vector<uint32_t>> rank_value;  // leaves: rank -> value index
  std::vector<std::vector<uint32_t>> pair_l, pair_r;  // internal: rank -> child ranks
  std::vector<uint32_t> distinct;
};

// Bit-packed request tuples for the device tuple index: the informative
// slots (more than one value), ascending, each ceil(log2 n_values) bits,
// concatenated first-most-significant into 64-bit words (lexicographic
// tuple order = numeric order of the word sequence).
struct TupleWords {
  std::vector<int> informative;         // slot of each informative column
  std::vector<uint8_t> bits;            // per column
  std::vector<int> word, shift;         // per column: word index, bit offset in it
  std::vector<std::pair<int, int>> span;  // per word: columns [c0, c1)
  std::vector<int> word_bits;           // per word: bits used
};
TupleWords tuple_word_layout(const mtcg_problem& p);

// Device builder (index.cu): radix sorts on GPU `device`, same TupleIndex as
// the host builder. `postorder` lists children before parents; `words` holds
// the packed tuples word-major ([word][request], layout `lay`). Returns false
// when it does not apply (no requests, no room for its scratch).
bool build_tuple_index_device(const mtcg_problem& p, const std::vector<int>& postorder, const TupleWords& lay,
                              const std::vector<uint64_t>& words, int device, TupleIndex& ti);

// The tuple index alone (index_plan's checks, then the device builder on
// `device` >= 0 or the host builder): diagnostics / tests.
TupleIndex tuple_index(const mtcg_problem& p, int device);

// Validates `p` with the reference's checks and messages, builds the tuple
// index and the schedule. cap_bytes = 0: no cap. Throws DataError /
// MemoryCapError.
// request_dependent_slots (row-chunked evaluation): the slots whose value
// varies over the requests of the WHOLE problem (this `p` holds one chunk of
// them). Nodes over request-independent slots only form a prologue, scheduled
// first in a canonical order and run once per slice for all chunks; the
// tables they hand to request-dependent parents stay resident at offsets that
// are the same in every chunk's schedule.
Compiled compile_problem(const mtcg_problem& p, const mtcg_options& opt,
                         uint64_t cap_bytes,
                         const std::vector<char>* request_dependent_slots = nullptr,
                         int index_device = -1);
// index_device >= 0: build the tuple index on that GPU (build_tuple_index_device)

}  // namespace mtcg
