// Host program compiler: turns a symbolic Plan + slice set into a DAG of
// kernel launches with a static HBM arena (offsets only; pointers are bound
// per device by the runtime).
#pragma once
#include <cstdint>
#include <vector>

#include "plan.hpp"
#include "program.h"

namespace tc {

enum NodeClass : int8_t { NC_LEAF = 0, NC_TINY = 1, NC_STREAM = 2, NC_GEMM = 3, NC_GENERIC = 4, NC_ALIAS = 5 };

// Where an operand lives at run time.
enum LocKind : int8_t { LOC_LEAF = 0, LOC_SLICED = 1, LOC_ARENA = 2, LOC_SMEM = 3 };
struct Loc {
  LocKind kind;
  int64_t off;  // doubles (LEAF: into leaf values, SLICED: into sliced buffer) or bytes (ARENA)
};

enum StepKind : int8_t {
  ST_SELECT, ST_TINY, ST_STREAM, ST_GEMM, ST_GENERIC, ST_ROOTCOPY, ST_ETA, ST_GEMM_REDUCE
};

struct Step {
  StepKind kind;
  int slot = -1;  // node for STREAM/GEMM/GENERIC
  bool inv = false;  // slice-invariant: runs once per pass (prologue), not per slice
  bool blk = false;  // depends on no index but the fastest sliced one's predecessors: once per block
  int cat() const { return inv ? 0 : blk ? 1 : 2; }  // 0 prologue, 1 block, 2 per slice
  std::vector<int> deps;
  // kernel parameters with pointer fields holding Loc-encoded placeholders
  StreamParams sp{};
  GemmParams gp{};
  GenericParams np{};
  int32_t ns = 0, nf = 0;          // stream template selector
  int32_t bm = 6, bn = 6;          // GEMM tile bits (template selector)
  Loc la{}, lb{}, lc{}, lws{};     // operand/output/workspace locations
  int64_t la_bytes = 0, lb_bytes = 0, lc_bytes = 0;  // their extents
  int64_t gdig_off = 0;            // generic digits offset (in GDigit units)
  int64_t work = 0;                // elements (for launch sizing)
  double alg_bytes = 0, alg_flops = 0;  // algorithmic traffic / flops of the node(s)
};

struct Program {
  int64_t R = 1;                 // result entries
  int64_t num_slices = 1;
  std::vector<int> chosen;       // sliced index ids, pick order
  std::vector<int64_t> chosen_dim;
  std::vector<int8_t> cls;       // per slot
  std::vector<std::vector<int>> layout;  // per slot, LSB-first index ids (effective)
  std::vector<Loc> loc;          // per slot
  // sliced leaves
  int64_t sliced_doubles = 0;
  std::vector<SelEntry> sel_ent;
  std::vector<SelTerm> sel_terms;
  // tiny forest
  std::vector<TinyNode> tiny_nodes;  // ga/gb/gout hold Loc-encoded placeholders
  std::vector<Loc> tiny_ga, tiny_gb, tiny_gout;
  std::vector<TinyDigit> tiny_digits;
  std::vector<TinyGroup> tiny_groups;
  int32_t tiny_smem_doubles = 0;
  int32_t tiny_stage_doubles = 0;  // per-batch staged global operands (max over batches)
  int32_t tiny_dig_max = 0;        // per-batch digit block (max over batches)
  // generic digits
  std::vector<GDigit> gdigits;
  // compressed (tied) leaf values, placed after the raw leaf values on device
  std::vector<double> cvals;
  // dense result entry -> physical root offset (-1: structural zero); empty = identity
  std::vector<int64_t> root_map;
  int n_tied_leaves = 0;
  // arena
  int64_t arena_bytes = 0;
  int64_t lane_base = 0;          // start of the per-slice region ([pinned | invariant | per-slice])
  int64_t lane_arena_bytes = 0;   // a slice lane's private copy: offsets [lane_base, lane_base + lane_arena_bytes)
  Loc root_loc{};
  std::vector<Step> steps;
  // stats
  int n_tiny = 0, n_stream = 0, n_gemm = 0, n_generic = 0, n_alias = 0;
  u128 alg_bytes = 0, alg_flops = 0;    // dense (reference) per-node work, summed
  u128 phys_bytes = 0, phys_flops = 0;  // executed work over physical variables
  u128 phys_bytes_inv = 0, phys_flops_inv = 0;  // ... of it, slice-invariant (hoisted: once per pass)
  bool hoisted = false;          // slice-invariant nodes run once per pass (compile.cpp)
  // slice blocks: a per-slice node that does not depend on the fastest-varying
  // sliced index (the last chosen) computes the same tensor for the block_dim
  // consecutive slices that differ only in it: it runs once per block
  int32_t block_dim = 1;         // slices per block (1: no block tier)
  // Slice order.  Slices run in an iteration order that may differ from the
  // reference's lexicographic one (the fold still takes each result from its
  // lexicographic row): the "fast" chosen indices vary fastest, so a block is
  // the slices that differ only in them.  Per chosen index j (lexicographic
  // position): its place value in the iteration id and in the lexicographic id.
  std::vector<int64_t> ord_pv_iter, ord_pv_lex, ord_dim;
  bool permuted = false;         // iteration order != lexicographic
  int64_t closed_granule = 1;    // a range [b, e) with b, e multiples of this maps onto itself
  u128 phys_bytes_blk = 0, phys_flops_blk = 0;  // ... of phys_bytes, block tier (once per block)
  int64_t pinned_bytes = 0;      // arena prefix holding hoisted tensors read by per-slice nodes
  u128 mem_estimate = 0, peak_observed = 0;
};

// no_reuse_limit: if all intermediates together need at most this many bytes,
// every buffer gets its own memory (no write-after-read edges in the DAG).
Program compile_program(const Plan& p, const std::vector<int>& chosen, int64_t no_reuse_limit = 0);

}  // namespace tc
