// Symbolic plan: validation, per-slot index sets, the exact memory model and
// the greedy slice chooser.  Host-only C++ (no CUDA).
#pragma once
#include <cstdint>
#include <iterator>
#include <string>
#include <vector>

#include "tc.h"

namespace tc {

using u128 = unsigned __int128;

inline tc_u128 to_abi(u128 v) { return tc_u128{(uint64_t)v, (uint64_t)(v >> 64)}; }

struct Error {
  int status;
  std::string msg;
};

// Read-only view of a run of ints (a slot's index set / order in a pool).
struct ISpan {
  const int *b = nullptr, *e = nullptr;
  const int* begin() const { return b; }
  const int* end() const { return e; }
  std::reverse_iterator<const int*> rbegin() const { return std::reverse_iterator<const int*>(e); }
  std::reverse_iterator<const int*> rend() const { return std::reverse_iterator<const int*>(b); }
  size_t size() const { return (size_t)(e - b); }
  bool empty() const { return b == e; }
  int operator[](size_t i) const { return b[i]; }
};

// Per-slot int lists stored back to back (slots are filled in order 0..S-1):
// one allocation instead of one vector per slot.
struct SlotPool {
  std::vector<int> pool;
  std::vector<int64_t> off{0};
  ISpan operator[](int s) const { return ISpan{pool.data() + off[s], pool.data() + off[s + 1]}; }
  size_t size() const { return off.size() - 1; }
  void close_slot() { off.push_back((int64_t)pool.size()); }
};

// Reference-compatible symbolic view of (TensorNetwork, ContractionTree).
struct Plan {
  int NI = 0, NL = 0, NN = 0, root = 0;
  std::vector<int> dom, srank;
  std::vector<int64_t> lidx_off, lval_off;
  std::vector<int> lidx;
  std::vector<double> lval;
  std::vector<int> left, right;

  // derived
  std::vector<int> parent;                 // per slot, -1 for root
  SlotPool sets;       // per slot: sorted index ids (node_index_sets)
  SlotPool ref_order;  // per slot: reference index order (tensor.py:108)
  std::vector<int> occ0, occ1;             // leaves holding index i (-1 if none)
  std::vector<char> is_bond;
  std::vector<int> bonds_sorted;           // bond ids sorted by sort_rank
  std::vector<int> seq;                    // full postorder (slots, leaves included)
  bool all_finite = true;                  // every leaf value is finite (tie compression exact)

  int nslots() const { return NL + NN; }
  bool is_leaf(int s) const { return s < NL; }
  int kid_l(int s) const { return left[s - NL]; }
  int kid_r(int s) const { return right[s - NL]; }
  int64_t leaf_size(int l) const { return lval_off[l + 1] - lval_off[l]; }
};

// Build + validate.  Throws Error.
Plan build_plan(const tc_plan_desc& d);

// 8 * prod(dom[i]) over set minus drop; throws TC_OVERFLOW.
u128 set_bytes(const Plan& p, ISpan set, const std::vector<char>& drop);
inline u128 set_bytes(const Plan& p, const std::vector<int>& set, const std::vector<char>& drop) {
  return set_bytes(p, ISpan{set.data(), set.data() + set.size()}, drop);
}

// slicing.py:52-67
u128 mem_cost(const Plan& p, const std::vector<char>& drop);

// slicing.py:70-79 (incremental, parallel over candidates)
int choose_slice_index(const Plan& p, const std::vector<char>& already);

// Work-aware slice chooser (not in the reference): pick bonds until the largest
// intermediate has at most max_entries entries; each pick must shrink the
// current largest intermediates and, among those, keeps the most roofline work
// inside the sliced nodes (adding index c doubles the total work of every node
// NOT containing c).  Returns the picks in order.
std::vector<int> choose_slices_work(const Plan& p, const std::vector<int>& already, u128 max_entries,
                                    int max_picks, double hbm_bytes_per_s, double flops_per_s);

// slicing.py:91-109 accounting only (no arithmetic): the tracked peak
u128 tracked_peak(const Plan& p, const std::vector<char>& drop);

u128 contraction_ops(const Plan& p);
int max_rank(const Plan& p);

std::vector<char> mask_of(const Plan& p, const int32_t* ids, int n);

}  // namespace tc
