// Symbolic plan: see plan.hpp.  Every routine here restates a reference
// function exactly (integer arithmetic, 128-bit byte counts):
//   node_index_sets   network.py:166-175   (child sets XOR)
//   mem_cost          slicing.py:52-67     (strict left-first postorder peak)
//   choose_slice_index slicing.py:70-79    (argmin (cost, sort_key))
//   _execute_tracked  slicing.py:91-109    (live-byte accounting)
//   contraction_ops   network.py:190-201
#include "plan.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <thread>

namespace tc {

static void fail(int st, const std::string& m) { throw Error{st, m}; }

static bool contains(ISpan s, int i) { return std::binary_search(s.begin(), s.end(), i); }

Plan build_plan(const tc_plan_desc& d) {
  Plan p;
  if (d.num_indices < 0 || d.num_leaves < 1 || d.num_nodes < 0)
    fail(TC_BAD_ARG, "plan: negative sizes or no leaves");
  p.NI = d.num_indices;
  p.NL = d.num_leaves;
  p.NN = d.num_nodes;
  p.dom.assign(d.domain, d.domain + p.NI);
  p.srank.assign(d.sort_rank, d.sort_rank + p.NI);
  for (int i = 0; i < p.NI; ++i)
    if (p.dom[i] < 1) fail(TC_BAD_ARG, "plan: index with empty domain");
  p.lidx_off.assign(d.leaf_idx_off, d.leaf_idx_off + p.NL + 1);
  p.lval_off.assign(d.leaf_val_off, d.leaf_val_off + p.NL + 1);
  if (p.lidx_off[0] != 0 || p.lval_off[0] != 0) fail(TC_BAD_ARG, "plan: offsets must start at 0");
  for (int l = 0; l < p.NL; ++l)
    if (p.lidx_off[l + 1] < p.lidx_off[l] || p.lval_off[l + 1] < p.lval_off[l])
      fail(TC_BAD_ARG, "plan: decreasing offsets");
  p.lidx.assign(d.leaf_idx, d.leaf_idx + p.lidx_off[p.NL]);
  p.lval.assign(d.leaf_val, d.leaf_val + p.lval_off[p.NL]);
  p.left.assign(d.left, d.left + p.NN);
  p.right.assign(d.right, d.right + p.NN);
  p.root = d.root_slot;

  const int S = p.nslots();
  p.occ0.assign(p.NI, -1);
  p.occ1.assign(p.NI, -1);
  // leaves: sets and orders are the leaf index lists (sorted / as given)
  p.sets.pool.reserve((size_t)p.lidx_off[p.NL] * 4 + 16);
  p.ref_order.pool.reserve((size_t)p.lidx_off[p.NL] * 4 + 16);
  p.sets.off.reserve(S + 1);
  p.ref_order.off.reserve(S + 1);
  for (int l = 0; l < p.NL; ++l) {
    const int* ids = p.lidx.data() + p.lidx_off[l];
    const int nid = (int)(p.lidx_off[l + 1] - p.lidx_off[l]);
    u128 size = 1;
    for (int q = 0; q < nid; ++q) {
      const int i = ids[q];
      if (i < 0 || i >= p.NI) fail(TC_BAD_ARG, "plan: leaf index id out of range");
      if (p.occ0[i] < 0) p.occ0[i] = l;
      else if (p.occ1[i] < 0) {
        if (p.occ0[i] == l) fail(TC_BAD_ARG, "duplicate index in tensor");
        p.occ1[i] = l;
      } else {
        fail(TC_INDEX_OVERUSE, "index appears 3 or more times");
      }
      size *= (u128)p.dom[i];
    }
    if (size != (u128)p.leaf_size(l)) fail(TC_BAD_ARG, "plan: leaf value count does not match its domains");
    p.ref_order.pool.insert(p.ref_order.pool.end(), ids, ids + nid);
    p.ref_order.close_slot();
    const size_t s0 = p.sets.pool.size();
    p.sets.pool.insert(p.sets.pool.end(), ids, ids + nid);
    std::sort(p.sets.pool.begin() + s0, p.sets.pool.end());
    p.sets.close_slot();
  }
  p.is_bond.assign(p.NI, 0);
  for (int i = 0; i < p.NI; ++i)
    if (p.occ1[i] >= 0) {
      p.is_bond[i] = 1;
      p.bonds_sorted.push_back(i);
    }
  std::sort(p.bonds_sorted.begin(), p.bonds_sorted.end(),
            [&](int a, int b) { return p.srank[a] < p.srank[b]; });

  // tree structure: each slot consumed exactly once, children before parent
  p.parent.assign(S, -1);
  for (int k = 0; k < p.NN; ++k) {
    int me = p.NL + k;
    for (int c : {p.left[k], p.right[k]}) {
      if (c < 0 || c >= me) fail(TC_PLAN_MISMATCH, "contraction tree leaves do not match the network");
      if (p.parent[c] != -1) fail(TC_PLAN_MISMATCH, "contraction tree uses an operand twice");
      p.parent[c] = me;
    }
    const int a = p.left[k], b = p.right[k];
    // the pools never reallocate while a span of them is read below
    const ISpan A = p.sets[a], B = p.sets[b];
    if (p.sets.pool.size() + A.size() + B.size() > p.sets.pool.capacity() ||
        p.ref_order.pool.size() + A.size() + B.size() > p.ref_order.pool.capacity()) {
      p.sets.pool.reserve(2 * p.sets.pool.capacity() + A.size() + B.size());
      p.ref_order.pool.reserve(2 * p.ref_order.pool.capacity() + A.size() + B.size());
    }
    const ISpan A2 = p.sets[a], B2 = p.sets[b], RA = p.ref_order[a], RB = p.ref_order[b];
    std::set_symmetric_difference(A2.begin(), A2.end(), B2.begin(), B2.end(), std::back_inserter(p.sets.pool));
    p.sets.close_slot();
    for (int i : RA)
      if (!contains(B2, i)) p.ref_order.pool.push_back(i);
    for (int i : RB)
      if (!contains(A2, i)) p.ref_order.pool.push_back(i);
    p.ref_order.close_slot();
  }
  int expect_root = p.NN > 0 ? p.NL + p.NN - 1 : 0;
  if (p.root != expect_root) fail(TC_PLAN_MISMATCH, "contraction tree root is not the last node");
  for (int s = 0; s < S; ++s)
    if (s != p.root && p.parent[s] == -1)
      fail(TC_PLAN_MISMATCH, "contraction tree leaves do not match the network");

  // full postorder sequence (leaves included), ContractionTree.postorder
  p.seq.reserve(S);
  {
    std::vector<int> st{p.root}, out;
    out.reserve(S);
    while (!st.empty()) {
      int v = st.back();
      st.pop_back();
      out.push_back(v);
      if (!p.is_leaf(v)) {
        st.push_back(p.kid_l(v));
        st.push_back(p.kid_r(v));
      }
    }
    p.seq.assign(out.rbegin(), out.rend());
  }
  for (double x : p.lval)
    if (!std::isfinite(x)) {
      p.all_finite = false;
      break;
    }
  return p;
}

static inline u128 mul_chk(u128 a, u128 b) {
  u128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw Error{TC_OVERFLOW, "tensor size exceeds 128 bits"};
  return r;
}
static inline u128 add_chk(u128 a, u128 b) {
  u128 r = a + b;
  if (r < a) throw Error{TC_OVERFLOW, "byte count exceeds 128 bits"};
  return r;
}

u128 set_bytes(const Plan& p, ISpan set, const std::vector<char>& drop) {
  u128 out = 8;
  for (int i : set)
    if (!drop[i]) out = mul_chk(out, (u128)p.dom[i]);
  return out;
}

std::vector<char> mask_of(const Plan& p, const int32_t* ids, int n) {
  std::vector<char> m(p.NI, 0);
  for (int k = 0; k < n; ++k) {
    if (ids[k] < 0 || ids[k] >= p.NI) throw Error{TC_BAD_ARG, "index id out of range"};
    m[ids[k]] = 1;
  }
  return m;
}

static inline u128 umax(u128 a, u128 b) { return a > b ? a : b; }

// sizes + peaks for every slot (internal nodes in postorder)
static void full_eval(const Plan& p, const std::vector<char>& drop, std::vector<u128>& size,
                      std::vector<u128>& peak) {
  const int S = p.nslots();
  size.resize(S);
  peak.resize(S);
  for (int l = 0; l < p.NL; ++l) {
    size[l] = set_bytes(p, p.sets[l], drop);
    peak[l] = size[l];
  }
  for (int k = 0; k < p.NN; ++k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    size[v] = set_bytes(p, p.sets[v], drop);
    peak[v] = umax(peak[a], umax(add_chk(size[a], peak[b]), add_chk(add_chk(size[a], size[b]), size[v])));
  }
}

u128 mem_cost(const Plan& p, const std::vector<char>& drop) {
  std::vector<u128> size, peak;
  full_eval(p, drop, size, peak);
  return peak[p.root];
}

// Re-evaluate mem_cost with one more index `c` dropped, touching only the two
// leaf->root paths (nodes whose set contains c are exactly the nodes strictly
// below the LCA on those paths).
struct Scratch {
  std::vector<u128> size, peak;
  std::vector<int> stamp;
  int cur = 0;
};

static u128 cost_with(const Plan& p, const std::vector<u128>& bsize, const std::vector<u128>& bpeak,
                      int c, Scratch& w) {
  ++w.cur;
  const u128 d = (u128)p.dom[c];
  auto S = [&](int v) { return w.stamp[v] == w.cur ? w.size[v] : bsize[v]; };
  auto P = [&](int v) { return w.stamp[v] == w.cur ? w.peak[v] : bpeak[v]; };
  auto eval_internal = [&](int v, bool has_c) {
    int a = p.kid_l(v), b = p.kid_r(v);
    u128 out = has_c ? bsize[v] / d : bsize[v];
    u128 sa = S(a), sb = S(b);
    w.size[v] = out;
    w.peak[v] = umax(P(a), umax(sa + P(b), sa + sb + out));
    w.stamp[v] = w.cur;
  };
  int lca = -1;
  for (int leafv : {p.occ0[c], p.occ1[c]}) {
    w.size[leafv] = bsize[leafv] / d;
    w.peak[leafv] = w.size[leafv];
    w.stamp[leafv] = w.cur;
    int v = p.parent[leafv];
    while (v >= 0 && contains(p.sets[v], c)) {
      eval_internal(v, true);
      v = p.parent[v];
    }
    lca = v;
  }
  for (int v = lca; v >= 0; v = p.parent[v]) eval_internal(v, false);
  return P(p.root);
}

int choose_slice_index(const Plan& p, const std::vector<char>& already) {
  std::vector<int> cand;
  for (int i : p.bonds_sorted)
    if (!already[i]) cand.push_back(i);
  if (cand.empty()) throw Error{TC_NO_CANDIDATES, "no bond index left to slice"};
  std::vector<u128> bsize, bpeak;
  full_eval(p, already, bsize, bpeak);

  unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 64u));
  if (cand.size() < 64) nt = 1;
  std::vector<u128> best_cost(nt, ~(u128)0);
  std::vector<int> best_idx(nt, -1);
  std::vector<Error> errs(nt, Error{TC_OK, ""});
  auto work = [&](unsigned t) {
    try {
      Scratch w;
      w.size.resize(p.nslots());
      w.peak.resize(p.nslots());
      w.stamp.assign(p.nslots(), 0);
      for (size_t k = t; k < cand.size(); k += nt) {
        u128 cost = cost_with(p, bsize, bpeak, cand[k], w);
        // candidates are visited in sort_rank order within a thread, so a
        // strict < keeps the smallest sort_key among equal costs
        if (cost < best_cost[t]) {
          best_cost[t] = cost;
          best_idx[t] = (int)k;
        }
      }
    } catch (const Error& e) {
      errs[t] = e;
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  for (auto& e : errs)
    if (e.status != TC_OK) throw e;
  int bk = -1;
  u128 bc = ~(u128)0;
  for (unsigned t = 0; t < nt; ++t) {
    if (best_idx[t] < 0) continue;
    if (best_cost[t] < bc || (best_cost[t] == bc && best_idx[t] < bk)) {
      bc = best_cost[t];
      bk = best_idx[t];
    }
  }
  return cand[bk];
}

std::vector<int> choose_slices_work(const Plan& p, const std::vector<int>& already, u128 max_entries,
                                    int max_picks, double bw, double fp) {
  std::vector<char> drop(p.NI, 0);
  for (int i : already) drop.at(i) = 1;
  std::vector<int> picks;
  const int S = p.nslots();
  std::vector<double> lsz(S), work(S);
  for (int it = 0; it < max_picks; ++it) {
    // current sizes (log2 for dim-2 plans is exact enough for ranking; use doubles)
    double mx = 0;
    for (int s = 0; s < S; ++s) {
      double z = 1;
      for (int i : p.sets[s])
        if (!drop[i]) z *= p.dom[i];
      lsz[s] = z;
      if (s >= p.NL) mx = std::max(mx, z);
    }
    if ((u128)mx <= max_entries) break;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k, a = p.left[k], b = p.right[k];
      // |A u B| = |A||B|/|shared|, |shared|^2 = |A||B|/|C| for a pairwise contraction
      const double sh = std::sqrt(std::max(1.0, lsz[a] * lsz[b] / std::max(1.0, lsz[v])));
      const double un = lsz[a] * lsz[b] / sh;
      work[v] = std::max(8.0 * (lsz[a] + lsz[b] + lsz[v]) / bw, 2.0 * un / fp);
    }
    int best = -1;
    double best_hits = -1, best_w = -1;
    for (int c : p.bonds_sorted) {
      if (drop[c]) continue;
      double hits = 0, w = 0;
      for (int leafv : {p.occ0[c], p.occ1[c]}) {
        for (int v = p.parent[leafv]; v >= 0 && std::binary_search(p.sets[v].begin(), p.sets[v].end(), c);
             v = p.parent[v]) {
          if (lsz[v] >= mx) hits += 1;
          w += work[v];
        }
      }
      if (hits > best_hits || (hits == best_hits && w > best_w)) {
        best = c;
        best_hits = hits;
        best_w = w;
      }
    }
    if (best < 0) throw Error{TC_NO_CANDIDATES, "no bond index left to slice"};
    picks.push_back(best);
    drop[best] = 1;
  }
  return picks;
}

u128 tracked_peak(const Plan& p, const std::vector<char>& drop) {
  std::vector<u128> size(p.nslots());
  u128 live = 0, peak = 0;
  for (int v : p.seq) {
    size[v] = set_bytes(p, p.sets[v], drop);
    if (p.is_leaf(v)) {
      live = add_chk(live, size[v]);
    } else {
      live = add_chk(live, size[v]);
      peak = umax(peak, live);
      live -= size[p.kid_l(v)] + size[p.kid_r(v)];
    }
    peak = umax(peak, live);
  }
  return peak;
}

u128 contraction_ops(const Plan& p) {
  u128 total = 0;
  std::vector<char> none(p.NI, 0);
  for (int k = 0; k < p.NN; ++k) {
    std::vector<int> uni;
    const ISpan a = p.sets[p.left[k]];
    const ISpan b = p.sets[p.right[k]];
    std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(uni));
    total = add_chk(total, set_bytes(p, uni, none) / 8);
  }
  return total;
}

int max_rank(const Plan& p) {
  size_t r = 0;
  for (int s = 0; s < p.nslots(); ++s) r = std::max(r, p.sets[s].size());
  return (int)r;
}

}  // namespace tc
