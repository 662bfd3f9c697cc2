// Native planning heuristics: min-fill / min-degree elimination orders, the
// elimination tree decomposition, its binarization and tree_to_branch
// (reference pkg/src/tensorcount/decomposition.py:244-411), with the
// reference's exact output (see include/tc_decompose.h).
//
// The reference rescores every remaining vertex after each elimination
// (O(V) fill-in computations per step); here scores are maintained
// incrementally under the elimination's edge updates (removing v changes the
// fill of its neighbours, each fill edge (a, b) changes the fill of a, b and
// of their common neighbours), which gives the same integers.  Ties are broken
// by the same Mersenne-Twister draws as random.Random(seed).choice
// (CPython's _randbelow: k = bit_length(n) bits per draw, rejection).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ograph.hpp"
#include "plan.hpp"
#include "tc.h"
#include "tc_decompose.h"

namespace tc {
int set_last_error(int status, const std::string& msg);  // runtime.cu
}

struct tc_decomp_result {
  tc_decomp_info info{};
  std::vector<int32_t> node_kind, adj, bag, order, leaf_node, leaf_edge;
  std::vector<int64_t> node_num, adj_off{0}, bag_off{0};
};

namespace {
using namespace tc;

// CPython's MT19937 (Modules/_randommodule.c) from a getstate() snapshot
struct PyMT {
  uint32_t mt[624];
  int mti;
  uint32_t next() {
    constexpr uint32_t kUpper = 0x80000000u, kLower = 0x7fffffffu, kMag = 0x9908b0dfu;
    if (mti >= 624) {
      int k = 0;
      uint32_t y;
      for (; k < 624 - 397; ++k) {
        y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
        mt[k] = mt[k + 397] ^ (y >> 1) ^ ((y & 1u) ? kMag : 0u);
      }
      for (; k < 623; ++k) {
        y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
        mt[k] = mt[k + (397 - 624)] ^ (y >> 1) ^ ((y & 1u) ? kMag : 0u);
      }
      y = (mt[623] & kUpper) | (mt[0] & kLower);
      mt[623] = mt[396] ^ (y >> 1) ^ ((y & 1u) ? kMag : 0u);
      mti = 0;
    }
    uint32_t y = mt[mti++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  // random.Random._randbelow_with_getrandbits(n), n < 2^32
  uint32_t below(uint32_t n) {
    const int k = 32 - __builtin_clz(n);
    uint32_t r = next() >> (32 - k);
    while (r >= n) r = next() >> (32 - k);
    return r;
  }
};

// sorted neighbour lists
bool has(const std::vector<int>& a, int x) { return std::binary_search(a.begin(), a.end(), x); }
void insert_sorted(std::vector<int>& a, int x) { a.insert(std::lower_bound(a.begin(), a.end(), x), x); }
void erase_sorted(std::vector<int>& a, int x) {
  auto it = std::lower_bound(a.begin(), a.end(), x);
  if (it != a.end() && *it == x) a.erase(it);
}

struct Elim {
  int nv;
  std::vector<std::vector<int>> A;
  std::vector<int64_t> fill;
  std::vector<int> mark;
  int stamp = 0;
  // |N(a) n N(b)| (marks N(b))
  int64_t common(int a, int b) {
    ++stamp;
    for (int x : A[b]) mark[x] = stamp;
    int64_t c = 0;
    for (int x : A[a]) c += mark[x] == stamp;
    return c;
  }
  int64_t fill_of(int v) {
    ++stamp;
    for (int x : A[v]) mark[x] = stamp;
    int64_t e = 0;
    for (int a : A[v])
      for (int b : A[a])
        if (b > a && mark[b] == stamp) ++e;
    const int64_t d = (int64_t)A[v].size();
    return d * (d - 1) / 2 - e;
  }
  // eliminate v: its neighbours become a clique; fill kept exact
  void eliminate(int v, bool keep_fill) {
    const std::vector<int> Nv = A[v];
    if (keep_fill) {
      for (int w : Nv) fill[w] -= (int64_t)A[w].size() - 1 - common(w, v);
    }
    for (int w : Nv) erase_sorted(A[w], v);
    A[v].clear();
    for (size_t i = 0; i < Nv.size(); ++i)
      for (size_t j = i + 1; j < Nv.size(); ++j) {
        const int a = Nv[i], b = Nv[j];
        if (has(A[a], b)) continue;
        if (keep_fill) {
          ++stamp;
          for (int x : A[b]) mark[x] = stamp;
          int64_t c = 0;
          for (int x : A[a])
            if (mark[x] == stamp) {
              ++c;
              fill[x] -= 1;  // the pair (a, b) inside N(x) becomes adjacent
            }
          fill[a] += (int64_t)A[a].size() - c;
          fill[b] += (int64_t)A[b].size() - c;
        }
        insert_sorted(A[a], b);
        insert_sorted(A[b], a);
      }
  }
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TC_OK;
  } catch (const Error& e) {
    return set_last_error(e.status, e.msg);
  } catch (const std::bad_alloc&) {
    return set_last_error(TC_OOM, "host out of memory");
  } catch (const std::exception& e) {
    return set_last_error(TC_BAD_ARG, e.what());
  }
}

// emit an OGraph (nodes in order) into the result: kinds / numbers per node
void emit_tree(const OGraph& t, const std::vector<int>& kind, const std::vector<int64_t>& num,
               const std::vector<std::vector<int>>* bags, tc_decomp_result& r, std::vector<int>& out_pos) {
  const std::vector<int> nodes = t.nodes();
  out_pos.assign(t.adj.size(), -1);
  for (size_t k = 0; k < nodes.size(); ++k) out_pos[nodes[k]] = (int)k;
  for (int u : nodes) {
    r.node_kind.push_back(kind[u]);
    r.node_num.push_back(num[u]);
    for (int w : t.adj[u]) r.adj.push_back(out_pos[w]);
    r.adj_off.push_back((int64_t)r.adj.size());
    if (bags) {
      for (int x : (*bags)[u]) r.bag.push_back(x);
      r.bag_off.push_back((int64_t)r.bag.size());
    }
  }
  r.info.num_nodes = (int32_t)nodes.size();
  r.info.num_adj = (int64_t)r.adj.size();
  r.info.num_bag = (int64_t)r.bag.size();
}

}  // namespace

extern "C" {

int tc_elim_td(int32_t nv, const int64_t* adj_off, const int32_t* adj, int32_t score, const uint32_t* mt_state,
               int32_t mt_index, int64_t counter_start, tc_decomp_result** out) {
  if (!out) return set_last_error(TC_BAD_ARG, "null output");
  *out = nullptr;
  auto* r = new (std::nothrow) tc_decomp_result;
  if (!r) return set_last_error(TC_OOM, "host out of memory");
  const int st = guarded([&] {
    if (nv < 0 || (score != 0 && score != 1) || !mt_state || mt_index < 0 || mt_index > 624)
      throw Error{TC_BAD_ARG, "bad elimination arguments"};
    // ---- _heuristic_order (decomposition.py:301-319) ----------------------
    Elim E;
    E.nv = nv;
    E.A.resize(nv);
    E.mark.assign(nv, 0);
    for (int v = 0; v < nv; ++v) {
      for (int64_t q = adj_off[v]; q < adj_off[v + 1]; ++q) {
        const int w = adj[q];
        if (w < 0 || w >= nv || w == v) throw Error{TC_BAD_ARG, "bad adjacency"};
        E.A[v].push_back(w);
      }
      std::sort(E.A[v].begin(), E.A[v].end());
      E.A[v].erase(std::unique(E.A[v].begin(), E.A[v].end()), E.A[v].end());
    }
    for (int v = 0; v < nv; ++v)
      for (int w : E.A[v])
        if (!has(E.A[w], v)) throw Error{TC_BAD_ARG, "adjacency is not symmetric"};
    const bool by_fill = score == 0;
    if (by_fill) {
      E.fill.resize(nv);
      for (int v = 0; v < nv; ++v) E.fill[v] = E.fill_of(v);
    }
    PyMT mt;
    std::memcpy(mt.mt, mt_state, sizeof(mt.mt));
    mt.mti = mt_index;
    std::vector<int> remaining(nv);
    for (int v = 0; v < nv; ++v) remaining[v] = v;  // sorted(str) order from the caller
    std::vector<std::vector<int>> bags;
    std::vector<int> ties;
    while (!remaining.empty()) {
      int64_t best = INT64_MAX;
      for (int v : remaining) best = std::min<int64_t>(best, by_fill ? E.fill[v] : (int64_t)E.A[v].size());
      ties.clear();
      for (int v : remaining)
        if ((by_fill ? E.fill[v] : (int64_t)E.A[v].size()) == best) ties.push_back(v);
      const int v = ties[mt.below((uint32_t)ties.size())];
      r->order.push_back(v);
      std::vector<int> bag = E.A[v];  // _eliminate's bag: {v} | nbrs
      insert_sorted(bag, v);
      bags.push_back(std::move(bag));
      E.eliminate(v, by_fill);
      remaining.erase(std::find(remaining.begin(), remaining.end(), v));
    }
    // ---- _elimination_tree_decomposition (decomposition.py:258-275) -------
    const int K = (int)r->order.size();
    std::vector<int> pos(nv, -1);
    for (int k = 0; k < K; ++k) pos[r->order[k]] = k;
    OGraph t;
    std::vector<int64_t> num;
    std::vector<std::vector<int>> tbag;
    int64_t counter = counter_start;
    auto fresh_td = [&](std::vector<int> b) {
      const int u = t.new_node();
      num.push_back(counter++);
      tbag.push_back(std::move(b));
      return u;
    };
    if (K == 0) {
      t.add_node(fresh_td({}));
    } else {
      for (int k = 0; k < K; ++k) fresh_td(bags[k]);
      for (int k = 0; k < K; ++k) t.add_node(k);
      for (int k = 0; k < K; ++k) {
        int target = -1;
        for (int x : bags[k])
          if (pos[x] > k && (target < 0 || pos[x] < target)) target = pos[x];
        if (target < 0 && k + 1 < K) target = k + 1;
        if (target >= 0) t.add_edge(k, target);
      }
    }
    // ---- binarize_tree_decomposition (decomposition.py:278-294) -----------
    t.recopy();
    for (size_t p = 0; p < t.order.size();) {
      const int n = t.order[p];
      if (!t.alive[n] || t.degree(n) <= 3) {
        ++p;
        continue;
      }
      const std::vector<int> nbrs = t.adj[n];
      const int copy = fresh_td(tbag[n]);
      t.add_edge(n, copy);
      for (size_t q = 2; q < nbrs.size(); ++q) {
        t.remove_edge(n, nbrs[q]);
        t.add_edge(copy, nbrs[q]);
      }
    }
    std::vector<int> kind(t.adj.size(), 0), opos;
    emit_tree(t, kind, num, &tbag, *r, opos);
    r->info.num_order = K;
    r->info.counter_end = counter;
  });
  if (st != TC_OK) {
    delete r;
    return st;
  }
  *out = r;
  return TC_OK;
}

int tc_tree_to_branch(int32_t nn, const int64_t* adj_off, const int32_t* adj, const int32_t* node_rank,
                      const int64_t* bag_off, const int32_t* bag, int32_t nv, int32_t ne, const int32_t* edge_u,
                      const int32_t* edge_v, int64_t counter_start, tc_decomp_result** out) {
  if (!out) return set_last_error(TC_BAD_ARG, "null output");
  *out = nullptr;
  auto* r = new (std::nothrow) tc_decomp_result;
  if (!r) return set_last_error(TC_OOM, "host out of memory");
  const int st = guarded([&] {
    if (nn < 1 || nv < 0 || ne < 1) throw Error{TC_BAD_ARG, "bad tree_to_branch arguments"};
    // node_order = sorted(td.tree.nodes, key=str)
    std::vector<int> node_order(nn, -1);
    for (int k = 0; k < nn; ++k) {
      if (node_rank[k] < 0 || node_rank[k] >= nn || node_order[node_rank[k]] >= 0)
        throw Error{TC_BAD_ARG, "node ranks are not a permutation"};
      node_order[node_rank[k]] = k;
    }
    // host = first node (in node_order) whose bag holds both endpoints
    std::vector<std::vector<int>> holds(nv);  // vertex -> node ranks holding it, ascending
    for (int rk = 0; rk < nn; ++rk) {
      const int k = node_order[rk];
      for (int64_t q = bag_off[k]; q < bag_off[k + 1]; ++q) {
        const int x = bag[q];
        if (x < 0 || x >= nv) throw Error{TC_BAD_ARG, "bag vertex out of range"};
        if (holds[x].empty() || holds[x].back() != rk) holds[x].push_back(rk);
      }
    }
    std::vector<std::vector<int>> hosted(nn);
    for (int e = 0; e < ne; ++e) {
      const auto& a = holds[edge_u[e]];
      const auto& b = holds[edge_v[e]];
      int host = -1;
      for (size_t i = 0, j = 0; i < a.size() && j < b.size();) {
        if (a[i] < b[j]) ++i;
        else if (b[j] < a[i]) ++j;
        else {
          host = a[i];
          break;
        }
      }
      if (host < 0) throw Error{TC_BAD_ARG, "NoHostBag: " + std::to_string(e)};
      hosted[node_order[host]].push_back(e);
    }
    // the td tree in networkx order
    OGraph td;
    for (int k = 0; k < nn; ++k) td.new_node();
    for (int k = 0; k < nn; ++k) td.add_node(k);
    for (int k = 0; k < nn; ++k)
      for (int64_t q = adj_off[k]; q < adj_off[k + 1]; ++q) td.adj[k].push_back(adj[q]);
    // one copy of each td node per attachment (tree arcs + hosted edges)
    OGraph t;
    std::vector<int> kind;
    std::vector<int64_t> num;
    int64_t counter = counter_start;
    auto fresh = [&](int kd) {
      const int u = t.new_node();
      kind.push_back(kd);
      num.push_back(counter++);
      return u;
    };
    std::vector<std::vector<int>> slots(nn);
    std::vector<int> cursor(nn, 0);
    for (int rk = 0; rk < nn; ++rk) {
      const int k = node_order[rk];
      const int needed = std::max(1, td.degree(k) + (int)hosted[k].size());
      for (int c = 0; c < needed; ++c) slots[k].push_back(fresh(1));
      t.add_node(slots[k][0]);
      for (int c = 0; c + 1 < needed; ++c) t.add_edge(slots[k][c], slots[k][c + 1]);
    }
    auto take = [&](int k) { return slots[k][cursor[k]++]; };
    td.for_edges([&](int n, int m) {
      const int a = take(n);
      const int b = take(m);
      t.add_edge(a, b);
    });
    std::vector<char> mapped;
    for (int rk = 0; rk < nn; ++rk) {
      const int k = node_order[rk];
      for (int e : hosted[k]) {
        const int lf = fresh(2);
        r->leaf_node.push_back(lf);
        r->leaf_edge.push_back(e);
        t.add_edge(take(k), lf);
      }
    }
    mapped.assign(t.adj.size(), 0);
    for (int lf : r->leaf_node) mapped[lf] = 1;
    smooth(t, mapped);  // _prune_and_smooth (decomposition.py:395-411)
    std::vector<int> opos;
    emit_tree(t, kind, num, nullptr, *r, opos);
    for (int& lf : r->leaf_node) lf = opos[lf];
    r->info.num_leaf_map = (int32_t)r->leaf_node.size();
    r->info.counter_end = counter;
  });
  if (st != TC_OK) {
    delete r;
    return st;
  }
  *out = r;
  return TC_OK;
}

int tc_validate_td(int32_t nn, const int64_t* adj_off, const int32_t* adj, const int64_t* bag_off,
                   const int32_t* bag, int32_t nv, int32_t ne, const int32_t* edge_u, const int32_t* edge_v,
                   int32_t* shape, int32_t* bad_edge, int8_t* disconnected) {
  if (!shape || !bad_edge || (nv > 0 && !disconnected)) return set_last_error(TC_BAD_ARG, "null output");
  return guarded([&] {
    *shape = 0;
    *bad_edge = -1;
    for (int v = 0; v < nv; ++v) disconnected[v] = 0;
    // _check_tree_shape (decomposition.py:81-85): non-empty, connected, |E| = |V| - 1
    if (nn == 0) {
      *shape = 1;
      return;
    }
    int64_t ends = 0;
    for (int k = 0; k < nn; ++k)
      for (int64_t q = adj_off[k]; q < adj_off[k + 1]; ++q) {
        if (adj[q] < 0 || adj[q] >= nn) throw Error{TC_BAD_ARG, "bad tree adjacency"};
        ++ends;
      }
    bool ok = ends == 2 * (int64_t)(nn - 1);
    if (ok) {
      std::vector<char> seen(nn, 0);
      std::vector<int> st{0};
      seen[0] = 1;
      int cnt = 1;
      while (!st.empty()) {
        const int u = st.back();
        st.pop_back();
        for (int64_t q = adj_off[u]; q < adj_off[u + 1]; ++q)
          if (!seen[adj[q]]) seen[adj[q]] = 1, ++cnt, st.push_back(adj[q]);
      }
      ok = cnt == nn;
    }
    if (!ok) {
      *shape = 2;
      return;
    }
    // host bags: the first edge (in order) none of whose bags holds both ends
    std::vector<std::vector<int>> holds(std::max(0, nv));
    std::vector<int> bag_size(nn);
    for (int k = 0; k < nn; ++k)
      for (int64_t q = bag_off[k]; q < bag_off[k + 1]; ++q) {
        const int x = bag[q];
        if (x >= 0 && x < nv && (holds[x].empty() || holds[x].back() != k)) holds[x].push_back(k);
      }
    for (int e = 0; e < ne && *bad_edge < 0; ++e) {
      const auto& a = holds[edge_u[e]];
      const auto& b = holds[edge_v[e]];
      bool host = false;
      for (size_t i = 0, j = 0; i < a.size() && j < b.size() && !host;) {
        if (a[i] < b[j]) ++i;
        else if (b[j] < a[i]) ++j;
        else host = true;
      }
      if (!host) *bad_edge = e;
    }
    // per vertex: its bags induce a connected subtree iff nodes - edges == 1
    std::vector<int64_t> induced_edges(std::max(0, nv), 0);
    std::vector<int> mark(std::max(0, nv), -1);
    for (int u = 0; u < nn; ++u) {
      for (int64_t q = bag_off[u]; q < bag_off[u + 1]; ++q)
        if (bag[q] >= 0 && bag[q] < nv) mark[bag[q]] = u;
      for (int64_t q = adj_off[u]; q < adj_off[u + 1]; ++q) {
        const int w = adj[q];
        if (w <= u) continue;  // each tree edge once
        for (int64_t r = bag_off[w]; r < bag_off[w + 1]; ++r)
          if (bag[r] >= 0 && bag[r] < nv && mark[bag[r]] == u) ++induced_edges[bag[r]];
      }
    }
    for (int v = 0; v < nv; ++v)
      if (!holds[v].empty() && (int64_t)holds[v].size() - induced_edges[v] != 1) disconnected[v] = 1;
  });
}

int tc_decomp_info_get(const tc_decomp_result* r, tc_decomp_info* info) {
  if (!r || !info) return set_last_error(TC_BAD_ARG, "null argument");
  *info = r->info;
  return TC_OK;
}

int tc_decomp_fetch(const tc_decomp_result* r, int32_t* node_kind, int64_t* node_num, int64_t* adj_off, int32_t* adj,
                    int64_t* bag_off, int32_t* bag, int32_t* order, int32_t* leaf_node, int32_t* leaf_edge) {
  if (!r) return set_last_error(TC_BAD_ARG, "null result");
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(node_kind, r->node_kind);
  cp(node_num, r->node_num);
  cp(adj_off, r->adj_off);
  cp(adj, r->adj);
  cp(bag_off, r->bag_off);
  cp(bag, r->bag);
  cp(order, r->order);
  cp(leaf_node, r->leaf_node);
  cp(leaf_edge, r->leaf_edge);
  return TC_OK;
}

void tc_decomp_free(tc_decomp_result* r) { delete r; }

}  // extern "C"
