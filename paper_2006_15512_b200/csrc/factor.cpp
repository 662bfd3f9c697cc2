// Native FactorTree step: factor_branch_audit (reference
// pkg/src/tensorcount/factoring.py:270-333) restated in C++ with the
// reference's exact output (see include/tc_factor.h for the function map).
//
// The reference builds its plan with networkx graphs and sorts by str() of
// node labels; the result (piece order, bond numbering, tree shape, left /
// right children) depends on those orders, so they are reproduced here:
//   * OGraph keeps nodes and adjacency in insertion order with networkx's
//     semantics (add_edge appends unseen endpoints and neighbours,
//     remove_edge / remove_node delete in place, EdgeView yields (u, v) with
//     u the earlier node, once per edge);
//   * every str()-sort compares the actual str / repr text (bd node texts come
//     from the caller; fresh labels are built as Python prints them:
//     ('x', '000000000012'), zero-padded as fresh_node does,
//     decomposition.py:23-26).
// Widths (decomposition.py:166-241) are computed with subtree sums over an
// LCA structure instead of the reference's Counter merges (same numbers).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ograph.hpp"
#include "plan.hpp"
#include "tc.h"
#include "tc_factor.h"

namespace tc {
int set_last_error(int status, const std::string& msg);  // runtime.cu
}

struct tc_factor_result {
  tc_factor_info info{};
  std::vector<int32_t> piece_src, piece_kind, piece_idx, bond_ordinal, bond_k, bond_domain, left, right;
  std::vector<int64_t> piece_idx_off{0}, piece_val_off{0};
  std::vector<double> piece_val;
};

namespace {
using namespace tc;

[[noreturn]] void raise(const char* kind, const std::string& msg) { throw Error{TC_BAD_ARG, std::string(kind) + ": " + msg}; }

// ---- rooted tree with LCA (widths, Steiner subtrees) -----------------------
struct Rooted {
  int n = 0, L = 1;
  std::vector<int> parent, depth, tin, post;  // post: children before parents
  std::vector<std::vector<int>> up;
  void build(const OGraph& g, int root) {
    n = (int)g.adj.size();
    parent.assign(n, -1);
    depth.assign(n, 0);
    tin.assign(n, -1);
    post.clear();
    std::vector<int> pre;
    std::vector<std::pair<int, int>> st{{root, -1}};
    int t = 0;
    while (!st.empty()) {
      auto [u, p] = st.back();
      st.pop_back();
      parent[u] = p;
      depth[u] = p < 0 ? 0 : depth[p] + 1;
      tin[u] = t++;
      pre.push_back(u);
      for (int w : g.adj[u])
        if (w != p) st.push_back({w, u});
    }
    post.assign(pre.rbegin(), pre.rend());
    L = 1;
    while ((1 << L) < std::max(2, t)) ++L;
    up.assign(L, std::vector<int>(n, -1));
    for (int u : pre) up[0][u] = parent[u] < 0 ? u : parent[u];
    for (int k = 1; k < L; ++k)
      for (int u : pre) up[k][u] = up[k - 1][up[k - 1][u]];
  }
  int lca(int a, int b) const {
    if (depth[a] < depth[b]) std::swap(a, b);
    for (int k = L - 1; k >= 0; --k)
      if (depth[a] - (1 << k) >= depth[b]) a = up[k][a];
    if (a == b) return a;
    for (int k = L - 1; k >= 0; --k)
      if (up[k][a] != up[k][b]) a = up[k][a], b = up[k][b];
    return parent[a];
  }
};

// max over arcs of the number of terminal sets the arc splits (some but not
// all of the set below it): width_branch / width_carving.
int max_split(const OGraph& g, int root, const std::vector<std::vector<int>>& sets) {
  Rooted R;
  R.build(g, root);
  std::vector<int64_t> s(g.adj.size(), 0);
  std::vector<int> v;
  for (const auto& set : sets) {
    if (set.size() < 2) continue;
    v = set;
    std::sort(v.begin(), v.end(), [&](int a, int b) { return R.tin[a] < R.tin[b]; });
    v.erase(std::unique(v.begin(), v.end()), v.end());
    // nodes below which the set is present: +1 per member, -1 per lca of
    // tin-consecutive members; present everywhere below the set's lca: -1 there
    int all = v[0];
    for (size_t i = 0; i < v.size(); ++i) {
      s[v[i]] += 1;
      if (i) s[R.lca(v[i - 1], v[i])] -= 1;
      all = R.lca(all, v[i]);
    }
    s[all] -= 1;
  }
  int best = 0;
  for (int u : R.post) {
    if (R.parent[u] >= 0) {
      best = std::max<int64_t>(best, s[u]);
      s[R.parent[u]] += s[u];
    }
  }
  return best;
}

std::string fresh_label(const char* prefix, int64_t& counter) {
  char b[64];
  std::snprintf(b, sizeof b, "('%s', '%012lld')", prefix, (long long)counter++);
  return b;
}

struct Factor {
  const tc_factor_input& in;
  tc_factor_result& out;
  int T, NI, N;
  std::vector<std::string_view> sstr, srepr;  // bd node texts
  std::vector<int> own0, own1;                // owners of each index (-1: none / free vertex)
  OGraph bd;

  explicit Factor(const tc_factor_input& i, tc_factor_result& o) : in(i), out(o) {
    T = in.num_tensors;
    NI = in.num_indices;
    N = in.num_nodes;
  }
  int rank(int t) const { return (int)(in.idx_off[t + 1] - in.idx_off[t]); }
  const int32_t* idx(int t) const { return in.idx + in.idx_off[t]; }
  const double* val(int t) const { return in.val_ptr[t]; }
  int64_t size(int t) const { return in.val_off[t + 1] - in.val_off[t]; }
  bool str_less(int a, int b) const { return sstr[a] < sstr[b]; }

  void run();
};

void Factor::run() {
  if (T < 1 || NI < 0 || N < 0) raise("ValueError", "bad factor input sizes");
  for (int i = 0; i < N; ++i) {
    sstr.emplace_back(in.str_buf + in.str_off[i], (size_t)(in.str_off[i + 1] - in.str_off[i]));
    srepr.emplace_back(in.repr_buf + in.repr_off[i], (size_t)(in.repr_off[i + 1] - in.repr_off[i]));
  }
  own0.assign(NI, -1);
  own1.assign(NI, -1);
  for (int t = 0; t < T; ++t)
    for (int q = 0; q < rank(t); ++q) {
      const int i = idx(t)[q];
      if (i < 0 || i >= NI) raise("ValueError", "index id out of range");
      if (own0[i] < 0) own0[i] = t;
      else if (own1[i] < 0) own1[i] = t;
      else raise("ValueError", "index appears more than twice");
    }

  // phase timings on stderr when TC_FACTOR_TIMING is set (diagnostics)
  static const bool timing = std::getenv("TC_FACTOR_TIMING") != nullptr;
  auto tlast = std::chrono::steady_clock::now();
  auto tmark = [&](const char* name) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[factor] %-14s %8.2f ms\n", name, std::chrono::duration<double, std::milli>(now - tlast).count());
    tlast = now;
  };
  // ---- validate_branch_decomposition (decomposition.py:81-86, 111-134) ----
  const std::string what = "branch decomposition";
  if (N == 0) raise("InvalidDecomposition", what + ": empty tree");
  for (int u = 0; u < N; ++u) bd.new_node();
  for (int u = 0; u < N; ++u) bd.add_node(u);
  int64_t ne = 0;
  for (int u = 0; u < N; ++u)
    for (int64_t q = in.adj_off[u]; q < in.adj_off[u + 1]; ++q) {
      const int w = in.adj[q];
      if (w < 0 || w >= N || w == u) raise("InvalidDecomposition", what + ": decomposition graph is not a tree");
      bd.adj[u].push_back(w);
      ++ne;
    }
  bool tree_ok = ne == 2 * (int64_t)(N - 1);
  if (tree_ok) {  // connected
    std::vector<char> seen(N, 0);
    std::vector<int> st{0};
    seen[0] = 1;
    int cnt = 1;
    while (!st.empty()) {
      const int u = st.back();
      st.pop_back();
      for (int w : bd.adj[u])
        if (!seen[w]) seen[w] = 1, ++cnt, st.push_back(w);
    }
    tree_ok = cnt == N;
  }
  if (!tree_ok) raise("InvalidDecomposition", what + ": decomposition graph is not a tree");
  std::vector<int> leaf_of_index(NI, -1), index_of_leaf(N, -1);
  bool bij = true;
  for (int k = 0; k < in.num_leaf_map; ++k) {
    const int u = in.leaf_node[k], i = in.leaf_index[k];
    if (u < 0 || u >= N || i < 0 || i >= NI || leaf_of_index[i] >= 0 || index_of_leaf[u] >= 0) {
      bij = false;
      break;
    }
    leaf_of_index[i] = u;
    index_of_leaf[u] = i;
  }
  for (int i = 0; i < NI && bij; ++i) bij = own0[i] < 0 || leaf_of_index[i] >= 0;  // every edge of g mapped
  for (int i = 0; i < NI && bij; ++i) bij = leaf_of_index[i] < 0 || own0[i] >= 0;   // and only those
  if (!bij) raise("InvalidDecomposition", what + ": leaves are not a bijection onto the target set");
  for (int u = 0; u < N; ++u) {
    const int deg = bd.degree(u);
    if (index_of_leaf[u] >= 0) {
      if (deg > 1)
        raise("InvalidDecomposition", what + ": mapped leaf " + std::string(srepr[u]) + " has degree " + std::to_string(deg));
    } else if (N > 2 && deg != 3) {
      raise("InvalidDecomposition",
            what + ": internal node " + std::string(srepr[u]) + " has degree " + std::to_string(deg) + ", expected 3");
    }
  }
  for (int u = 0; u < N; ++u)
    if (bd.degree(u) <= 1 && index_of_leaf[u] < 0 && N > 1)
      raise("InvalidDecomposition", what + ": unmapped leaf node " + std::string(srepr[u]));

  tmark("validate");
  // ---- width_branch (decomposition.py:166-191) ----------------------------
  const int Z = T;  // key of the free vertex ("z")
  {
    std::vector<std::vector<int>> sets(T + 1);
    for (int i = 0; i < NI; ++i)
      if (own0[i] >= 0) {
        sets[own0[i]].push_back(leaf_of_index[i]);
        sets[own1[i] >= 0 ? own1[i] : Z].push_back(leaf_of_index[i]);
      }
    out.info.branch_width = N > 1 ? max_split(bd, 0, sets) : 0;
  }
  if (out.info.branch_width == 0) {
    out.info.trivial = 1;
    return;
  }

  tmark("width_branch");
  // ---- Part 1: spanning subtrees and pieces (factoring.py:287-310) --------
  Rooted R;
  R.build(bd, 0);
  // terminals per key in leaf_map order
  std::vector<std::vector<int>> term(T + 1);
  for (int k = 0; k < in.num_leaf_map; ++k) {
    const int u = in.leaf_node[k], i = in.leaf_index[k];
    term[own0[i]].push_back(u);
    term[own1[i] >= 0 ? own1[i] : Z].push_back(u);
  }
  std::vector<int> stamp(N, -1);
  std::vector<std::vector<int>> S(T + 1);  // subtree nodes per key (insertion order irrelevant)
  auto steiner = [&](int key) {
    auto& tv = term[key];
    auto& s = S[key];
    if (tv.empty()) return;
    std::vector<int> v = tv;
    std::sort(v.begin(), v.end(), [&](int a, int b) { return R.tin[a] < R.tin[b]; });
    auto mark = [&](int u) {
      if (stamp[u] != key) stamp[u] = key, s.push_back(u);
    };
    mark(v[0]);
    for (size_t q = 1; q < v.size(); ++q) {
      int a = v[q - 1], b = v[q];
      const int c = R.lca(a, b);
      for (; a != c; a = R.parent[a]) mark(a);
      for (; b != c; b = R.parent[b]) mark(b);
      mark(c);
    }
  };
  const bool has_free = !term[Z].empty();
  std::vector<char> isolated(T, 0);
  for (int t = 0; t < T; ++t) {
    if (rank(t) == 0) {
      isolated[t] = 1;
      continue;
    }
    steiner(t);
  }
  if (has_free) steiner(Z);
  // S-neighbours of u in key's subtree: bd neighbours carrying the key's stamp;
  // stamps are overwritten per key, so keep a membership test per key instead
  std::unordered_map<int64_t, int> hv_id;  // (key, node) -> H vertex
  std::vector<int> hv_key, hv_node;
  auto hvk = [&](int key, int u) { return (int64_t)key * N + u; };
  for (int key = 0; key <= T; ++key)
    for (int u : S[key]) {
      hv_id.emplace(hvk(key, u), (int)hv_key.size());
      hv_key.push_back(key);
      hv_node.push_back(u);
    }
  auto in_sub = [&](int key, int u) { return hv_id.count(hvk(key, u)) != 0; };
  auto sub_nbrs_sorted = [&](int key, int u) {
    std::vector<int> o;
    for (int w : bd.adj[u])
      if (in_sub(key, w)) o.push_back(w);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return str_less(a, b); });
    return o;
  };

  tmark("steiner");
  // kinds (detect_kind, factoring.py:105-144).  The reduction's copy tensors
  // are dense 2^occ arrays (reduction.py:32-39, up to 1 GB on C4): the
  // off-diagonal zero test runs on worker threads over chunks of 2^20
  // entries; then the first non-factorable tensor in network order raises.
  std::vector<int> kind(T, 0);  // 0 trivial, 1 copy, 2 clause, -1 neither
  std::vector<std::vector<double>> diag(T);
  std::vector<std::vector<int>> pol(T);  // per position: satisfying value
  std::vector<int64_t> dstep(T, 0);      // offset of (1, ..., 1); 0: domains differ
  std::vector<char> offdiag(T, 0);       // a nonzero off-diagonal entry was seen
  {
    struct Chunk {
      int t;
      int64_t e0, e1;
    };
    std::vector<Chunk> chunks;
    constexpr int64_t kChunk = (int64_t)1 << 20;
    for (int t = 0; t < T; ++t) {
      if (isolated[t] || S[t].size() <= 1) continue;
      const int r = rank(t);
      const int32_t* ix = idx(t);
      bool eq = true;
      for (int q = 1; q < r; ++q) eq &= in.domain[ix[q]] == in.domain[ix[0]];
      if (!eq) continue;
      const int64_t d = in.domain[ix[0]];
      int64_t step = 0, pw = 1;
      for (int q = 0; q < r; ++q) step += pw, pw *= d;
      dstep[t] = step;
      for (int64_t e = 0; e < size(t); e += kChunk) chunks.push_back({t, e, std::min(size(t), e + kChunk)});
    }
    std::atomic<size_t> next_c{0};
    auto worker = [&] {
      for (size_t q; (q = next_c.fetch_add(1)) < chunks.size();) {
        const Chunk& c = chunks[q];
        const double* v = val(c.t);
        const int64_t step = dstep[c.t];
        bool nz = false;
        int64_t nd = (c.e0 + step - 1) / step * step;  // next diagonal position
        for (int64_t e = c.e0; e < c.e1 && !nz; ++e) {
          if (e == nd) {
            nd += step;
            continue;
          }
          nz = v[e] != 0.0;
        }
        if (nz) offdiag[c.t] = 1;  // benign race: every writer stores 1
      }
    };
    int64_t total = 0;
    for (auto& c : chunks) total += c.e1 - c.e0;
    const int nth = total > (1 << 22) ? (int)std::min<size_t>(16, std::max(1u, std::thread::hardware_concurrency())) : 1;
    std::vector<std::thread> th;
    for (int w = 1; w < nth; ++w) th.emplace_back(worker);
    worker();
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < T; ++t) {
    if (isolated[t] || S[t].size() <= 1) continue;
    const int r = rank(t);
    const int32_t* ix = idx(t);
    const double* v = val(t);
    const int64_t n = size(t);
    if (dstep[t] && !offdiag[t]) {  // a generalised diagonal (multiples of step below n are the diagonal)
      const int64_t d = in.domain[ix[0]];
      diag[t].resize(d);
      for (int64_t k = 0; k < d; ++k) diag[t][k] = v[k * dstep[t]];
      kind[t] = 1;
      continue;
    }
    bool dim2 = true;
    for (int q = 0; q < r; ++q) dim2 &= in.domain[ix[q]] == 2;
    kind[t] = -1;
    if (dim2) {
      bool ok01 = true;
      int64_t zeros = 0, zat = -1;
      for (int64_t e = 0; e < n && ok01 && zeros <= 1; ++e) {
        if (v[e] == 0.0) ++zeros, zat = e;
        else if (v[e] != 1.0) ok01 = false;
      }
      if (ok01 && zeros == 1) {
        pol[t].resize(r);
        for (int q = 0; q < r; ++q) pol[t][q] = 1 - (int)((zat >> (r - 1 - q)) & 1);
        kind[t] = 2;
      }
    }
  }
  for (int t = 0; t < T; ++t)
    if (kind[t] < 0)
      raise("NotFactorable", "tensor #" + std::to_string(t) + " is neither a diagonal nor an acceptance tensor");

  tmark("kinds");
  // piece order: ordinals by str(ordinal), nodes by str(node); then isolated
  std::vector<int> ords;
  for (int t = 0; t < T; ++t)
    if (!isolated[t]) ords.push_back(t);
  std::sort(ords.begin(), ords.end(), [](int a, int b) { return std::to_string(a) < std::to_string(b); });
  std::vector<int> piece_of_hv(hv_key.size(), -1);
  std::vector<int> piece_of_isolated(T, -1);
  int npieces = 0;
  for (int t : ords) {
    std::vector<int> nodes = S[t];
    std::sort(nodes.begin(), nodes.end(), [&](int a, int b) { return str_less(a, b); });
    // bonds: S edges sorted by [str(a), str(b)] with the pair sorted (_fresh_bonds)
    std::unordered_map<int64_t, int> bond_of;  // (u, w) -> bond id
    if (nodes.size() > 1) {
      std::vector<std::pair<int, int>> edges;
      for (int u : nodes)
        for (int w : bd.adj[u])
          if (in_sub(t, w) && str_less(u, w)) edges.push_back({u, w});
      std::sort(edges.begin(), edges.end(), [&](const auto& x, const auto& y) {
        if (sstr[x.first] != sstr[y.first]) return sstr[x.first] < sstr[y.first];
        return sstr[x.second] < sstr[y.second];
      });
      const int d = kind[t] == 1 ? (int)diag[t].size() : 2;
      for (size_t k = 0; k < edges.size(); ++k) {
        const int b = (int)out.bond_ordinal.size();
        out.bond_ordinal.push_back(t);
        out.bond_k.push_back((int)k);
        out.bond_domain.push_back(d);
        bond_of[(int64_t)edges[k].first * N + edges[k].second] = b;
        bond_of[(int64_t)edges[k].second * N + edges[k].first] = b;
      }
    }
    // leaf node -> position of its index in the tensor
    std::unordered_map<int, int> pos_of_leaf;
    for (int q = 0; q < rank(t); ++q) pos_of_leaf[leaf_of_index[idx(t)[q]]] = q;
    // carrier / clause root: the leaf whose index has the smallest sort key
    int carrier = -1;
    for (int q = 0; q < rank(t); ++q)
      if (carrier < 0 || in.sort_rank[idx(t)[q]] < in.sort_rank[idx(t)[pos_of_leaf[carrier]]])
        carrier = leaf_of_index[idx(t)[q]];
    // clause: parent of every node when rooted at the carrier
    std::unordered_map<int, int> par;
    if (kind[t] == 2) {
      par[carrier] = -1;
      std::vector<int> st{carrier};
      while (!st.empty()) {
        const int u = st.back();
        st.pop_back();
        for (int w : bd.adj[u])
          if (in_sub(t, w) && !par.count(w)) par[w] = u, st.push_back(w);
      }
    }
    for (int u : nodes) {
      const int p = npieces++;
      piece_of_hv[hv_id[hvk(t, u)]] = p;
      out.piece_src.push_back(t);
      if (nodes.size() == 1) {  // trivial dimension tree: the tensor itself (factoring.py:157-159)
        out.piece_kind.push_back(0);
        for (int q = 0; q < rank(t); ++q) out.piece_idx.push_back(idx(t)[q]);
        out.piece_idx_off.push_back((int64_t)out.piece_idx.size());
        out.piece_val.insert(out.piece_val.end(), val(t), val(t) + size(t));
        out.piece_val_off.push_back((int64_t)out.piece_val.size());
        continue;
      }
      out.piece_kind.push_back(kind[t]);
      // _piece_indices: own index, then bonds to neighbours by str
      std::vector<int> ids;
      int own = -1;
      auto it = pos_of_leaf.find(u);
      if (it != pos_of_leaf.end()) {
        own = it->second;
        ids.push_back(idx(t)[own]);
      }
      const std::vector<int> nb = sub_nbrs_sorted(t, u);
      for (int w : nb) ids.push_back(-1 - bond_of[(int64_t)u * N + w]);
      const int r = (int)ids.size();
      for (int x : ids) out.piece_idx.push_back(x);
      out.piece_idx_off.push_back((int64_t)out.piece_idx.size());
      if (kind[t] == 1) {  // _factor_copy
        const int64_t d = (int64_t)diag[t].size();
        int64_t n = 1, step = 0, pw = 1;
        for (int q = 0; q < r; ++q) n *= d, step += pw, pw *= d;
        const size_t base = out.piece_val.size();
        out.piece_val.resize(base + n, 0.0);
        for (int64_t k = 0; k < d; ++k) out.piece_val[base + k * step] = u == carrier ? diag[t][k] : 1.0;
      } else {  // _factor_clause
        const int up = par[u];
        const size_t base = out.piece_val.size();
        out.piece_val.resize(base + ((size_t)1 << r), 0.0);
        for (int64_t combo = 0; combo < ((int64_t)1 << r); ++combo) {
          auto bit = [&](int q) { return (int)((combo >> (r - 1 - q)) & 1); };
          bool sat = false;
          int upbit = -1;
          for (int q = (own >= 0 ? 1 : 0); q < r; ++q) {
            const int w = nb[q - (own >= 0 ? 1 : 0)];
            if (w == up) upbit = bit(q);
            else sat = sat || bit(q) == 1;  // a child arc
          }
          if (own >= 0) sat = sat || bit(0) == pol[t][own];
          const bool ok = up >= 0 ? upbit == (sat ? 1 : 0) : sat;
          out.piece_val[base + combo] = ok ? 1.0 : 0.0;
        }
      }
      out.piece_val_off.push_back((int64_t)out.piece_val.size());
    }
  }
  for (int t = 0; t < T; ++t)
    if (isolated[t]) {
      piece_of_isolated[t] = npieces++;
      out.piece_src.push_back(t);
      out.piece_kind.push_back(0);
      out.piece_idx_off.push_back((int64_t)out.piece_idx.size());
      out.piece_val.insert(out.piece_val.end(), val(t), val(t) + size(t));
      out.piece_val_off.push_back((int64_t)out.piece_val.size());
    }

  tmark("pieces");
  // ---- Part 2: H (factoring.py:371-399) -----------------------------------
  const int NH = (int)hv_key.size();
  std::vector<std::vector<int>> hedges;  // endpoint pairs
  std::vector<int> hdeg(NH, 0);
  auto hedge = [&](int a, int b) {
    hedges.push_back({a, b});
    ++hdeg[a];
    ++hdeg[b];
  };
  for (int key = 0; key <= T; ++key)
    for (int u : S[key])
      for (int w : bd.adj[u])
        if (u < w && in_sub(key, w)) hedge(hv_id[hvk(key, u)], hv_id[hvk(key, w)]);
  for (int k = 0; k < in.num_leaf_map; ++k) {
    const int u = in.leaf_node[k], i = in.leaf_index[k];
    const int k0 = own0[i], k1 = own1[i] >= 0 ? own1[i] : Z;
    hedge(hv_id[hvk(k0, u)], hv_id[hvk(k1, u)]);
  }

  tmark("H");
  // ---- Part 3: carving of H through bd.tree (factoring.py:402-466) --------
  auto key_repr = [&](int key) { return key == Z ? std::string("'z'") : std::to_string(key); };
  std::vector<std::vector<int>> members(N);
  for (int h = 0; h < NH; ++h) members[hv_node[h]].push_back(h);
  for (int u = 0; u < N; ++u) {
    auto& m = members[u];
    if (m.size() < 2) continue;
    std::vector<std::pair<std::string, int>> keyed;
    for (int h : m) keyed.push_back({"(" + key_repr(hv_key[h]) + ", " + std::string(srepr[u]) + ")", h});
    std::sort(keyed.begin(), keyed.end());
    for (size_t q = 0; q < m.size(); ++q) m[q] = keyed[q].second;
  }
  // assignment[u][j]: H vertices at node u assigned to the arc to bd.adj[u][j]
  std::vector<std::vector<std::vector<int>>> assign(N);
  for (int u = 0; u < N; ++u) {
    const auto& nbr = bd.adj[u];
    assign[u].resize(nbr.size());
    if (nbr.empty()) continue;
    std::vector<int> arcs(nbr.size());  // positions into nbr, sorted by str of the neighbour
    for (size_t j = 0; j < nbr.size(); ++j) arcs[j] = (int)j;
    std::sort(arcs.begin(), arcs.end(), [&](int a, int b) { return str_less(nbr[a], nbr[b]); });
    std::vector<int> load(nbr.size(), 0);
    std::vector<std::string> arc_text(nbr.size());  // str(sorted(arc, key=str)): a list of nodes -> reprs
    for (size_t j = 0; j < nbr.size(); ++j) {
      const int lo = str_less(u, nbr[j]) ? u : nbr[j], hi = lo == u ? nbr[j] : u;
      arc_text[j] = "[" + std::string(srepr[lo]) + ", " + std::string(srepr[hi]) + "]";
    }
    auto allowed = [&](int h) {
      std::vector<int> own;
      const int key = hv_key[h];
      for (int w : sub_nbrs_sorted(key, u))
        for (size_t j = 0; j < nbr.size(); ++j)
          if (nbr[j] == w) own.push_back((int)j);
      return own.empty() ? arcs : own;
    };
    for (int h : members[u])
      if (hdeg[h] >= 3) {
        const auto al = allowed(h);
        int best = al[0];
        for (int j : al)
          if (load[j] < load[best] || (load[j] == load[best] && arc_text[j] < arc_text[best])) best = j;
        load[best]++;
        assign[u][best].push_back(h);
      }
    for (int h : members[u])
      if (hdeg[h] < 3) assign[u][allowed(h)[0]].push_back(h);
  }
  // s: hubs (one per bd node, same ids), then chains of x nodes with H leaves
  OGraph s;
  std::vector<std::string> label;
  int64_t counter = 0;
  for (int u = 0; u < N; ++u) {
    s.new_node();
    label.push_back("('hub', " + std::string(srepr[u]) + ")");
  }
  for (int u = 0; u < N; ++u) s.add_node(u);
  std::vector<int> leaf_hv;  // s node -> H vertex (-1: none)
  std::vector<char> mapped;
  auto fresh = [&](const char* prefix) {
    const int x = s.new_node();
    label.push_back(fresh_label(prefix, counter));
    return x;
  };
  std::vector<int> hleaves;  // in creation order (s_leaf_map order)
  bd.for_edges([&](int u, int v) {
    std::vector<int> chain{u};
    const int ju = (int)(std::find(bd.adj[u].begin(), bd.adj[u].end(), v) - bd.adj[u].begin());
    const int jv = (int)(std::find(bd.adj[v].begin(), bd.adj[v].end(), u) - bd.adj[v].begin());
    std::vector<int> seq = assign[u][ju];
    seq.insert(seq.end(), assign[v][jv].rbegin(), assign[v][jv].rend());
    for (int h : seq) {
      const int x = fresh("x");
      const int lf = fresh("hleaf");
      if ((int)leaf_hv.size() <= lf) leaf_hv.resize(lf + 1, -1);
      leaf_hv[lf] = h;
      hleaves.push_back(lf);
      s.add_edge(x, lf);
      chain.push_back(x);
    }
    chain.push_back(v);
    for (size_t q = 0; q + 1 < chain.size(); ++q) s.add_edge(chain[q], chain[q + 1]);
  });
  for (int u = 0; u < N; ++u)
    if (bd.degree(u) == 1) s.remove_node(u);
  leaf_hv.resize(s.adj.size(), -1);
  mapped.assign(s.adj.size(), 0);
  for (int lf : hleaves) mapped[lf] = 1;
  smooth(s, mapped);

  tmark("carving");
  // ---- width_carving(S, H) (decomposition.py:214-241) ---------------------
  {
    std::vector<int> s_of_hv(NH, -1);
    for (int lf : hleaves) s_of_hv[leaf_hv[lf]] = lf;
    std::vector<std::vector<int>> sets;
    sets.reserve(hedges.size());
    for (auto& e : hedges) sets.push_back({s_of_hv[e[0]], s_of_hv[e[1]]});
    const auto nodes = s.nodes();
    out.info.carving_width = nodes.size() > 1 ? max_split(s, nodes[0], sets) : 0;
  }

  tmark("width_carving");
  // ---- Part 5: free vertex, scalars, contraction tree (factoring.py:487-565)
  auto attach = [&](int lf) {  // _attach_leaf
    if (s.n_alive == 0) {
      s.add_node(lf);
      return;
    }
    if (s.n_alive == 1) {
      s.add_edge(s.nodes()[0], lf);
      return;
    }
    int bu = -1, bv = -1;
    const std::string *b1 = nullptr, *b2 = nullptr;
    s.for_edges([&](int u, int v) {
      const std::string* x = &label[u];
      const std::string* y = &label[v];
      if (*y < *x) std::swap(x, y);
      if (bu < 0 || *x < *b1 || (*x == *b1 && *y < *b2)) bu = u, bv = v, b1 = x, b2 = y;
    });
    const int mid = fresh("attach");
    s.remove_edge(bu, bv);
    s.add_edge(bu, mid);
    s.add_edge(mid, bv);
    s.add_edge(mid, lf);
  };
  std::vector<int> piece_of_s;  // s node -> piece (-1: none)
  int zleaf = -1;
  s.recopy();  // tree = s_tree.copy() (factoring.py:504)
  {
    std::vector<int> zl;
    for (int lf : hleaves)
      if (hv_key[leaf_hv[lf]] == Z) zl.push_back(lf);
    if (!zl.empty()) {
      int keep = zl[0];
      for (int lf : zl)
        if (label[lf] > label[keep]) keep = lf;
      for (int lf : zl)
        if (lf != keep) s.remove_node(lf);
      std::vector<char> m2(s.adj.size(), 0);
      for (int lf : hleaves)
        if (hv_key[leaf_hv[lf]] != Z) m2[lf] = 1;
      m2[keep] = 1;
      smooth(s, m2);
      zleaf = keep;
    } else {
      zleaf = fresh("zleaf");
      attach(zleaf);
    }
    piece_of_s.assign(s.adj.size(), -1);
    for (int lf : hleaves)
      if (hv_key[leaf_hv[lf]] != Z) piece_of_s[lf] = piece_of_hv[leaf_hv[lf]];
    for (int t = 0; t < T; ++t)
      if (isolated[t]) {
        const int sc = fresh("scalar");
        attach(sc);
        piece_of_s.resize(s.adj.size(), -1);
        piece_of_s[sc] = piece_of_isolated[t];
      }
    piece_of_s.resize(s.adj.size(), -1);
  }
  tmark("part5");
  // carving_to_contraction_tree (factoring.py:531-565) on cd.tree.copy()
  s.recopy();
  if (s.n_alive == 1) raise("PlanMismatch", "carving decomposition has no tensor leaves");
  const std::vector<int> zn = s.adj[zleaf];
  s.remove_node(zleaf);
  const int root = zn[0];
  std::vector<int> slot(s.adj.size(), -1);
  std::vector<char> used(npieces, 0);
  int next = npieces;
  struct Fr {
    int node, parent, state;
    int kids[2];
  };
  std::vector<Fr> st{{root, -1, 0, {-1, -1}}};
  while (!st.empty()) {
    Fr& f = st.back();
    if (f.state == 0) {
      int nk = 0;
      for (int w : s.adj[f.node])
        if (w != f.parent) {
          if (nk < 2) f.kids[nk] = w;
          ++nk;
        }
      if (nk == 0) {
        const int p = piece_of_s[f.node];
        if (p < 0) raise("PlanMismatch", "unmapped carving leaf " + label[f.node]);
        if (used[p]) raise("PlanMismatch", "carving leaves do not match the network's tensors");
        used[p] = 1;
        slot[f.node] = p;
        st.pop_back();
        continue;
      }
      if (nk != 2) raise("PlanMismatch", "carving node " + label[f.node] + " has " + std::to_string(nk) + " children");
      f.state = 1;
      const int c = f.kids[0], n0 = f.node;
      st.push_back({c, n0, 0, {-1, -1}});
    } else if (f.state == 1) {
      f.state = 2;
      const int c = f.kids[1], n0 = f.node;
      st.push_back({c, n0, 0, {-1, -1}});
    } else {
      out.left.push_back(slot[f.kids[0]]);
      out.right.push_back(slot[f.kids[1]]);
      slot[f.node] = next++;
      st.pop_back();
    }
  }
  for (int p = 0; p < npieces; ++p)
    if (!used[p]) raise("PlanMismatch", "carving leaves do not match the network's tensors");
  tmark("tree");
  out.info.num_pieces = npieces;
  out.info.num_bonds = (int)out.bond_ordinal.size();
  out.info.total_idx = (int64_t)out.piece_idx.size();
  out.info.total_val = (int64_t)out.piece_val.size();
  out.info.num_nodes = (int)out.left.size();
  out.info.root_slot = slot[root];
}

}  // namespace

extern "C" {

int tc_factor_branch(const tc_factor_input* in, tc_factor_result** out) {
  if (!out) return set_last_error(TC_BAD_ARG, "null output");
  *out = nullptr;
  if (!in) return set_last_error(TC_BAD_ARG, "null input");
  auto* r = new (std::nothrow) tc_factor_result;
  if (!r) return set_last_error(TC_OOM, "host out of memory");
  try {
    Factor f(*in, *r);
    f.run();
  } catch (const Error& e) {
    delete r;
    return set_last_error(e.status, e.msg);
  } catch (const std::bad_alloc&) {
    delete r;
    return set_last_error(TC_OOM, "host out of memory");
  } catch (const std::exception& e) {
    delete r;
    return set_last_error(TC_BAD_ARG, e.what());
  }
  *out = r;
  return TC_OK;
}

int tc_factor_info_get(const tc_factor_result* r, tc_factor_info* info) {
  if (!r || !info) return set_last_error(TC_BAD_ARG, "null argument");
  *info = r->info;
  return TC_OK;
}

int tc_factor_fetch(const tc_factor_result* r, int32_t* piece_src, int32_t* piece_kind, int64_t* piece_idx_off,
                    int32_t* piece_idx, int64_t* piece_val_off, double* piece_val, int32_t* bond_ordinal,
                    int32_t* bond_k, int32_t* bond_domain, int32_t* left, int32_t* right) {
  if (!r) return set_last_error(TC_BAD_ARG, "null result");
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(piece_src, r->piece_src);
  cp(piece_kind, r->piece_kind);
  cp(piece_idx_off, r->piece_idx_off);
  cp(piece_idx, r->piece_idx);
  cp(piece_val_off, r->piece_val_off);
  cp(piece_val, r->piece_val);
  cp(bond_ordinal, r->bond_ordinal);
  cp(bond_k, r->bond_k);
  cp(bond_domain, r->bond_domain);
  cp(left, r->left);
  cp(right, r->right);
  return TC_OK;
}

void tc_factor_free(tc_factor_result* r) { delete r; }

}  // extern "C"
