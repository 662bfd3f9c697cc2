// networkx.Graph semantics with insertion order, for the host-side planning
// restatements (factor.cpp, decompose.cpp).  The reference's plans depend on
// networkx's orders: node dict and adjacency dicts in insertion order,
// EdgeView yielding (u, v) once with u the earlier node, Graph.copy()
// re-inserting every adjacency pair.
#pragma once
#include <algorithm>
#include <vector>

namespace tc {

struct OGraph {
  std::vector<std::vector<int>> adj;  // live neighbours, insertion order
  std::vector<char> alive;
  std::vector<int> order;  // nodes in insertion order (removed ones skipped)
  int n_alive = 0;
  int new_node() {
    const int u = (int)adj.size();
    adj.emplace_back();
    alive.push_back(0);
    return u;
  }
  void add_node(int u) {
    if (!alive[u]) {
      alive[u] = 1;
      order.push_back(u);
      ++n_alive;
    }
  }
  bool has_edge(int u, int v) const { return std::find(adj[u].begin(), adj[u].end(), v) != adj[u].end(); }
  void add_edge(int u, int v) {
    add_node(u);
    add_node(v);
    if (has_edge(u, v)) return;
    adj[u].push_back(v);
    adj[v].push_back(u);
  }
  static void erase(std::vector<int>& a, int v) {
    auto it = std::find(a.begin(), a.end(), v);
    if (it != a.end()) a.erase(it);
  }
  void remove_edge(int u, int v) {
    erase(adj[u], v);
    erase(adj[v], u);
  }
  void remove_node(int u) {
    for (int w : adj[u]) erase(adj[w], u);
    adj[u].clear();
    alive[u] = 0;
    --n_alive;
  }
  int degree(int u) const { return (int)adj[u].size(); }
  std::vector<int> nodes() const {
    std::vector<int> o;
    o.reserve(n_alive);
    for (int u : order)
      if (alive[u]) o.push_back(u);
    return o;
  }
  // Graph.copy(): nodes in order, then add_edges_from over every (u, v) of
  // the adjacency in order -- which re-inserts the neighbour lists (a node's
  // earlier-listed neighbours come first in the copy)
  void recopy() {
    std::vector<std::vector<int>> na(adj.size());
    order = nodes();
    for (int u : order)
      for (int v : adj[u]) {
        if (std::find(na[u].begin(), na[u].end(), v) == na[u].end()) na[u].push_back(v);
        if (std::find(na[v].begin(), na[v].end(), u) == na[v].end()) na[v].push_back(u);
      }
    adj.swap(na);
  }
  template <class F>
  void for_edges(F f) const {  // EdgeView order
    std::vector<char> seen(adj.size(), 0);
    for (int u : order) {
      if (!alive[u]) continue;
      for (int w : adj[u])
        if (!seen[w]) f(u, w);
      seen[u] = 1;
    }
  }
};

// _smooth_carving (factoring.py:469-484) / _prune_and_smooth (decomposition.py:
// 395-411): drop unmapped
// leaves, suppress unmapped degree-2 nodes, until nothing changes.
inline void smooth(OGraph& t, const std::vector<char>& mapped) {
  for (bool changed = true; changed;) {
    changed = false;
    for (int u : t.nodes()) {
      if (u < (int)mapped.size() && mapped[u]) continue;
      const int deg = t.degree(u);
      if (deg <= 1 && t.n_alive > 1) {
        t.remove_node(u);
        changed = true;
      } else if (deg == 2) {
        const int a = t.adj[u][0], b = t.adj[u][1];
        t.remove_node(u);
        t.add_edge(a, b);
        changed = true;
      }
    }
  }
}

}  // namespace tc
