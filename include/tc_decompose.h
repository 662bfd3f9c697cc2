/*
 * tc_decompose.h — C-ABI of the native planning heuristics (host only, in libtc.so).
 *
 * Replaces the reference's pure-Python decomposition builders:
 *   _heuristic_order          pkg/src/tensorcount/decomposition.py:301-319
 *     _fill_in / _degree      decomposition.py:322-332 (min-fill / min-degree scores)
 *   _eliminate                decomposition.py:244-255
 *   _elimination_tree_decomposition  decomposition.py:258-275
 *   binarize_tree_decomposition      decomposition.py:278-294
 *   tree_to_branch (+ _prune_and_smooth)  decomposition.py:346-411
 *   validate_tree_decomposition      decomposition.py:81-108
 * with the reference's exact output: the same elimination order (ties broken
 * by the same Mersenne-Twister draws as random.Random(seed).choice, the
 * caller passes the generator state), the same bags, the same decomposition
 * trees with networkx node / adjacency order, and fresh node names numbered
 * as fresh_node does (decomposition.py:23-26) from a caller-supplied counter.
 */
#ifndef TC_DECOMPOSE_H_
#define TC_DECOMPOSE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_decomp_result tc_decomp_result;

/* Elimination order + tree decomposition (+ binarization) of a simple graph.
 * Vertices are 0..nv-1 in sorted(str) order (the reference's `remaining`);
 * adj: neighbour ids (parallel edges collapsed).  score: 0 min-fill, 1 min-degree.
 * mt_state: 624 words + index of random.Random(seed).getstate().
 * Fresh tree nodes are numbered counter_start, counter_start+1, ... */
int tc_elim_td(int32_t nv, const int64_t* adj_off, const int32_t* adj, int32_t score, const uint32_t* mt_state,
               int32_t mt_index, int64_t counter_start, tc_decomp_result** out);

/* tree_to_branch.  The tree decomposition: td nodes 0..nn-1 in networkx order
 * with adjacency lists; node_rank[k]: position of node k in sorted(td.tree.nodes,
 * key=str); bags (CSR of vertex ids).  Graph edges in sorted(g.edges, key=str)
 * order with their two endpoints.  status TC_BAD_ARG with tc_last_error()
 * "NoHostBag: <edge position>" when an edge has no host bag. */
int tc_tree_to_branch(int32_t nn, const int64_t* adj_off, const int32_t* adj, const int32_t* node_rank,
                      const int64_t* bag_off, const int32_t* bag, int32_t nv, int32_t ne, const int32_t* edge_u,
                      const int32_t* edge_v, int64_t counter_start, tc_decomp_result** out);

/* The structural checks of validate_tree_decomposition (decomposition.py:81-108)
 * that cost O(|E| x |bags|) in Python: the tree shape, a host bag for every
 * edge, and connected bags per vertex.  Vertex ids >= nv are vertices outside
 * the graph.  Results: *shape 0 ok, 1 empty tree, 2 not a tree; *bad_edge the
 * first edge (in the given order) without a host bag or -1; disconnected[v] = 1
 * for every vertex whose bags are disconnected. */
int tc_validate_td(int32_t nn, const int64_t* adj_off, const int32_t* adj, const int64_t* bag_off,
                   const int32_t* bag, int32_t nv, int32_t ne, const int32_t* edge_u, const int32_t* edge_v,
                   int32_t* shape, int32_t* bad_edge, int8_t* disconnected);

typedef struct tc_decomp_info {
  int32_t num_nodes;       /* tree nodes (networkx order)                       */
  int64_t num_adj;         /* total adjacency entries                            */
  int64_t num_bag;         /* total bag entries (tree decompositions)            */
  int32_t num_order;       /* elimination order length (tc_elim_td)              */
  int32_t num_leaf_map;    /* leaf_map entries (tc_tree_to_branch)               */
  int64_t counter_end;     /* next fresh-name number                             */
} tc_decomp_info;

int tc_decomp_info_get(const tc_decomp_result* r, tc_decomp_info* info);
/* node_kind[k]: 0 ("td", n), 1 ("bd", n), 2 ("bdleaf", n); node_num[k]: n.
 * adj_off/adj: adjacency in insertion order; bag_off/bag: vertex ids per node;
 * order: elimination order; leaf_node/leaf_edge: leaf_map in insertion order. */
int tc_decomp_fetch(const tc_decomp_result* r, int32_t* node_kind, int64_t* node_num, int64_t* adj_off, int32_t* adj,
                    int64_t* bag_off, int32_t* bag, int32_t* order, int32_t* leaf_node, int32_t* leaf_edge);
void tc_decomp_free(tc_decomp_result* r);

#ifdef __cplusplus
}
#endif

#endif /* TC_DECOMPOSE_H_ */
