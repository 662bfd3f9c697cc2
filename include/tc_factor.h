/*
 * tc_factor.h — C-ABI of the native FactorTree step (host only, in libtc.so).
 *
 * Replaces the reference's pure-Python construction of the executable plan
 * (M, T) from a branch decomposition:
 *   factor_branch_audit   pkg/src/tensorcount/factoring.py:270-333
 *     _spanning_subtree       factoring.py:86-101
 *     detect_kind / _diagonal_values / _clause_polarities  factoring.py:105-144
 *     _fresh_bonds / _piece_indices / _factor_copy / _factor_clause  :176-251
 *     _build_h                factoring.py:371-399
 *     _build_carving_of_h     factoring.py:402-466 (+ _smooth_carving :469-484)
 *     _attach_leaf / _to_network_carving  factoring.py:487-528
 *     carving_to_contraction_tree  factoring.py:531-565
 *   width_branch / width_carving   decomposition.py:166-191, 214-241
 *   validate_branch_decomposition  decomposition.py:81-86, 111-134
 * The output is the reference's (M, T) exactly: the same pieces (indices,
 * bond ids, values) in the same network order and the same tree shape with
 * the same left/right children, so serialize_plan(M, T) is identical and the
 * counts are bit-identical.  Every order the reference takes from networkx
 * (node / adjacency insertion order, EdgeView order) or from str()/repr() of
 * decomposition-tree node labels is reproduced: the caller passes the tree in
 * networkx order and the str / repr text of every node.
 *
 * Errors: TC_BAD_ARG with tc_last_error() starting "InvalidDecomposition: ",
 * "NotFactorable: " or "PlanMismatch: " (the reference exception to raise).
 */
#ifndef TC_FACTOR_H_
#define TC_FACTOR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_factor_input {
  /* the network n: tensors in network order, index ids dense 0..num_indices-1 */
  int32_t num_tensors;
  const int64_t* idx_off;   /* [num_tensors+1]                               */
  const int32_t* idx;       /* index ids per tensor, row-major order          */
  const int64_t* val_off;   /* [num_tensors+1] cumulative entry counts        */
  const double* const* val_ptr; /* [num_tensors] FP64 values of each tensor,
                               C-contiguous, read in place (the reduction's
                               dense 2^occ copy tensors are not copied)        */
  int32_t num_indices;
  const int32_t* domain;    /* [num_indices]                                  */
  const int32_t* sort_rank; /* [num_indices] rank of Index.sort_key()         */
  /* the branch decomposition bd: bd.tree in networkx order */
  int32_t num_nodes;
  const int64_t* adj_off;   /* [num_nodes+1]                                  */
  const int32_t* adj;       /* neighbours in adjacency insertion order        */
  const int64_t* str_off;   /* [num_nodes+1] into str_buf: str(node)          */
  const char* str_buf;
  const int64_t* repr_off;  /* [num_nodes+1] into repr_buf: repr(node)        */
  const char* repr_buf;
  int32_t num_leaf_map;     /* bd.leaf_map entries in dict order              */
  const int32_t* leaf_node; /* [num_leaf_map] tree node                       */
  const int32_t* leaf_index;/* [num_leaf_map] index id                        */
} tc_factor_input;

typedef struct tc_factor_result tc_factor_result;

typedef struct tc_factor_info {
  int32_t trivial;        /* 1: width 0, the caller builds the trivial plan (factoring.py:336-370) */
  int32_t branch_width;
  int32_t carving_width;
  int32_t num_pieces;     /* M's tensors */
  int32_t num_bonds;      /* fresh bond indices (("b", ordinal), k) */
  int64_t total_idx;      /* sum of piece ranks */
  int64_t total_val;      /* sum of piece sizes */
  int32_t num_nodes;      /* internal nodes of T (= num_pieces - 1) */
  int32_t root_slot;
} tc_factor_info;

/* Build (M, T).  *out is NULL on error. */
int tc_factor_branch(const tc_factor_input* in, tc_factor_result** out);
int tc_factor_info_get(const tc_factor_result* r, tc_factor_info* info);
/* piece_src[p]: network ordinal of the tensor piece p comes from;
 * piece_kind[p]: 0 the original tensor object itself, 1 copy piece, 2 clause piece;
 * piece_idx_off/piece_idx: index references, >= 0 an input index id, < 0 bond -1-b;
 * piece_val_off/piece_val: FP64 values (row-major); bond_ordinal/bond_k/bond_domain;
 * left/right: T in postorder (slots as serialize_plan: pieces then internal nodes). */
int tc_factor_fetch(const tc_factor_result* r, int32_t* piece_src, int32_t* piece_kind, int64_t* piece_idx_off,
                    int32_t* piece_idx, int64_t* piece_val_off, double* piece_val, int32_t* bond_ordinal,
                    int32_t* bond_k, int32_t* bond_domain, int32_t* left, int32_t* right);
void tc_factor_free(tc_factor_result* r);

#ifdef __cplusplus
}
#endif

#endif /* TC_FACTOR_H_ */
