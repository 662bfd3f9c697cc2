"""Flatten a (TensorNetwork, ContractionTree) pair into the integer/float arrays
that cross the C-ABI (``include/tc.h``, ``tc_plan_desc``).

Works on the reference's objects (``tensorcount.network.TensorNetwork`` /
``ContractionTree`` / ``tensor.Tensor`` / ``Index``) and on this package's
mirror types alike: only ``n.tensors``, ``tensor.indices``, ``tensor.values``,
``index.id``, ``index.domain_size``, ``index.sort_key()``, ``node.is_leaf``,
``node.tensor``, ``node.left`` and ``node.right`` are read.

Slot numbering follows ``serialize_plan`` (reference ``network.py:235-258``):
leaves are numbered by network order, internal nodes continue the numbering in
postorder (left subtree, right subtree, node; ``network.py:114-124``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class FlatPlan:
    indices: list            # Index objects, position = dense id
    domain: np.ndarray       # int32[I]
    sort_rank: np.ndarray    # int32[I], rank of Index.sort_key() (tie-break order)
    leaf_idx_off: np.ndarray  # int64[L+1]
    leaf_idx: np.ndarray     # int32[sum rank]  (row-major order: first index slowest)
    leaf_val_off: np.ndarray  # int64[L+1]
    leaf_val: np.ndarray     # float64[sum size], C-contiguous per leaf
    left: np.ndarray         # int32[NN]  operand slots of internal node k (postorder)
    right: np.ndarray        # int32[NN]
    root_slot: int           # slot of the root (a leaf slot when NN == 0)

    @property
    def num_leaves(self):
        return len(self.leaf_idx_off) - 1

    @property
    def num_nodes(self):
        return len(self.left)


def _postorder_internal(t):
    """Internal nodes in reference postorder, iteratively (deep spines)."""
    out = []
    stack = [t]
    while stack:
        node = stack.pop()
        out.append(node)
        if not node.is_leaf:
            stack.append(node.left)
            stack.append(node.right)
    out.reverse()
    return out


def flatten(n, t, index_table=None) -> FlatPlan:
    tensors = list(n.tensors)
    leaf_slot = {}
    for k, ten in enumerate(tensors):
        leaf_slot[id(ten)] = k

    # dense index ids in order of first appearance over the network
    if index_table is None:
        index_table = {}
    indices = []
    idx_list = []
    idx_off = [0]
    val_chunks = []
    val_off = [0]
    for ten in tensors:
        for ix in ten.indices:
            d = index_table.get(ix)
            if d is None:
                d = len(index_table)
                index_table[ix] = d
                indices.append(ix)
            idx_list.append(d)
        idx_off.append(len(idx_list))
        v = np.ascontiguousarray(np.asarray(ten.values, dtype=np.float64)).reshape(-1)
        val_chunks.append(v)
        val_off.append(val_off[-1] + v.size)
    if len(indices) != len(index_table):
        # caller-supplied table: rebuild the position list
        indices = [None] * len(index_table)
        for ix, d in index_table.items():
            indices[d] = ix
    domain = np.array([ix.domain_size for ix in indices], dtype=np.int32)
    order = sorted(range(len(indices)), key=lambda d: indices[d].sort_key())
    sort_rank = np.empty(len(indices), dtype=np.int32)
    sort_rank[order] = np.arange(len(indices), dtype=np.int32)

    nodes = _postorder_internal(t)
    slot_of = {}
    left, right = [], []
    nl = len(tensors)
    nxt = nl
    for node in nodes:
        if node.is_leaf:
            s = leaf_slot.get(id(node.tensor))
            if s is None:
                s = -1  # not a network tensor: reported as PlanMismatch by the caller
            slot_of[id(node)] = s
        else:
            left.append(slot_of[id(node.left)])
            right.append(slot_of[id(node.right)])
            slot_of[id(node)] = nxt
            nxt += 1
    return FlatPlan(
        indices=indices,
        domain=domain,
        sort_rank=sort_rank,
        leaf_idx_off=np.array(idx_off, dtype=np.int64),
        leaf_idx=np.array(idx_list, dtype=np.int32),
        leaf_val_off=np.array(val_off, dtype=np.int64),
        leaf_val=np.concatenate(val_chunks) if val_chunks else np.zeros(0),
        left=np.array(left, dtype=np.int32),
        right=np.array(right, dtype=np.int32),
        root_slot=slot_of[id(t)],
    )
