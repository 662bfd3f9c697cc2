"""Flatten a (TensorNetwork, ContractionTree) pair into the integer/float arrays
that cross the C-ABI (``include/tc.h``, ``tc_plan_desc``).

Works on the reference's objects (``tensorcount.network.TensorNetwork`` /
``ContractionTree`` / ``tensor.Tensor`` / ``Index``) and on this package's
mirror types alike: only ``n.tensors``, ``tensor.indices``, ``tensor.values``,
``index.id``, ``index.domain_size``, ``index.sort_key()``, ``node.tensor``,
``node.left`` and ``node.right`` are read.

Slot numbering follows ``serialize_plan`` (reference ``network.py:235-258``):
leaves are numbered by network order, internal nodes continue the numbering in
postorder (left subtree, right subtree, node; ``network.py:114-124``).

This runs on every call of the public API, so the work is done by a small
CPython C extension (``csrc/flatten_ext.c`` -> ``lib/_tcflat*.so``); the
pure-Python ``flatten_py`` below is its specification.  In both, index
identity is keyed on ``Index.id`` (the reference's equality, ``tensor.py:29-33``),
values are gathered with one ``np.concatenate``, and ``sort_key`` ranks (only
needed by the greedy slice chooser) can be skipped.
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


def sort_ranks(indices) -> np.ndarray:
    order = sorted(range(len(indices)), key=lambda d: indices[d].sort_key())
    r = np.empty(len(indices), dtype=np.int32)
    r[order] = np.arange(len(indices), dtype=np.int32)
    return r


def _native():
    """The C flattener (csrc/flatten_ext.c, built in-tree by build.py), or None."""
    global _NATIVE
    if _NATIVE is False:
        import importlib.util
        import os

        from .build import flat_ext_path

        path = flat_ext_path()
        _NATIVE = None
        if os.path.exists(path):
            spec = importlib.util.spec_from_file_location("_tcflat", path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            _NATIVE = mod
    return _NATIVE


_NATIVE = False


def flatten(n, t, with_sort_rank: bool = True) -> FlatPlan:
    nat = _native()
    if nat is not None:
        indices, dom, ioff, iarr, voff, vals, lft, rgt, root = nat.flatten(n.tensors, t)
        return FlatPlan(
            indices=indices,
            domain=np.frombuffer(dom, dtype=np.int32),
            sort_rank=sort_ranks(indices) if with_sort_rank else np.arange(len(indices), dtype=np.int32),
            leaf_idx_off=np.frombuffer(ioff, dtype=np.int64),
            leaf_idx=np.frombuffer(iarr, dtype=np.int32),
            leaf_val_off=np.frombuffer(voff, dtype=np.int64),
            leaf_val=np.frombuffer(vals, dtype=np.float64),
            left=np.frombuffer(lft, dtype=np.int32),
            right=np.frombuffer(rgt, dtype=np.int32),
            root_slot=int(root),
        )
    return flatten_py(n, t, with_sort_rank)


def flatten_py(n, t, with_sort_rank: bool = True) -> FlatPlan:
    """Pure-Python flattener (same output as the native one; fallback when
    the host extension is not built, and its cross-check in the tests)."""
    tensors = n.tensors
    nl = len(tensors)
    pos = {}
    indices = []
    idx_list = []
    ranks = np.empty(nl, dtype=np.int64)
    vals = []
    leaf_slot = {}
    for k, ten in enumerate(tensors):
        leaf_slot[id(ten)] = k
        inds = ten.indices
        ranks[k] = len(inds)
        for ix in inds:
            d = pos.get(ix.id)
            if d is None:
                d = pos[ix.id] = len(indices)
                indices.append(ix)
            idx_list.append(d)
        vals.append(ten.values)
    flat_vals = [np.ravel(v) for v in vals]
    sizes = np.fromiter((v.size for v in flat_vals), dtype=np.int64, count=nl)
    idx_off = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(ranks, out=idx_off[1:])
    val_off = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(sizes, out=val_off[1:])
    leaf_val = np.concatenate(flat_vals).astype(np.float64, copy=False) if flat_vals else np.zeros(0)
    domain = np.fromiter((ix.domain_size for ix in indices), dtype=np.int32, count=len(indices))
    sort_rank = sort_ranks(indices) if with_sort_rank else np.arange(len(indices), dtype=np.int32)

    # internal nodes in reference postorder, iteratively (deep spines)
    left, right = [], []
    slot_of = {}
    nxt = nl
    stack = [t]
    seq = []
    while stack:
        node = stack.pop()
        seq.append(node)
        if node.tensor is None:
            stack.append(node.left)
            stack.append(node.right)
    for node in reversed(seq):
        if node.tensor is not None:
            slot_of[id(node)] = leaf_slot.get(id(node.tensor), -1)
        else:
            left.append(slot_of[id(node.left)])
            right.append(slot_of[id(node.right)])
            slot_of[id(node)] = nxt
            nxt += 1
    return FlatPlan(
        indices=indices,
        domain=domain,
        sort_rank=sort_rank,
        leaf_idx_off=idx_off,
        leaf_idx=np.array(idx_list, dtype=np.int32),
        leaf_val_off=val_off,
        leaf_val=leaf_val,
        left=np.array(left, dtype=np.int32),
        right=np.array(right, dtype=np.int32),
        root_slot=slot_of[id(t)],
    )
