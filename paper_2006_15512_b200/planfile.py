"""``.tcplan`` — the plan + leaf interchange format.

One compressed ``.npz`` holding exactly what crosses the C-ABI
(``flatten.FlatPlan``) plus the index ids (``repr``, restored with
``ast.literal_eval``) and a JSON metadata blob (generator, reference count,
planning time ...).  The internal-node list is the reference's
``serialize_plan`` text (``network.py:235-258``) in array form, so a plan made
once by the CPU planner is executed bit-for-bit identically by the reference
arm and by the B200 arm.
"""

from __future__ import annotations

import ast
import json

import numpy as np

from .flatten import FlatPlan


def save(path, flat: FlatPlan, meta: dict | None = None):
    ids = json.dumps([repr(ix.id) for ix in flat.indices])
    np.savez_compressed(
        path,
        domain=flat.domain,
        sort_rank=flat.sort_rank,
        leaf_idx_off=flat.leaf_idx_off,
        leaf_idx=flat.leaf_idx,
        leaf_val_off=flat.leaf_val_off,
        leaf_val=flat.leaf_val,
        left=flat.left,
        right=flat.right,
        root_slot=np.array([flat.root_slot], dtype=np.int64),
        ids=np.frombuffer(ids.encode(), dtype=np.uint8),
        meta=np.frombuffer(json.dumps(meta or {}).encode(), dtype=np.uint8),
    )


def load(path, index_cls=None):
    """Return (FlatPlan, meta).  ``index_cls`` builds the Index objects
    (default: this package's ``tensor.Index``)."""
    if index_cls is None:
        from .tensor import Index as index_cls
    z = np.load(path, allow_pickle=False)
    ids = [ast.literal_eval(s) for s in json.loads(bytes(z["ids"]).decode())]
    domain = z["domain"].astype(np.int32)
    indices = [index_cls(i, int(d)) for i, d in zip(ids, domain)]
    flat = FlatPlan(
        indices=indices,
        domain=domain,
        sort_rank=z["sort_rank"].astype(np.int32),
        leaf_idx_off=z["leaf_idx_off"].astype(np.int64),
        leaf_idx=z["leaf_idx"].astype(np.int32),
        leaf_val_off=z["leaf_val_off"].astype(np.int64),
        leaf_val=z["leaf_val"].astype(np.float64),
        left=z["left"].astype(np.int32),
        right=z["right"].astype(np.int32),
        root_slot=int(z["root_slot"][0]),
    )
    meta = json.loads(bytes(z["meta"]).decode())
    return flat, meta


def to_objects(flat: FlatPlan, tensor_cls=None, network_cls=None, tree_cls=None):
    """Rebuild (network, tree) objects — this package's mirror types by
    default, or the reference's classes when passed (the CPU reference arm)."""
    if tensor_cls is None:
        from .tensor import Tensor as tensor_cls
    if network_cls is None:
        from .network import TensorNetwork as network_cls
    if tree_cls is None:
        from .network import ContractionTree as tree_cls
    tensors = []
    for k in range(flat.num_leaves):
        inds = tuple(flat.indices[d] for d in flat.leaf_idx[flat.leaf_idx_off[k]:flat.leaf_idx_off[k + 1]])
        vals = flat.leaf_val[flat.leaf_val_off[k]:flat.leaf_val_off[k + 1]]
        tensors.append(tensor_cls(inds, vals.copy()))
    n = network_cls(tuple(tensors))
    nodes = [tree_cls(tensor=t) for t in n.tensors]
    for l, r in zip(flat.left.tolist(), flat.right.tolist()):
        nodes.append(tree_cls(left=nodes[l], right=nodes[r]))
    return n, nodes[flat.root_slot]
