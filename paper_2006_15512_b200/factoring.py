"""FactorTree: the executable plan (M, T) from a branch decomposition, native.

Drop-in for the reference's ``factor_branch_audit`` / ``factor_branch``
(``pkg/src/tensorcount/factoring.py:263-333``), the planning step right before
the execution path.  Every tensor is split into rank-<=3
pieces along its spanning subtree of the branch decomposition, the piece graph
H is threaded through the decomposition tree as a carving decomposition and
read as a contraction tree.  The construction runs in C++ (``csrc/factor.cpp``,
C-ABI ``include/tc_factor.h``) and returns exactly the reference's result: the
same pieces (indices, fresh bond ids ``(("b", ordinal), k)``, values) in the
same order and the same tree with the same left / right children, so
``serialize_plan(M, T)`` and every count are identical.

Python only moves the objects across: the network's index table, the
decomposition tree in networkx order with the ``str`` / ``repr`` text of every
node (the reference sorts by them), and back the pieces and the tree.  Inputs
may be the reference's objects or this package's; results use the caller's
classes.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidDecomposition, NotFactorable, PlanMismatch, TooManyFreeIndices
from .flatten import _native, flatten_py, sort_ranks

_ERRORS = {"InvalidDecomposition": InvalidDecomposition, "NotFactorable": NotFactorable,
           "PlanMismatch": PlanMismatch, "ValueError": ValueError}


@dataclass
class FactorBranchResult:
    """Mirror of the reference's dataclass (``factoring.py:254-260``)."""

    network: object
    tree: object
    branch_width: int
    carving_width: int  # -1 for the trivial (width-0) plan
    piece_map: dict     # id(piece) -> original tensor


def _classes(n, tree_cls):
    tensor_cls = type(n.tensors[0])
    network_cls = type(n)
    if tree_cls is None:
        tree_cls = getattr(sys.modules.get(network_cls.__module__), "ContractionTree", None)
        if tree_cls is None:
            from .network import ContractionTree as tree_cls
    index_cls = None
    for t in n.tensors:
        if t.indices:
            index_cls = type(t.indices[0])
            break
    return tensor_cls, network_cls, tree_cls, index_cls


def _left_deep(tree_cls, tensors):
    node = tree_cls(tensor=tensors[0])
    for t in tensors[1:]:
        node = tree_cls(left=node, right=tree_cls(tensor=t))
    return node


def _trivial_plan(n, tree_cls, w):
    """Width-0 / edge-free networks: one left-deep tree per connected
    component (components in network order, members in the reference's
    depth-first order, ``factoring.py:336-370``), joined left to right."""
    nbrs = {id(t): set() for t in n.tensors}
    first = {}
    for t in n.tensors:
        for ix in t.indices:
            o = first.get(ix)
            if o is None:
                first[ix] = id(t)
            else:
                nbrs[id(t)].add(o)
                nbrs[o].add(id(t))
    obj = {id(t): t for t in n.tensors}
    seen = set()
    root = None
    for t in n.tensors:
        if id(t) in seen:
            continue
        seen.add(id(t))
        todo, comp = [id(t)], []
        while todo:
            u = todo.pop()
            comp.append(obj[u])
            for v in nbrs[u]:
                if v not in seen:
                    seen.add(v)
                    todo.append(v)
        sub = _left_deep(tree_cls, comp)
        root = sub if root is None else tree_cls(left=root, right=sub)
    return FactorBranchResult(n, root, w, -1, {id(t): t for t in n.tensors})


def _text_table(items):
    parts = [s.encode("utf-8") for s in items]
    off = np.zeros(len(parts) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in parts], out=off[1:])
    return off, b"".join(parts)


def factor_branch_audit(n, bd, g=None, tree_cls=None) -> FactorBranchResult:
    """(M, T, branch width, carving width, piece map) exactly as the reference."""
    t0 = time.perf_counter()
    tensor_cls, network_cls, tree_cls, index_cls = _classes(n, tree_cls)
    if len(n.free_indices) > 3:
        raise TooManyFreeIndices(f"{len(n.free_indices)} free indices, at most 3 allowed")
    has_edges = bool(g.edges) if g is not None else any(t.indices for t in n.tensors)
    if not has_edges:
        return _trivial_plan(n, tree_cls, 0)

    # the network's index table (first appearance order) and the address of
    # every tensor's values (read in place: the reduction's copy tensors are
    # dense 2^occ arrays, reduction.py:32-39)
    nat = _native()
    probe = tree_cls(tensor=n.tensors[0])
    if nat is not None:
        indices, dom, ioff, iarr, voff, vptr, _, _, _, keepalive = nat.flatten(n.tensors, probe, True)
        domain = np.frombuffer(dom, dtype=np.int32)
        idx_off = np.frombuffer(ioff, dtype=np.int64)
        idx = np.frombuffer(iarr, dtype=np.int32)
        val_off = np.frombuffer(voff, dtype=np.int64)
        val_ptr = np.frombuffer(vptr, dtype=np.uint64)
    else:
        fl = flatten_py(n, probe, with_sort_rank=False)
        indices, domain, idx_off, idx = fl.indices, fl.domain, fl.leaf_idx_off, fl.leaf_idx
        keepalive = [np.ascontiguousarray(t.values, dtype=np.float64) for t in n.tensors]
        val_off = np.zeros(len(keepalive) + 1, dtype=np.int64)
        np.cumsum([a.size for a in keepalive], out=val_off[1:])
        val_ptr = np.array([a.ctypes.data for a in keepalive], dtype=np.uint64)
    srank = sort_ranks(indices)
    ipos = {ix: k for k, ix in enumerate(indices)}

    # the decomposition tree in networkx order, node texts for the str sorts
    tree = bd.tree
    nodes = list(tree.nodes)
    npos = {u: k for k, u in enumerate(nodes)}
    adj_lists = [[npos[w] for w in tree.adj[u]] for u in nodes]
    adj_off = np.zeros(len(nodes) + 1, dtype=np.int64)
    np.cumsum([len(a) for a in adj_lists], out=adj_off[1:])
    adj = np.fromiter((w for a in adj_lists for w in a), dtype=np.int32, count=int(adj_off[-1]))
    str_off, str_buf = _text_table(str(u) for u in nodes)
    repr_off, repr_buf = _text_table(repr(u) for u in nodes)
    lm_node, lm_index = [], []
    for u, e in bd.leaf_map.items():
        if u not in npos or e not in ipos:
            raise InvalidDecomposition("branch decomposition: leaves are not a bijection onto the target set")
        lm_node.append(npos[u])
        lm_index.append(ipos[e])
    lm_node = np.asarray(lm_node, dtype=np.int32)
    lm_index = np.asarray(lm_index, dtype=np.int32)

    arrays = [domain, srank, idx_off, idx, val_off, val_ptr, adj_off, adj, str_off, repr_off, lm_node, lm_index]
    domain, srank, idx_off, idx, val_off, val_ptr, adj_off, adj, str_off, repr_off, lm_node, lm_index = (
        np.ascontiguousarray(a) for a in arrays)
    p = _lib._p
    fin = _lib.FactorInput(
        num_tensors=len(n.tensors), idx_off=p(idx_off, _lib.I64P), idx=p(idx, _lib.I32P),
        val_off=p(val_off, _lib.I64P), val_ptr=p(val_ptr, C.POINTER(C.c_void_p)), num_indices=len(indices),
        domain=p(domain, _lib.I32P), sort_rank=p(srank, _lib.I32P), num_nodes=len(nodes),
        adj_off=p(adj_off, _lib.I64P), adj=p(adj, _lib.I32P), str_off=p(str_off, _lib.I64P), str_buf=str_buf,
        repr_off=p(repr_off, _lib.I64P), repr_buf=repr_buf, num_leaf_map=len(lm_node),
        leaf_node=p(lm_node, _lib.I32P), leaf_index=p(lm_index, _lib.I32P))
    L = _lib.lib()
    h = C.c_void_p()
    t_in = time.perf_counter()
    st = L.tc_factor_branch(C.byref(fin), C.byref(h))
    t_native = time.perf_counter()
    del keepalive
    if st != 0:
        msg = L.tc_last_error().decode(errors="replace")
        kind, _, text = msg.partition(": ")
        if kind in _ERRORS:
            raise _ERRORS[kind](text)
        _lib.check(st)
    try:
        info = _lib.FactorInfo()
        _lib.check(L.tc_factor_info_get(h, C.byref(info)))
        if info.trivial:
            return _trivial_plan(n, tree_cls, 0)
        P, B = info.num_pieces, info.num_bonds
        src = np.empty(P, np.int32)
        kind = np.empty(P, np.int32)
        ioff = np.empty(P + 1, np.int64)
        pidx = np.empty(max(1, info.total_idx), np.int32)
        voff = np.empty(P + 1, np.int64)
        pval = np.empty(max(1, info.total_val), np.float64)
        b_ord = np.empty(max(1, B), np.int32)
        b_k = np.empty(max(1, B), np.int32)
        b_dom = np.empty(max(1, B), np.int32)
        left = np.empty(max(1, info.num_nodes), np.int32)
        right = np.empty(max(1, info.num_nodes), np.int32)
        _lib.check(L.tc_factor_fetch(h, p(src, _lib.I32P), p(kind, _lib.I32P), p(ioff, _lib.I64P),
                                     p(pidx, _lib.I32P), p(voff, _lib.I64P), p(pval, _lib.F64P),
                                     p(b_ord, _lib.I32P), p(b_k, _lib.I32P), p(b_dom, _lib.I32P),
                                     p(left, _lib.I32P), p(right, _lib.I32P)))
    finally:
        L.tc_factor_free(h)

    bonds = [index_cls((("b", o), k), d) for o, k, d in zip(b_ord[:B].tolist(), b_k[:B].tolist(),
                                                            b_dom[:B].tolist())]
    ts = n.tensors
    ioff_l, voff_l, pidx_l = ioff.tolist(), voff.tolist(), pidx.tolist()
    pieces = []
    for q, (s, k) in enumerate(zip(src.tolist(), kind.tolist())):
        if k == 0:
            pieces.append(ts[s])
            continue
        inds = tuple(indices[i] if i >= 0 else bonds[-1 - i] for i in pidx_l[ioff_l[q]:ioff_l[q + 1]])
        pieces.append(tensor_cls(inds, pval[voff_l[q]:voff_l[q + 1]]))
    m = network_cls(tuple(pieces))
    tnodes = [tree_cls(tensor=t) for t in pieces]
    for a, b in zip(left[:info.num_nodes].tolist(), right[:info.num_nodes].tolist()):
        tnodes.append(tree_cls(left=tnodes[a], right=tnodes[b]))
    piece_map = {id(pc): ts[s] for pc, s in zip(pieces, src.tolist())}
    if os.environ.get("TC_FACTOR_TIMING"):  # diagnostics
        t1 = time.perf_counter()
        print(f"[factor] inputs {1e3 * (t_in - t0):.1f} ms, native {1e3 * (t_native - t_in):.1f} ms, "
              f"objects {1e3 * (t1 - t_native):.1f} ms", file=sys.stderr)
    return FactorBranchResult(m, tnodes[info.root_slot], info.branch_width, info.carving_width, piece_map)


def factor_branch(n, bd, g=None, tree_cls=None):
    """(M, T) — reference ``factoring.py:263-267``."""
    r = factor_branch_audit(n, bd, g, tree_cls)
    return r.network, r.tree
