"""Planning heuristics, native: min-fill / min-degree tree decompositions and
tree_to_branch.

Drop-ins for the reference's ``min_fill_tree_decomposition``,
``min_degree_tree_decomposition`` (``pkg/src/tensorcount/decomposition.py:297-340``,
elimination order + ``_eliminate`` + ``binarize_tree_decomposition``) and
``tree_to_branch`` (``:346-411``).  The work runs in C++ (``csrc/decompose.cpp``,
C-ABI ``include/tc_decompose.h``) and returns exactly the reference's
decompositions: the same elimination order (ties broken by the same
``random.Random(seed).choice`` draws — the generator state crosses the
boundary), the same bags, and networkx trees with the same node names
(``fresh_node``'s ``(prefix, "%012d")`` numbering, continued from the
module's counter), node order and adjacency order, so ``factor_branch_audit``
builds the same plan from them.  ctypes releases the GIL for the native call,
so the portfolio's planner threads (``portfolio.py:158-223``) run in parallel.
"""

from __future__ import annotations

import ctypes as C
import itertools
import random
from dataclasses import dataclass

import networkx as nx
import numpy as np

from . import _lib
from .errors import InvalidDecomposition, NoHostBag

_fresh = itertools.count()  # fresh_node's counter (decomposition.py:20-26); the reference's when patched
_PREFIX = ("td", "bd", "bdleaf")


@dataclass
class TreeDecomposition:
    """Mirror of decomposition.py:29-39."""

    tree: nx.Graph
    bags: dict

    def __post_init__(self):
        self.bags = {n: frozenset(b) for n, b in self.bags.items()}

    def width(self) -> int:
        return max(len(b) for b in self.bags.values()) - 1


@dataclass
class BranchDecomposition:
    """Mirror of decomposition.py:42-45."""

    tree: nx.Graph
    leaf_map: dict


class _Counter:
    """Hands out a block of fresh_node numbers from a module's itertools.count."""

    def __init__(self, module=None, attr="_fresh"):
        self.module, self.attr = module, attr

    def start(self) -> int:
        if self.module is None:
            global _fresh
            return next(_fresh)
        return next(getattr(self.module, self.attr))

    def finish(self, end: int):
        if self.module is None:
            global _fresh
            _fresh = itertools.count(end)
        else:
            setattr(self.module, self.attr, itertools.count(end))


def _graph(labels, adj_off, adj):
    """An nx.Graph whose node order and every adjacency order are exactly the
    given ones (networkx keeps dict insertion order)."""
    tree = nx.Graph()
    tree.add_nodes_from(labels)
    A = tree._adj
    off = adj_off.tolist()
    al = adj.tolist()
    for k, u in enumerate(labels):
        A[u] = {labels[w]: None for w in al[off[k]:off[k + 1]]}
    for u in labels:
        du = A[u]
        for v, dd in du.items():
            if dd is None:
                dd = {}
                du[v] = dd
                A[v][u] = dd
    return tree


def _fetch(h, with_bags):
    L = _lib.lib()
    info = _lib.DecompInfo()
    _lib.check(L.tc_decomp_info_get(h, C.byref(info)))
    nn = info.num_nodes
    kind = np.empty(nn, np.int32)
    num = np.empty(nn, np.int64)
    adj_off = np.empty(nn + 1, np.int64)
    adj = np.empty(max(1, info.num_adj), np.int32)
    bag_off = np.empty(nn + 1 if with_bags else 1, np.int64)
    bag = np.empty(max(1, info.num_bag), np.int32)
    order = np.empty(max(1, info.num_order), np.int32)
    leaf_node = np.empty(max(1, info.num_leaf_map), np.int32)
    leaf_edge = np.empty(max(1, info.num_leaf_map), np.int32)
    p = _lib._p
    _lib.check(L.tc_decomp_fetch(h, p(kind, _lib.I32P), p(num, _lib.I64P), p(adj_off, _lib.I64P), p(adj, _lib.I32P),
                                 p(bag_off, _lib.I64P), p(bag, _lib.I32P), p(order, _lib.I32P),
                                 p(leaf_node, _lib.I32P), p(leaf_edge, _lib.I32P)))
    labels = [(_PREFIX[k], f"{x:012d}") for k, x in zip(kind.tolist(), num.tolist())]
    return info, labels, adj_off, adj, bag_off, bag, order[:info.num_order], leaf_node[:info.num_leaf_map], \
        leaf_edge[:info.num_leaf_map]


def _elimination_td(g, seed, score, td_cls=TreeDecomposition, counter=None):
    counter = counter or _Counter()
    verts = sorted(g.vertices, key=lambda v: str(v))  # _ordered_vertices (decomposition.py:297-298)
    vid = {v: k for k, v in enumerate(verts)}
    sadj = g.simple_adjacency()
    lists = [[vid[w] for w in sadj[v]] for v in verts]
    adj_off = np.zeros(len(verts) + 1, np.int64)
    np.cumsum([len(a) for a in lists], out=adj_off[1:])
    adj = np.fromiter((w for a in lists for w in a), np.int32, count=int(adj_off[-1]))
    state = random.Random(seed).getstate()[1]
    mt = np.asarray(state[:624], dtype=np.uint32)
    L = _lib.lib()
    h = C.c_void_p()
    start = counter.start()
    p = _lib._p
    _lib.check(L.tc_elim_td(len(verts), p(adj_off, _lib.I64P), p(adj, _lib.I32P), score,
                            p(mt, C.POINTER(C.c_uint32)), int(state[624]), start, C.byref(h)))
    try:
        info, labels, t_off, t_adj, bag_off, bag, order, _, _ = _fetch(h, True)
    finally:
        L.tc_decomp_free(h)
    counter.finish(int(info.counter_end))
    tree = _graph(labels, t_off, t_adj)
    bo, bl = bag_off.tolist(), bag.tolist()
    bags = {u: frozenset(verts[x] for x in bl[bo[k]:bo[k + 1]]) for k, u in enumerate(labels)}
    return td_cls(tree, bags)


def min_fill_tree_decomposition(g, seed: int = 0, td_cls=TreeDecomposition, counter=None):
    """decomposition.py:335-336."""
    return _elimination_td(g, seed, 0, td_cls, counter)


def min_degree_tree_decomposition(g, seed: int = 0, td_cls=TreeDecomposition, counter=None):
    """decomposition.py:339-340."""
    return _elimination_td(g, seed, 1, td_cls, counter)


def tree_to_branch(td, g, bd_cls=BranchDecomposition, counter=None):
    """Branch decomposition of width <= width_tree + 1 (decomposition.py:346-392)."""
    if not g.edges:
        raise InvalidDecomposition("tree_to_branch requires a graph with edges")
    counter = counter or _Counter()
    nodes = list(td.tree.nodes)
    npos = {u: k for k, u in enumerate(nodes)}
    lists = [[npos[w] for w in td.tree.adj[u]] for u in nodes]
    adj_off = np.zeros(len(nodes) + 1, np.int64)
    np.cumsum([len(a) for a in lists], out=adj_off[1:])
    adj = np.fromiter((w for a in lists for w in a), np.int32, count=int(adj_off[-1]))
    rank = np.empty(len(nodes), np.int32)
    rank[sorted(range(len(nodes)), key=lambda k: str(nodes[k]))] = np.arange(len(nodes), dtype=np.int32)
    vid = {}
    bag_lists = []
    for u in nodes:
        bag_lists.append([vid.setdefault(x, len(vid)) for x in td.bags[u]])
    edges = sorted(g.edges, key=str)
    eu, ev = [], []
    for e in edges:
        a, b = tuple(g.endpoints(e))
        eu.append(vid.setdefault(a, len(vid)))
        ev.append(vid.setdefault(b, len(vid)))
    bag_off = np.zeros(len(nodes) + 1, np.int64)
    np.cumsum([len(b) for b in bag_lists], out=bag_off[1:])
    bag = np.fromiter((x for b in bag_lists for x in b), np.int32, count=int(bag_off[-1]))
    eu = np.asarray(eu, np.int32)
    ev = np.asarray(ev, np.int32)
    L = _lib.lib()
    h = C.c_void_p()
    start = counter.start()
    p = _lib._p
    st = L.tc_tree_to_branch(len(nodes), p(adj_off, _lib.I64P), p(adj, _lib.I32P), p(rank, _lib.I32P),
                             p(bag_off, _lib.I64P), p(bag, _lib.I32P), len(vid), len(edges), p(eu, _lib.I32P),
                             p(ev, _lib.I32P), start, C.byref(h))
    if st != 0:
        msg = L.tc_last_error().decode(errors="replace")
        if msg.startswith("NoHostBag: "):
            counter.finish(start)
            raise NoHostBag(f"no bag contains both endpoints of edge {edges[int(msg.split(': ')[1])]!r}")
        _lib.check(st)
    try:
        info, labels, t_off, t_adj, _, _, _, leaf_node, leaf_edge = _fetch(h, False)
    finally:
        L.tc_decomp_free(h)
    counter.finish(int(info.counter_end))
    tree = _graph(labels, t_off, t_adj)
    leaf_map = {labels[k]: edges[e] for k, e in zip(leaf_node.tolist(), leaf_edge.tolist())}
    return bd_cls(tree, leaf_map)


def validate_tree_decomposition(td, g):
    """InvalidDecomposition unless td is a tree decomposition of g
    (decomposition.py:88-108, same checks, order and messages); the
    O(|E| x |bags|) host-bag and connectivity scans run natively."""
    what = "tree decomposition"
    nodes = list(td.tree.nodes)
    npos = {u: k for k, u in enumerate(nodes)}
    lists = [[npos[w] for w in td.tree.adj[u]] for u in nodes]
    adj_off = np.zeros(len(nodes) + 1, np.int64)
    np.cumsum([len(a) for a in lists], out=adj_off[1:])
    adj = np.fromiter((w for a in lists for w in a), np.int32, count=int(adj_off[-1]))
    verts = list(g.vertices)
    vid = {v: k for k, v in enumerate(verts)}
    if set(td.bags) != set(nodes):
        shape_only = True
    else:
        shape_only = False
    bag_lists = [[vid.get(x, len(verts)) for x in td.bags[u]] for u in nodes] if not shape_only else [[]] * len(nodes)
    bag_off = np.zeros(len(nodes) + 1, np.int64)
    np.cumsum([len(b) for b in bag_lists], out=bag_off[1:])
    bag = np.fromiter((x for b in bag_lists for x in b), np.int32, count=int(bag_off[-1]))
    edges = list(g.edges)
    ends = [tuple(g.edges[e]) for e in edges]
    eu = np.asarray([vid[a] for a, _ in ends], np.int32)
    ev = np.asarray([vid[b] for _, b in ends], np.int32)
    shape, bad_edge = C.c_int32(), C.c_int32()
    disc = np.zeros(max(1, len(verts)), np.int8)
    p = _lib._p
    _lib.check(_lib.lib().tc_validate_td(len(nodes), p(adj_off, _lib.I64P), p(adj, _lib.I32P), p(bag_off, _lib.I64P),
                                         p(bag, _lib.I32P), len(verts), len(edges), p(eu, _lib.I32P),
                                         p(ev, _lib.I32P), C.byref(shape), C.byref(bad_edge),
                                         p(disc, C.POINTER(C.c_int8))))
    if shape.value == 1:
        raise InvalidDecomposition(f"{what}: empty tree")
    if shape.value == 2:
        raise InvalidDecomposition(f"{what}: decomposition graph is not a tree")
    if shape_only:
        raise InvalidDecomposition(f"{what}: bags do not label every node")
    covered = set().union(*td.bags.values()) if td.bags else set()
    if covered != set(g.vertices):
        missing = set(g.vertices) - covered
        if missing:
            raise InvalidDecomposition(f"{what}: vertices {missing} in no bag")
        raise InvalidDecomposition(f"{what}: bags contain unknown vertices")
    if bad_edge.value >= 0:
        raise InvalidDecomposition(f"{what}: edge {edges[bad_edge.value]!r} has no host bag")
    for v in g.vertices:
        if disc[vid[v]]:
            raise InvalidDecomposition(f"{what}: bags containing {v!r} are disconnected")


def width_tree(td, g=None) -> int:
    """decomposition.py:144-147."""
    if g is not None:
        validate_tree_decomposition(td, g)
    return td.width()
