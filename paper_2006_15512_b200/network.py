"""Networks and contraction trees, mirroring the reference's ``network.py``.

* ``TensorNetwork`` — at most two occurrences per index; free/bond sets
  (ref ``network.py:29-57``).
* ``ContractionTree`` / ``leaf`` / ``join`` / ``left_deep_tree`` — frozen
  binary tree with iterative postorder, left before right
  (ref ``network.py:83-140``).
* ``execute`` — Algorithm 2 (ref ``network.py:151-163``), run on the B200 by
  libtc; raises ``PlanMismatch`` like ``_check_plan`` (``network.py:143-148``).
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass

from .errors import IndexOveruse, PlanMismatch


@dataclass(frozen=True, eq=False)
class TensorNetwork:
    tensors: tuple

    def __post_init__(self):
        ts = tuple(self.tensors)
        if not ts:
            raise ValueError("a tensor network must contain at least one tensor")
        object.__setattr__(self, "tensors", ts)
        occ = Counter()
        for t in ts:
            occ.update(t.indices)
        for ix, k in occ.items():
            if k > 2:
                raise IndexOveruse(f"index {ix.id!r} appears {k} times")
        object.__setattr__(self, "_free", frozenset(i for i, k in occ.items() if k == 1))
        object.__setattr__(self, "_bond", frozenset(i for i, k in occ.items() if k == 2))

    @property
    def free_indices(self) -> frozenset:
        return self._free

    @property
    def bond_indices(self) -> frozenset:
        return self._bond


@dataclass(frozen=True, eq=False, slots=True)
class ContractionTree:
    tensor: object = None
    left: "ContractionTree | None" = None
    right: "ContractionTree | None" = None

    def __post_init__(self):
        if self.tensor is None and (self.left is None or self.right is None):
            raise ValueError("internal node needs two children")
        if self.tensor is not None and (self.left is not None or self.right is not None):
            raise ValueError("leaf node cannot have children")

    @property
    def is_leaf(self) -> bool:
        return self.tensor is not None

    def leaves(self) -> list:
        out, stack = [], [self]
        while stack:
            node = stack.pop()
            if node.is_leaf:
                out.append(node.tensor)
            else:
                stack.extend((node.right, node.left))
        return out

    def postorder(self):
        seq, stack = [], [self]
        while stack:
            node = stack.pop()
            seq.append(node)
            if not node.is_leaf:
                stack.extend((node.left, node.right))
        return reversed(seq)


def leaf(t) -> ContractionTree:
    return ContractionTree(tensor=t)


def join(a: ContractionTree, b: ContractionTree) -> ContractionTree:
    return ContractionTree(left=a, right=b)


def left_deep_tree(tensors) -> ContractionTree:
    ts = list(tensors)
    node = leaf(ts[0])
    for t in ts[1:]:
        node = join(node, leaf(t))
    return node


def check_plan(n, t):
    """PlanMismatch unless the tree's leaves are exactly the network's tensors
    (by object identity, as ref ``network.py:143-148``)."""
    pl = t.leaves()
    if len(pl) != len(n.tensors) or set(map(id, pl)) != set(map(id, n.tensors)):
        raise PlanMismatch("contraction tree leaves do not match the network")


def execute(n, t, devices=None):
    """Contract the network pairwise along the tree on the GPU."""
    from .slicing import _run

    check_plan(n, t)
    return _run(n, t, mem_budget=None, devices=devices).result
