"""Value types of the execution path, mirroring the reference's ``tensor.py``.

* ``Index`` — named axis; equality/hash by ``id`` only, ``sort_key`` =
  (type name, str(id)) for deterministic tie-breaks (ref ``tensor.py:18-37``).
* ``Assignment`` — Index -> value with domain check (ref ``tensor.py:40-47``).
* ``Tensor`` — immutable FP64 values reshaped to the index domains,
  row-major, first index slowest (ref ``tensor.py:50-89``).
* ``contract_pair`` — ONE pairwise contraction, executed on the B200 through
  libtc (ref ``tensor.py:96-108``; output index order ``kept_a ++ kept_b``).

These types hold host data only; every arithmetic operation on the path goes
through the CUDA library (``_lib.py``), never numpy.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import BindingOutOfDomain, IndexMismatch


class Index:
    """A named axis with a finite domain. Equality and hashing are by id."""

    __slots__ = ("id", "domain_size")

    def __init__(self, id, domain_size: int):
        if domain_size < 1:
            raise ValueError(f"index {id!r} has empty domain")
        self.id = id
        self.domain_size = int(domain_size)

    def __eq__(self, other):
        return hasattr(other, "domain_size") and hasattr(other, "id") and self.id == other.id

    def __hash__(self):
        return hash(self.id)

    def __repr__(self):
        return f"Index({self.id!r}, {self.domain_size})"

    def sort_key(self):
        return (str(type(self.id).__name__), str(self.id))


class Assignment(dict):
    """Map from Index to a value inside its domain."""

    def __init__(self, bindings=()):
        super().__init__(bindings)
        for ix, v in self.items():
            if not 0 <= v < ix.domain_size:
                raise BindingOutOfDomain(f"{v} outside domain of {ix.id!r}")


@dataclass(frozen=True, eq=False, slots=True)
class Tensor:
    indices: tuple
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        inds = tuple(self.indices)
        if len(set(inds)) != len(inds):
            raise ValueError("duplicate index in tensor")
        shape = tuple(ix.domain_size for ix in inds)
        object.__setattr__(self, "indices", inds)
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64).reshape(shape))

    @property
    def rank(self) -> int:
        return len(self.indices)

    @property
    def size(self) -> int:
        return int(self.values.size)

    def index_set(self) -> frozenset:
        return frozenset(self.indices)

    def entry(self, assignment) -> float:
        return float(self.values[tuple(assignment[ix] for ix in self.indices)])

    def transposed(self, order) -> "Tensor":
        """Same tensor with indices listed in ``order`` (a host view, no math)."""
        order = tuple(order)
        if len(order) != len(self.indices) or set(order) != set(self.indices):
            raise IndexMismatch("transpose order must be a permutation of the indices")
        pos = {ix: k for k, ix in enumerate(self.indices)}
        return Tensor(order, np.transpose(self.values, [pos[ix] for ix in order]))


def scalar(value: float) -> Tensor:
    return Tensor((), np.array(value, dtype=np.float64))


def contract_pair(a, b, device: int = 0):
    """Contract two tensors over their shared indices on the GPU.

    Same contract as reference ``tensor.py:96-108``: shared indices in a's
    order, result indices ``kept_a ++ kept_b``.  Runs a two-leaf plan through
    ``libtc`` (the same kernels as a full tree walk).
    """
    from .network import TensorNetwork, join, leaf
    from .slicing import _run

    # fresh wrappers: the operands may be the same object (contract_pair(a, a))
    n = TensorNetwork((type(a)(a.indices, a.values), type(b)(b.indices, b.values)))
    t = join(leaf(n.tensors[0]), leaf(n.tensors[1]))
    return _run(n, t, mem_budget=None, devices=[device]).result
