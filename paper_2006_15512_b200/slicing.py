"""Memory-bounded execution by index slicing — the drop-in for the reference's
``slicing.py`` (Algorithm 3, ``pkg/src/tensorcount/slicing.py:112-146``).

Same names, signatures, return type and error behaviour:

* ``mem_cost(n, t, drop=frozenset())``          — slicing.py:52-67 (exact, libtc)
* ``choose_slice_index(n, t, already=frozenset())`` — slicing.py:70-79 (libtc,
  incremental; identical picks incl. the sort_key tie-break)
* ``sliced_execute(n, t, mem_budget=None)``     — slicing.py:112-146, executed
  on the B200 by libtc.  Extra keyword-only arguments: ``slice_indices``
  (explicit slice set, skips the greedy), ``devices`` (list of CUDA ordinals).
* ``SlicedExecution``                           — slicing.py:82-88 (+ ``stats``)

Inputs may be this package's mirror types or the reference's own objects
(duck-typed); the result tensor is built with the caller's Tensor class.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import BudgetInfeasible, NoCandidates, PlanMismatch
from .flatten import _native, flatten

BYTES_PER_ENTRY = 8


@dataclass
class SlicedExecution:
    result: object
    sliced_indices: list = field(default_factory=list)
    mem_estimate: int = 0
    peak_observed: int = 0
    num_slices: int = 1
    stats: dict = field(default=None, repr=False, compare=False)


def _plan(n, t, with_sort_rank=True):
    flat = flatten(n, t, with_sort_rank=with_sort_rank)
    if flat.root_slot < 0 or (flat.left < 0).any() or (flat.right < 0).any():
        raise PlanMismatch("contraction tree leaves do not match the network")
    return flat, _lib.PlanHandle(flat)


def _ids(flat, indices):
    pos = {ix.id: k for k, ix in enumerate(flat.indices)}
    out = []
    for ix in indices:
        k = pos.get(ix.id)
        if k is None:
            continue  # an index absent from the network drops nothing
        out.append(k)
    return out


def mem_cost(n, t, drop=frozenset()) -> int:
    """Peak live bytes of strict postorder execution with ``drop`` sliced."""
    flat, h = _plan(n, t)
    return h.mem_cost(_ids(flat, drop))


def choose_slice_index(n, t, already=frozenset()):
    """Greedy pick: the bond minimising mem_cost, ties by smallest sort_key."""
    flat, h = _plan(n, t)
    k = h.choose_slice_index(_ids(flat, already))
    return flat.indices[k]


def _run_range(n, flat, h, mem_budget, sl, devices, slice_range):
    """Slices [b, e) of the plan only (the per-rank block of a sharded run, or
    a timed sample of a 2^30-slice job): their lexicographic sum."""
    b, e = (int(x) for x in slice_range)
    chosen = sl if sl is not None else (h.choose_slices(mem_budget) if mem_budget is not None else [])
    ex = _lib.Exec(h, chosen, (devices or [0])[0])
    ns = ex.num_slices()
    if not 0 <= b < e <= ns:
        raise ValueError(f"slice_range {slice_range} outside [0, {ns})")
    st = ex.run(b, e)
    folded, _ = ex.fetch()
    idx = h.result_indices(chosen)
    tensor_cls = type(n.tensors[0])
    shape = tuple(int(flat.domain[i]) for i in idx)
    result = tensor_cls(tuple(flat.indices[i] for i in idx), np.asarray(folded, dtype=np.float64).reshape(shape))
    return SlicedExecution(result=result, sliced_indices=[flat.indices[i] for i in chosen],
                           mem_estimate=st["mem_estimate"], peak_observed=st["peak_observed"], num_slices=e - b,
                           stats=st)


def _run(n, t, mem_budget=None, devices=None, slice_indices=None, slice_range=None):
    # sort_key ranks only matter to the greedy chooser (slicing.py:73-79)
    flat, h = _plan(n, t, with_sort_rank=mem_budget is not None and slice_indices is None)
    if slice_indices is None:
        sl = None
    else:
        # Index equality is by id (tensor.py:29-33); the callers' Index objects
        # are usually the network's own, found by one pointer scan in C
        nat = _native()
        if nat is not None:
            sl = nat.positions(flat.indices, list(slice_indices))
        else:
            pos = {ix.id: k for k, ix in enumerate(flat.indices)}
            sl = [pos.get(ix.id, -1) for ix in slice_indices]
    if sl is not None and any(k < 0 for k in sl):
        from .errors import NotABondIndex
        raise NotABondIndex("slice index is not an index of the network")
    if slice_range is not None:
        return _run_range(n, flat, h, mem_budget, sl, devices, slice_range)
    vals, idx, chosen, stats = h.sliced_execute(mem_budget, sl, devices)
    tensor_cls = type(n.tensors[0])
    inds = tuple(flat.indices[i] for i in idx)
    shape = tuple(int(flat.domain[i]) for i in idx)
    result = tensor_cls(inds, np.asarray(vals, dtype=np.float64).reshape(shape))
    return SlicedExecution(
        result=result,
        sliced_indices=[flat.indices[i] for i in chosen],
        mem_estimate=stats["mem_estimate"],
        peak_observed=stats["peak_observed"],
        num_slices=stats["num_slices"],
        stats=stats,
    )


def sliced_execute(n, t, mem_budget: int | None = None, *, slice_indices=None, devices=None,
                   slice_range=None) -> SlicedExecution:
    """Execute the plan within the byte budget on the GPU, slicing bond
    indices as needed and summing per-slice results in lexicographic order.

    ``slice_range=(b, e)`` (extension) executes slices b..e-1 only and returns
    their lexicographic sum (``num_slices = e - b``): one rank's block, or a
    timed sample of a job too large to run whole."""
    return _run(n, t, mem_budget=mem_budget, devices=devices, slice_indices=slice_indices, slice_range=slice_range)


__all__ = [
    "BYTES_PER_ENTRY",
    "BudgetInfeasible",
    "NoCandidates",
    "SlicedExecution",
    "choose_slice_index",
    "mem_cost",
    "sliced_execute",
]
