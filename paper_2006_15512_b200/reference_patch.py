"""Swap the B200 execution stage into an imported ``tensorcount`` package.

The reference has no plugin API for this path: ``driver.py:27``
binds ``sliced_execute`` at import and calls it at ``driver.py:235``;
``slicing.py`` and ``network.py`` are imported by the tests directly.  So the
swap is by module attribute:

    import tensorcount
    from paper_2006_15512_b200 import reference_patch
    reference_patch.install(tensorcount)      # count_formula now runs on the GPU

Errors raised by the backend are re-raised as the reference's own exception
classes (same names), and the return value is the reference's
``SlicedExecution`` dataclass, so callers cannot tell the difference.
"""

from __future__ import annotations

import functools
import importlib

from . import decomposition as own_decomposition
from . import errors as own_errors
from . import factoring as own_factoring
from . import network as own_network
from . import reduction as own_reduction
from . import slicing as own_slicing
from . import tensor as own_tensor

_SAVED = {}


def _translate(ref_errors):
    mapping = {}
    for name in ("IndexMismatch", "BindingOutOfDomain", "IndexOveruse", "PlanMismatch",
                 "NotABondIndex", "NoCandidates", "BudgetInfeasible", "InvalidDecomposition",
                 "NotFactorable", "TooManyFreeIndices", "NoHostBag"):
        mapping[getattr(own_errors, name)] = getattr(ref_errors, name)
    return mapping


def install(tensorcount=None, devices=None, contract_pair=False, execution=True, factoring=True, planning=True):
    """Patch ``tensorcount.{driver,slicing,network}`` to use libtc.  With
    ``contract_pair=True`` also ``tensorcount.tensor.contract_pair``
    (tensor.py:96-108) — the reference's own test suite imports it directly.
    ``factoring`` swaps in the native FactorTree step (``factoring.py``:
    ``factor_branch_audit`` / ``factor_branch``, also as bound by
    ``driver.py:22`` and ``__init__.py:5``) and the linear-time
    ``reduce_formula`` (``reduction.py``, also ``driver.py:24``, ``__init__.py:9``); ``planning`` the native
    min-fill / min-degree decompositions and ``tree_to_branch``
    (``decomposition.py``, also as bound by ``portfolio.py:18-31`` and
    ``driver.py:20``, fresh names from the reference's own counter);
    ``execution=False`` leaves the execution path on the reference (the
    CPU-only check of the host-side steps)."""
    if tensorcount is None:
        tensorcount = importlib.import_module("tensorcount")
    driver = importlib.import_module(tensorcount.__name__ + ".driver")
    ref_factoring = importlib.import_module(tensorcount.__name__ + ".factoring")
    ref_decomp = importlib.import_module(tensorcount.__name__ + ".decomposition")
    ref_portfolio = importlib.import_module(tensorcount.__name__ + ".portfolio")
    ref_reduction = importlib.import_module(tensorcount.__name__ + ".reduction")
    slicing = importlib.import_module(tensorcount.__name__ + ".slicing")
    network = importlib.import_module(tensorcount.__name__ + ".network")
    tensor = importlib.import_module(tensorcount.__name__ + ".tensor")
    ref_errors = importlib.import_module(tensorcount.__name__ + ".errors")
    emap = _translate(ref_errors)
    RefSE = slicing.SlicedExecution

    def wrap(fn, convert=None):
        @functools.wraps(fn)
        def inner(*a, **kw):
            try:
                out = fn(*a, **kw)
            except tuple(emap) as e:
                raise emap[type(e)](str(e)) from None
            return convert(out) if convert else out
        return inner

    def to_ref(se):
        return RefSE(se.result, list(se.sliced_indices), se.mem_estimate, se.peak_observed, se.num_slices)

    def sliced_execute(n, t, mem_budget=None, **kw):
        if devices is not None and "devices" not in kw:
            kw["devices"] = devices
        return own_slicing.sliced_execute(n, t, mem_budget, **kw)

    def execute(n, t):
        return own_network.execute(n, t, devices=devices)

    RefFBR = ref_factoring.FactorBranchResult
    tree_cls = network.ContractionTree

    def to_ref_fbr(r):
        return RefFBR(r.network, r.tree, r.branch_width, r.carving_width, r.piece_map)

    def factor_branch_audit(n, bd, g=None):
        return own_factoring.factor_branch_audit(n, bd, g, tree_cls=tree_cls)

    def factor_branch(n, bd, g=None):
        r = own_factoring.factor_branch_audit(n, bd, g, tree_cls=tree_cls)
        return r.network, r.tree

    counter = own_decomposition._Counter(ref_decomp)

    def min_fill(g, seed=0):
        return own_decomposition.min_fill_tree_decomposition(g, seed, ref_decomp.TreeDecomposition, counter)

    def min_degree(g, seed=0):
        return own_decomposition.min_degree_tree_decomposition(g, seed, ref_decomp.TreeDecomposition, counter)

    def tree_to_branch(td, g):
        return own_decomposition.tree_to_branch(td, g, ref_decomp.BranchDecomposition, counter)

    def time_cost(n, t, throughput=1e9):  # network.py:184-188 with the native plan (contraction_ops)
        _, h = own_slicing._plan(n, t, with_sort_rank=False)
        return h.info().contraction_ops.value() / throughput

    def max_rank(n, t):  # network.py:178-181
        _, h = own_slicing._plan(n, t, with_sort_rank=False)
        return int(h.info().max_rank)

    def serialize_plan(n, t):  # network.py:235-251: flatten numbers slots exactly like it
        flat, _ = own_slicing._plan(n, t, with_sort_rank=False)
        nl = flat.num_leaves
        lines = [f"contract {a} {b} -> {nl + k}" for k, (a, b) in enumerate(zip(flat.left.tolist(), flat.right.tolist()))]
        return "\n".join(lines) + ("\n" if lines else "")

    def reduce_formula(formula, weights):
        return own_reduction.reduce_formula(formula, weights, tensor.Index, tensor.Tensor, network.TensorNetwork)

    patched = {}
    if factoring:  # the FactorTree step's input: the reduction
        for mod in (ref_reduction, driver, tensorcount):
            patched[(mod, "reduce_formula")] = wrap(reduce_formula)
    if planning:
        for mod in (ref_decomp, ref_portfolio):
            patched[(mod, "min_fill_tree_decomposition")] = wrap(min_fill)
            patched[(mod, "min_degree_tree_decomposition")] = wrap(min_degree)
            patched[(mod, "validate_tree_decomposition")] = wrap(own_decomposition.validate_tree_decomposition)
            patched[(mod, "width_tree")] = wrap(own_decomposition.width_tree)
        patched[(ref_decomp, "tree_to_branch")] = wrap(tree_to_branch)
        patched[(driver, "tree_to_branch")] = wrap(tree_to_branch)
        patched[(driver, "time_cost")] = wrap(time_cost)
        for mod in (network, driver):  # count_formula's CountResult fields (driver.py:238-251)
            patched[(mod, "max_rank")] = wrap(max_rank)
            patched[(mod, "serialize_plan")] = wrap(serialize_plan)
    if factoring:
        patched.update({
            (ref_factoring, "factor_branch_audit"): wrap(factor_branch_audit, to_ref_fbr),
            (ref_factoring, "factor_branch"): wrap(factor_branch),
            (driver, "factor_branch_audit"): wrap(factor_branch_audit, to_ref_fbr),
            (tensorcount, "factor_branch"): wrap(factor_branch),
        })
    if execution:
        patched.update({
            (driver, "sliced_execute"): wrap(sliced_execute, to_ref),
            (slicing, "sliced_execute"): wrap(sliced_execute, to_ref),
            (slicing, "mem_cost"): wrap(own_slicing.mem_cost),
            (slicing, "choose_slice_index"): wrap(own_slicing.choose_slice_index),
            (network, "execute"): wrap(execute),
            (tensorcount, "sliced_execute"): wrap(sliced_execute, to_ref),
            (tensorcount, "execute"): wrap(execute),
        })
    else:
        contract_pair = False
    if contract_pair:
        dev = (devices or [0])[0]

        def contract_pair_gpu(a, b):
            return own_tensor.contract_pair(a, b, device=dev)

        patched[(tensor, "contract_pair")] = wrap(contract_pair_gpu)
    for (mod, name), fn in patched.items():
        _SAVED.setdefault((mod, name), getattr(mod, name))
        setattr(mod, name, fn)


def uninstall():
    for (mod, name), fn in _SAVED.items():
        setattr(mod, name, fn)
    _SAVED.clear()
