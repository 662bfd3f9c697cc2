"""The weighted-CNF -> tensor-network reduction in linear time.

Drop-in for the reference's ``reduce_formula`` (``pkg/src/tensorcount/reduction.py:80-101``),
the first step of FactorTree's input.  The reference
finds each variable's occurrences by scanning every clause for every variable
(``occurrence_indices``, ``reduction.py:22-29``, and again in
``reduce_formula``: O(variables x clauses), 16 s on the 30x30 grid); here one
pass over the literals builds the per-variable occurrence lists.  The output is
the reference's network object for object: Index ``(var, clause ordinal)``
(domain 2) shared by a variable's copy tensor and its clause tensor, copy
tensors first (variable order, indices in clause order, ``w0`` at the all-zeros
entry and ``w1`` at the all-ones entry of a dense ``2^occ`` array,
``reduction.py:32-39``), then clause tensors (clause order, indices in literal
order, 1.0 everywhere except 0.0 at the one falsifying assignment,
``reduction.py:42-66``); rank-0 scalars for occurrence-free variables
(``w0 + w1``) and empty clauses (0.0).
"""

from __future__ import annotations

import numpy as np


def reduce_formula(formula, weights, index_cls=None, tensor_cls=None, network_cls=None):
    """TensorNetwork whose contraction is the weighted model count.  The value
    classes default to this package's; pass the reference's to get its objects."""
    if index_cls is None:
        from .tensor import Index as index_cls
    if tensor_cls is None:
        from .tensor import Tensor as tensor_cls
    if network_cls is None:
        from .network import TensorNetwork as network_cls

    def scalar(x):
        return tensor_cls((), np.array(x, dtype=np.float64))

    clauses = formula.clauses
    occ = {}    # var -> clause ordinals (ascending, one per clause)
    index = {}  # (var, clause ordinal) -> Index, created variable-major like reduction.py:22-29
    for c_ord, clause in enumerate(clauses):
        for lit in clause:
            lst = occ.setdefault(abs(lit), [])
            if not lst or lst[-1] != c_ord:
                lst.append(c_ord)
    tensors = []
    for var in formula.variables():
        w0, w1 = weights.pair(var)
        ords = occ.get(var, ())
        inds = []
        for c_ord in ords:
            ix = index_cls((var, c_ord), 2)
            index[(var, c_ord)] = ix
            inds.append(ix)
        if not inds:
            tensors.append(scalar(w0 + w1))
            continue
        values = np.zeros((2,) * len(inds))
        values[(0,) * len(inds)] = w0
        values[(1,) * len(inds)] = w1
        tensors.append(tensor_cls(tuple(inds), values))
    for c_ord, clause in enumerate(clauses):
        if not clause:
            tensors.append(scalar(0.0))  # empty clause: unsatisfiable
            continue
        inds = tuple(index[(abs(lit), c_ord)] for lit in clause)
        # CnfFormula clauses have distinct variables (formula.py:36-46), so the
        # clause is satisfied unless every literal is false: one zero entry
        values = np.ones((2,) * len(inds))
        values[tuple(0 if lit > 0 else 1 for lit in clause)] = 0.0
        tensors.append(tensor_cls(inds, values))
    if not tensors:
        return network_cls((scalar(1.0),))  # empty formula over 0 vars
    return network_cls(tuple(tensors))
