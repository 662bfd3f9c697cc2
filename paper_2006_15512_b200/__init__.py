"""B200-native execution stage for tensor-network weighted model counting
(arXiv 2006.15512): the drop-in for ``tensorcount.slicing.sliced_execute``.

Public API mirrors the reference's execution path (tensor.py / network.py /
slicing.py); all arithmetic runs in libtc's sm_100a kernels.
"""

from .errors import (
    BindingOutOfDomain,
    BudgetInfeasible,
    CounterError,
    DeviceError,
    IndexMismatch,
    IndexOveruse,
    NoCandidates,
    NotABondIndex,
    PlanMismatch,
)
from .network import ContractionTree, TensorNetwork, execute, join, leaf, left_deep_tree
from .slicing import BYTES_PER_ENTRY, SlicedExecution, choose_slice_index, mem_cost, sliced_execute
from .tensor import Assignment, Index, Tensor, contract_pair, scalar

__version__ = "0.1.0"

__all__ = [
    "Assignment", "BYTES_PER_ENTRY", "BindingOutOfDomain", "BudgetInfeasible", "ContractionTree",
    "CounterError", "DeviceError", "Index", "IndexMismatch", "IndexOveruse", "NoCandidates",
    "NotABondIndex", "PlanMismatch", "SlicedExecution", "Tensor", "TensorNetwork",
    "choose_slice_index", "contract_pair", "execute", "join", "leaf", "left_deep_tree",
    "mem_cost", "scalar", "sliced_execute",
]
