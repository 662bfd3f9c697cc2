"""Errors raised on the execution path.

Names and meaning mirror the reference hierarchy
(``pkg/src/tensorcount/errors.py``): ``IndexMismatch`` (:32),
``BindingOutOfDomain`` (:36), ``IndexOveruse`` (:42), ``PlanMismatch`` (:46),
``NotABondIndex`` (:80), ``NoCandidates`` (:84), ``BudgetInfeasible`` (:88),
and for the native planning steps ``InvalidDecomposition`` (:52), ``NoHostBag`` (:64),
``NotFactorable`` (:70), ``TooManyFreeIndices`` (:74).

``reference_patch.install`` re-raises these as the reference's own classes
(same name) so code catching ``tensorcount.errors.BudgetInfeasible`` keeps
working after the backend swap.
"""

from __future__ import annotations


class CounterError(Exception):
    """Base class of execution-path errors."""


class IndexMismatch(CounterError):
    pass


class BindingOutOfDomain(CounterError):
    pass


class IndexOveruse(CounterError):
    pass


class PlanMismatch(CounterError):
    pass


class NotABondIndex(CounterError):
    pass


class NoCandidates(CounterError):
    pass


class BudgetInfeasible(CounterError):
    pass


class InvalidDecomposition(CounterError):
    pass


class NoHostBag(CounterError):
    pass


class NotFactorable(CounterError):
    pass


class TooManyFreeIndices(CounterError):
    pass


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside libtc (status TC_CUDA / TC_NCCL)."""
