"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/tc_oracle.c, the CPU
restatement of the reference execution path (slicing.py:52-146,
tensor.py:96-125).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module; the product package never does.

All functions take a ``FlatPlan`` (paper_2006_15512_b200/flatten.py), i.e. the
exact arrays that cross the libtc C-ABI, so checker and product see the same
input.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "liboracle.so")

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
U64P = C.POINTER(C.c_uint64)


class OPlan(C.Structure):
    _fields_ = [
        ("ni", C.c_int32), ("nl", C.c_int32), ("nn", C.c_int32), ("root", C.c_int32),
        ("dom", I32P), ("srank", I32P), ("lidx_off", I64P), ("lidx", I32P),
        ("lval_off", I64P), ("lval", F64P), ("left", I32P), ("right", I32P),
    ]


_lib = None


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(os.path.join(HERE, "tc_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        h = C.CDLL(LIB)
        h.oracle_mem_cost.argtypes = [C.POINTER(OPlan), I32P, C.c_int, U64P, U64P]
        h.oracle_mem_cost.restype = None
        h.oracle_choose_slice_index.argtypes = [C.POINTER(OPlan), I32P, C.c_int]
        h.oracle_choose_slice_index.restype = C.c_int
        h.oracle_sliced_execute.argtypes = [C.POINTER(OPlan), C.c_int, C.c_int64, I32P, C.c_int, F64P, C.c_int64,
                                            I32P, C.POINTER(C.c_int), I32P, C.POINTER(C.c_int), U64P, U64P, U64P,
                                            U64P, I64P]
        h.oracle_sliced_execute.restype = C.c_int
        _lib = h
    return _lib


class _Plan:
    def __init__(self, flat):
        self.keep = [
            np.ascontiguousarray(flat.domain, np.int32), np.ascontiguousarray(flat.sort_rank, np.int32),
            np.ascontiguousarray(flat.leaf_idx_off, np.int64), np.ascontiguousarray(flat.leaf_idx, np.int32),
            np.ascontiguousarray(flat.leaf_val_off, np.int64), np.ascontiguousarray(flat.leaf_val, np.float64),
            np.ascontiguousarray(flat.left, np.int32), np.ascontiguousarray(flat.right, np.int32),
        ]
        d, s, io, ix, vo, vv, lf, rt = self.keep
        self.s = OPlan(len(d), len(io) - 1, len(lf), int(flat.root_slot),
                       d.ctypes.data_as(I32P), s.ctypes.data_as(I32P), io.ctypes.data_as(I64P),
                       ix.ctypes.data_as(I32P), vo.ctypes.data_as(I64P), vv.ctypes.data_as(F64P),
                       lf.ctypes.data_as(I32P), rt.ctypes.data_as(I32P))


def _ids(ids):
    a = np.ascontiguousarray(np.asarray(list(ids), dtype=np.int32))
    return a, a.ctypes.data_as(I32P), len(a)


def mem_cost(flat, drop_ids=()) -> int:
    p = _Plan(flat)
    a, ptr, n = _ids(drop_ids)
    lo, hi = C.c_uint64(), C.c_uint64()
    lib().oracle_mem_cost(C.byref(p.s), ptr, n, C.byref(lo), C.byref(hi))
    return int(lo.value) | (int(hi.value) << 64)


def choose_slice_index(flat, already_ids=()) -> int:
    p = _Plan(flat)
    a, ptr, n = _ids(already_ids)
    return int(lib().oracle_choose_slice_index(C.byref(p.s), ptr, n))


class BudgetInfeasible(Exception):
    pass


def sliced_execute(flat, mem_budget=None, slice_ids=None):
    """Returns dict(values (row-major, reference index order), indices,
    chosen, mem_estimate, peak_observed, num_slices)."""
    p = _Plan(flat)
    if slice_ids is not None:
        mode, budget = 2, 0
    elif mem_budget is not None:
        mode, budget = 1, max(-(2**63) + 1, min(2**63 - 1, int(mem_budget)))
    else:
        mode, budget = 0, 0
    a, ptr, n = _ids(slice_ids or ())
    ni = len(flat.domain)
    cap = 1
    # result size <= product over free indices (root rank bounded by #indices)
    occ = np.bincount(flat.leaf_idx, minlength=ni) if len(flat.leaf_idx) else np.zeros(ni, int)
    for i in np.nonzero(occ == 1)[0]:
        cap *= int(flat.domain[i])
    out = np.zeros(max(1, cap), np.float64)
    oidx = np.zeros(max(1, ni), np.int32)
    rank = C.c_int()
    chosen = np.zeros(max(1, ni), np.int32)
    nch = C.c_int()
    el, eh, pl, ph = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    ns = C.c_int64()
    st = lib().oracle_sliced_execute(C.byref(p.s), mode, budget, ptr, n, out.ctypes.data_as(F64P), len(out),
                                     oidx.ctypes.data_as(I32P), C.byref(rank), chosen.ctypes.data_as(I32P),
                                     C.byref(nch), C.byref(el), C.byref(eh), C.byref(pl), C.byref(ph),
                                     C.byref(ns))
    if st == 3:
        raise BudgetInfeasible("cannot fit in budget even fully sliced")
    idx = oidx[: rank.value].tolist()
    size = 1
    for i in idx:
        size *= int(flat.domain[i])
    return dict(
        values=out[:size].copy(),
        indices=idx,
        chosen=chosen[: nch.value].tolist(),
        mem_estimate=int(el.value) | (int(eh.value) << 64),
        peak_observed=int(pl.value) | (int(ph.value) << 64),
        num_slices=int(ns.value),
    )
