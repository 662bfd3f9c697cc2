"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/wmc_dp.c, an exact
weighted model counter restating the reference's count oracle
``brute_force_count`` (pkg/src/tensorcount/formula.py:183-215) as a
clause-frontier dynamic program (see the C file's header).  It anchors counts
and per-slice values at sizes where the reference's dense execution cannot run
on this hardware.  Only tests/, tools/ and bench.py's parity record use it.

DIMACS parsing follows the reference's ``parse_dimacs`` (formula.py:78-160):
``w v w0 w1`` or ``w v p`` (-> (1-p, p)) weight lines, default (1, 1),
tautological clauses dropped, duplicate literals removed.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import oracle as _o

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)

_bound = False


def _lib():
    global _bound
    h = _o.lib()
    if not _bound:
        h.wmc_dp.argtypes = [C.c_int32, C.c_int32, I32P, I64P, F64P, F64P, C.POINTER(C.c_int8), C.c_int64,
                             F64P, I64P]
        h.wmc_dp.restype = C.c_int
        _bound = True
    return h


def parse(text):
    """(num_vars, clauses, weights{v: (w0, w1)}) with the reference's clause
    normalisation."""
    n = 0
    clauses, pending, weights = [], [], {}
    for raw in text.splitlines():
        line = raw.strip()
        if not line or line[0] in "c%":
            continue
        if line.startswith("p"):
            n = int(line.split()[2])
            continue
        if line.startswith("w"):
            p = line.split()
            vals = [float(x) for x in p[2:]]
            weights[int(p[1])] = (1.0 - vals[0], vals[0]) if len(vals) == 1 else (vals[0], vals[1])
            continue
        for tok in line.split():
            lit = int(tok)
            if lit:
                pending.append(lit)
                continue
            seen = []
            for l in pending:
                if l not in seen:
                    seen.append(l)
            pending = []
            if any(-l in seen for l in seen):
                continue  # tautology
            clauses.append(tuple(seen))
    return n, clauses, weights


def count(text, fix=None, max_states=0):
    """Exact WMC of a DIMACS text; ``fix`` = {var: 0|1} restricts the sum.
    Returns (count, peak_states)."""
    n, clauses, weights = parse(text)
    lits = np.array([l for c in clauses for l in c] or [0], dtype=np.int32)
    off = np.zeros(len(clauses) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(c) for c in clauses]) if clauses else []
    w0 = np.ones(n + 1)
    w1 = np.ones(n + 1)
    for v, (a, b) in weights.items():
        w0[v], w1[v] = a, b
    fx = np.full(n + 1, -1, dtype=np.int8)
    for v, b in (fix or {}).items():
        fx[v] = b
    out = C.c_double()
    peak = C.c_int64()
    rc = _lib().wmc_dp(n, len(clauses), lits.ctypes.data_as(I32P), off.ctypes.data_as(I64P),
                       w0.ctypes.data_as(F64P), w1.ctypes.data_as(F64P),
                       fx.ctypes.data_as(C.POINTER(C.c_int8)), int(max_states), C.byref(out), C.byref(peak))
    if rc:
        raise RuntimeError({-1: "out of memory", -2: "more than 256 pending clauses",
                            -3: "state limit exceeded"}.get(rc, f"wmc_dp error {rc}"))
    return float(out.value), int(peak.value)
