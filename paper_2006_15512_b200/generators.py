"""Synthetic CNF generators for the benchmark configurations.

These produce DIMACS text (with extended ``w v w0 w1`` weight lines, the form
parsed by the reference at ``pkg/src/tensorcount/formula.py:120-124``).  They
are input producers only; planning (reduce → min-fill → tree_to_branch →
factor_branch_audit) is done by the unmodified reference on the CPU and the
resulting plan is frozen in a ``.tcplan`` file (see ``planfile.py``).

Semantics follow ``pkg/tests/conftest.py:8-21`` (``random_cnf`` /
``random_weights``): k distinct variables per clause, sign from
``rng.random() < 0.5``, per-variable weights ``(U(0,1), U(0,1))``.
"""

from __future__ import annotations

import math
import random


def _dimacs(num_vars, clauses, weights):
    lines = [f"p cnf {num_vars} {len(clauses)}"]
    for c in clauses:
        lines.append(" ".join(str(l) for l in c) + " 0")
    if weights is not None:
        for v in sorted(weights):
            w0, w1 = weights[v]
            lines.append(f"w {v} {w0!r} {w1!r}")
    return "\n".join(lines) + "\n"


def uniform_3cnf(n: int, ratio: float, seed: int, weighted: bool = True) -> str:
    """Uniform random 3-CNF: m = round(n*ratio) clauses over 1..n."""
    rng = random.Random(seed)
    m = int(round(n * ratio))
    clauses = []
    for _ in range(m):
        vs = rng.sample(range(1, n + 1), 3)
        clauses.append(tuple(v if rng.random() < 0.5 else -v for v in vs))
    weights = None
    if weighted:
        weights = {v: (rng.uniform(0, 1), rng.uniform(0, 1)) for v in range(1, n + 1)}
    return _dimacs(n, clauses, weights)


def banded_3cnf(n: int, ratio: float, window: int, seed: int, weighted: bool = True) -> str:
    """Banded random 3-CNF: each clause draws its 3 variables from a sliding
    window [lo, lo+window), which bounds the primal bandwidth (and hence the
    plan width)."""
    rng = random.Random(seed)
    m = int(round(n * ratio))
    clauses = []
    for _ in range(m):
        lo = rng.randint(1, n - window + 1)
        vs = rng.sample(range(lo, lo + window), 3)
        clauses.append(tuple(v if rng.random() < 0.5 else -v for v in vs))
    weights = None
    if weighted:
        weights = {v: (rng.uniform(0, 1), rng.uniform(0, 1)) for v in range(1, n + 1)}
    return _dimacs(n, clauses, weights)


def grid_ising(L: int, seed: int, J: float = 0.5, h: float = 0.1) -> str:
    """L x L Ising model as weighted CNF.

    Spins s_{r,c} are variables 1..L^2.  Every right/down grid edge (u, v)
    gets an auxiliary variable e with e <-> (u xor v) as four clauses.  Spin
    weights are normalised (e^-f, e^f)/(e^-f + e^f), f ~ U(-h, h); edge
    weights are (e^j, e^-j), j ~ U(-J, J).
    """
    rng = random.Random(seed)

    def spin(r, c):
        return r * L + c + 1

    clauses = []
    weights = {}
    for r in range(L):
        for c in range(L):
            f = rng.uniform(-h, h)
            z = math.exp(-f) + math.exp(f)
            weights[spin(r, c)] = (math.exp(-f) / z, math.exp(f) / z)
    nxt = L * L + 1
    for r in range(L):
        for c in range(L):
            for (r2, c2) in ((r, c + 1), (r + 1, c)):
                if r2 >= L or c2 >= L:
                    continue
                u, v, e = spin(r, c), spin(r2, c2), nxt
                nxt += 1
                clauses += [(-e, u, v), (-e, -u, -v), (e, -u, v), (e, u, -v)]
                j = rng.uniform(-J, J)
                weights[e] = (math.exp(j), math.exp(-j))
    return _dimacs(nxt - 1, clauses, weights)


# Concrete inputs for BASELINE.json's configs.
CONFIGS = {
    # C1 restated: the literal n=60 instance is not CPU-runnable (max-rank 39)
    "c1a": dict(gen="uniform", n=30, ratio=3.0, seed=1),
    "c1b": dict(gen="uniform", n=40, ratio=3.0, seed=1),
    "c1a_unweighted": dict(gen="uniform", n=30, ratio=3.0, seed=1, weighted=False),
    "c2": dict(gen="banded", n=200, ratio=3.5, window=29, seed=1),
    "c3": dict(gen="grid", L=30, seed=1),
    # C4/C5: SURVEY §8d "reject any seed whose count is 0 (advance the seed)".
    # Seeds 1-10 of banded(400, 4.0, 36) are UNSAT (z3), 11 is the first SAT
    # seed.  C5 "2^12 slices of rank-30 subnetworks": window 34 (first SAT seed
    # 6) is the window whose 12-pick greedy prefix leaves per-slice max-rank
    # exactly 30 (windows 42-46 keep rank >= 39 after 12 picks; tools/scan_plans.py).
    "c4": dict(gen="banded", n=400, ratio=4.0, window=36, seed=11),
    "c5": dict(gen="banded", n=400, ratio=4.0, window=34, seed=6),
}


def config_dimacs(name: str) -> str:
    c = dict(CONFIGS[name])
    gen = c.pop("gen")
    if gen == "uniform":
        return uniform_3cnf(c["n"], c["ratio"], c["seed"], c.get("weighted", True))
    if gen == "banded":
        return banded_3cnf(c["n"], c["ratio"], c["window"], c["seed"], c.get("weighted", True))
    if gen == "grid":
        return grid_ising(c["L"], c["seed"])
    raise ValueError(gen)
