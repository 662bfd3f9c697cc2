"""Generate golden fixtures by running the UNMODIFIED reference here.

    python tests/golden/make_golden.py        -> tests/golden/cases.json

Each case is a flattened (network, tree) plan (the arrays of include/tc.h's
tc_plan_desc) plus what the reference returned for it:
  * ``sliced_execute`` (slicing.py:112-146): result values (float.hex, reference
    index order), sliced_indices, mem_estimate, peak_observed, num_slices —
    unbudgeted, greedy-budgeted and with explicit slice sets;
  * ``mem_cost`` (slicing.py:52-67) and ``choose_slice_index`` (:70-79);
  * for CNF-derived cases, the known answers the reference's own tests pin
    (EXAMPLE4 -> 7.0, psi_n -> 2^n - 2, README 1.25, ...) and brute_force_count.

Families mirror the reference tests: ``random_network`` chains with domains
2-3 (test_slicing.py:27-42, test_acceptance.py:122-140), random pairs
(test_tensor.py:87-95), driver-planned CNFs (driver.py:217-235).
Needs the reference importable (oracle/_ref or /root/reference/pkg/src).
"""

from __future__ import annotations

import itertools
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(p):
        sys.path.insert(1, p)
        break

from tensorcount.driver import plan_contraction  # noqa: E402
from tensorcount.errors import BudgetInfeasible  # noqa: E402
from tensorcount.formula import CnfFormula, WeightFunction, brute_force_count, parse_dimacs  # noqa: E402
from tensorcount.network import TensorNetwork, join, leaf, left_deep_tree  # noqa: E402
from tensorcount.reduction import reduce_formula  # noqa: E402
from tensorcount.slicing import choose_slice_index, mem_cost, sliced_execute  # noqa: E402
from tensorcount.tensor import Index, Tensor  # noqa: E402

from paper_2006_15512_b200.flatten import flatten  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cases.json")


def enc_plan(n, t):
    f = flatten(n, t)
    return f, dict(
        ids=[repr(ix.id) for ix in f.indices],
        domain=f.domain.tolist(),
        sort_rank=f.sort_rank.tolist(),
        leaf_idx_off=f.leaf_idx_off.tolist(),
        leaf_idx=f.leaf_idx.tolist(),
        leaf_val_off=f.leaf_val_off.tolist(),
        leaf_val=[float(x).hex() for x in f.leaf_val],
        left=f.left.tolist(),
        right=f.right.tolist(),
        root_slot=int(f.root_slot),
    )


def run_ref(f, n, t, **kw):
    pos = {ix: k for k, ix in enumerate(f.indices)}
    try:
        out = sliced_execute(n, t, **kw)
    except BudgetInfeasible as e:
        return dict(error="BudgetInfeasible", message=str(e))
    return dict(
        values=[float(x).hex() for x in np.asarray(out.result.values).reshape(-1)],
        indices=[pos[ix] for ix in out.result.indices],
        chosen=[pos[ix] for ix in out.sliced_indices],
        mem_estimate=str(out.mem_estimate),
        peak_observed=str(out.peak_observed),
        num_slices=out.num_slices,
    )


def explicit_slices(f, n, t, combo):
    """Slice-sum via the reference primitives for an explicit slice set
    (network_slice per assignment, test_slicing.py:127-151 pattern)."""
    from tensorcount.slicing import network_slice
    from tensorcount.tensor import Assignment
    from tensorcount.network import execute
    total = None
    for values in itertools.product(*(range(i.domain_size) for i in combo)):
        s = network_slice(n, Assignment(zip(combo, values)))
        # same tree shape over the sliced leaves (slicing.py:30-41)
        m = {id(a): b for a, b in zip(n.tensors, s.tensors)}
        built = {}
        for node in t.postorder():
            built[id(node)] = leaf(m[id(node.tensor)]) if node.is_leaf else join(built[id(node.left)], built[id(node.right)])
        part = execute(s, built[id(t)])
        total = part if total is None else Tensor(total.indices, total.values + part.transposed(total.indices).values)
    pos = {ix: k for k, ix in enumerate(f.indices)}
    return dict(values=[float(x).hex() for x in np.asarray(total.values).reshape(-1)],
                indices=[pos[ix] for ix in total.indices])


def random_network(rng, max_tensors=6, max_domain=3):
    k = rng.randint(2, max_tensors)
    bonds = [Index(("b", j), rng.randint(2, max_domain)) for j in range(k - 1)]
    tensors = []
    for j in range(k):
        inds = []
        if j > 0:
            inds.append(bonds[j - 1])
        if j < k - 1:
            inds.append(bonds[j])
        if rng.random() < 0.3:
            inds.append(Index(("f", j), rng.randint(2, max_domain)))
        size = int(np.prod([i.domain_size for i in inds])) if inds else 1
        vals = np.array([rng.uniform(-1, 1) for _ in range(size)]).reshape([i.domain_size for i in inds])
        tensors.append(Tensor(tuple(inds), vals))
    return TensorNetwork(tuple(tensors))


def net_cases(cases):
    rng = random.Random(20240817)
    for c in range(24):
        n = random_network(rng, max_tensors=6 if c < 16 else 9)
        t = left_deep_tree(n.tensors)
        f, plan = enc_plan(n, t)
        full = mem_cost(n, t)
        exp = dict(unsliced=run_ref(f, n, t))
        budget = max(8, int(full * 0.75))
        exp["budgeted"] = dict(budget=budget, **run_ref(f, n, t, mem_budget=budget))
        exp["infeasible"] = dict(budget=1, **run_ref(f, n, t, mem_budget=1))
        bonds = sorted(n.bond_indices, key=Index.sort_key)
        pos = {ix: k for k, ix in enumerate(f.indices)}
        exp["mem_cost"] = {"": str(full)}
        for b in bonds:
            exp["mem_cost"][str(pos[b])] = str(mem_cost(n, t, drop=frozenset({b})))
        if bonds:
            exp["choose"] = pos[choose_slice_index(n, t)]
        exp["explicit"] = []
        for size in (1, 2):
            for combo in list(itertools.combinations(bonds, size))[:3]:
                exp["explicit"].append(dict(ids=[pos[i] for i in combo], **explicit_slices(f, n, t, combo)))
        cases.append(dict(name=f"random_network_{c}", family="random_network", plan=plan, expected=exp))


def pair_cases(cases):
    rng = random.Random(7)
    pool = [Index(name, rng.choice([2, 3])) for name in "abcdefgh"]
    for c in range(25):
        ia = rng.sample(pool, rng.randint(0, 3))
        ib = rng.sample(pool, rng.randint(0, 3))
        if not ia and not ib:
            ib = [pool[0]]

        def rt(inds):
            size = int(np.prod([i.domain_size for i in inds])) if inds else 1
            return Tensor(tuple(inds), np.array([rng.uniform(-2, 2) for _ in range(size)]).reshape([i.domain_size for i in inds]))
        a, b = rt(ia), rt(ib)
        n = TensorNetwork((a, b))
        t = join(leaf(a), leaf(b))
        f, plan = enc_plan(n, t)
        cases.append(dict(name=f"pair_{c}", family="pair", plan=plan, expected=dict(unsliced=run_ref(f, n, t))))


EXAMPLE4 = "p cnf 4 4\n1 2 -3 0\n1 3 4 0\n-2 -3 0\n-3 -4 0\n"


def cnf_cases(cases):
    known = [
        ("example4", EXAMPLE4, 7.0),
        ("readme_1_25", "p cnf 2 1\nw 1 0.25\n1 2 0\n", 1.25),
        ("unit_0_25", "p cnf 1 1\nw 1 0.25\n1 0\n", 0.25),
        ("three_free", "p cnf 3 0\n", 8.0),
        ("empty_clause", "p cnf 2 1\n0\n", 0.0),
        ("or2", "p cnf 2 1\n1 2 0\n", 3.0),
    ]
    for n_vars in range(4, 11):
        f = CnfFormula(n_vars, (tuple(range(1, n_vars + 1)), tuple(-v for v in range(1, n_vars + 1))))
        from tensorcount.formula import serialize_dimacs
        known.append((f"psi_{n_vars}", serialize_dimacs(f, WeightFunction({})), float(2 ** n_vars - 2)))
    rng = random.Random(20240817)
    for c in range(16):
        nv, nc = rng.randint(5, 14), rng.randint(5, 30)
        k = min(3, nv)
        clauses = []
        for _ in range(nc):
            vs = rng.sample(range(1, nv + 1), k)
            clauses.append(tuple(v if rng.random() < 0.5 else -v for v in vs))
        w = {v: (rng.uniform(0, 1), rng.uniform(0, 1)) for v in range(1, nv + 1)}
        from tensorcount.formula import serialize_dimacs
        known.append((f"suite_{c}", serialize_dimacs(CnfFormula(nv, tuple(clauses)), WeightFunction(w)), None))
    for name, text, answer in known:
        formula, weights = parse_dimacs(text)
        n0 = reduce_formula(formula, weights)
        best, _, _ = plan_contraction(n0, alpha=0.0)
        n, t = best.network, best.tree
        f, plan = enc_plan(n, t)
        exp = dict(unsliced=run_ref(f, n, t), known=answer, brute_force=brute_force_count(formula, weights))
        full = mem_cost(n, t)
        if n.bond_indices:
            budget = max(8, full - 1)  # test_driver.py:171-177: just below the unsliced estimate
            exp["budgeted"] = dict(budget=budget, **run_ref(f, n, t, mem_budget=budget))
        cases.append(dict(name=f"cnf_{name}", family="cnf", dimacs=text, plan=plan, expected=exp))


def main():
    cases = []
    pair_cases(cases)
    net_cases(cases)
    cnf_cases(cases)
    json.dump(dict(generator="tests/golden/make_golden.py", reference="tensorcount (unmodified)", cases=cases),
              open(OUT, "w"), indent=0)
    print(len(cases), "cases ->", OUT)


if __name__ == "__main__":
    main()
