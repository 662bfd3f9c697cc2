"""GPU parity: libtc's sm_100a path vs the reference's golden outputs and the
CPU oracle, through the public drop-in API (mirror of slicing.sliced_execute /
network.execute / tensor.contract_pair).

Tolerances (north_star): FP64 results within 1e-9 relative of the reference
(observed: ~1e-15); unweighted counts below 2^53 exact; integer outputs
(sliced_indices, mem_estimate, peak_observed, num_slices) bit-exact.
"""

import itertools
import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, PLANS, case_flat, hexvals, load_cases
from oracle import oracle
from paper_2006_15512_b200 import (BudgetInfeasible, Index, Tensor, TensorNetwork, contract_pair, execute, join,
                                   leaf, left_deep_tree, planfile, sliced_execute)
from paper_2006_15512_b200 import _lib
from paper_2006_15512_b200.errors import PlanMismatch

pytestmark = pytest.mark.gpu
CASES = load_cases()
RTOL = 1e-9


def _aligned(res, flat_indices_order, want_idx):
    """result values re-ordered to the golden index order"""
    got_idx = [flat_indices_order.index(ix) for ix in res.indices]
    v = np.asarray(res.values)
    if got_idx == want_idx:
        return v.reshape(-1)
    perm = [got_idx.index(i) for i in want_idx]
    return np.transpose(v, perm).reshape(-1)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_unsliced_matches_reference(case):
    flat = case_flat(case)
    n, t = planfile.to_objects(flat)
    exp = case["expected"]["unsliced"]
    out = sliced_execute(n, t)
    idx = [flat.indices.index(ix) for ix in out.result.indices]
    assert idx == exp["indices"]  # reference order kept_a ++ kept_b
    assert np.allclose(np.asarray(out.result.values).reshape(-1), hexvals(exp["values"]), rtol=RTOL, atol=1e-12)
    assert out.mem_estimate == int(exp["mem_estimate"])
    assert out.peak_observed == int(exp["peak_observed"])
    assert out.num_slices == 1 and out.sliced_indices == []
    # network.execute (Algorithm 2) gives the same tensor
    e = execute(n, t)
    assert np.array_equal(np.asarray(e.values), np.asarray(out.result.values))


@pytest.mark.parametrize("case", [c for c in CASES if "budgeted" in c["expected"]],
                         ids=[c["name"] for c in CASES if "budgeted" in c["expected"]])
def test_budgeted_matches_reference(case):
    flat = case_flat(case)
    n, t = planfile.to_objects(flat)
    exp = case["expected"]["budgeted"]
    if "error" in exp:
        with pytest.raises(BudgetInfeasible):
            sliced_execute(n, t, mem_budget=exp["budget"])
        return
    out = sliced_execute(n, t, mem_budget=exp["budget"])
    assert [flat.indices.index(ix) for ix in out.sliced_indices] == exp["chosen"]
    assert out.mem_estimate == int(exp["mem_estimate"]) <= exp["budget"]
    assert out.peak_observed == int(exp["peak_observed"]) <= out.mem_estimate
    assert out.num_slices == exp["num_slices"]
    got = _aligned(out.result, flat.indices, exp["indices"])
    assert np.allclose(got, hexvals(exp["values"]), rtol=RTOL, atol=1e-10)


@pytest.mark.parametrize("case", [c for c in CASES if c["family"] == "random_network"],
                         ids=[c["name"] for c in CASES if c["family"] == "random_network"])
def test_explicit_slice_sets_and_infeasible(case):
    flat = case_flat(case)
    n, t = planfile.to_objects(flat)
    with pytest.raises(BudgetInfeasible):
        sliced_execute(n, t, mem_budget=1)
    for ex in case["expected"]["explicit"]:
        out = sliced_execute(n, t, slice_indices=[flat.indices[i] for i in ex["ids"]])
        got = _aligned(out.result, flat.indices, ex["indices"])
        assert np.allclose(got, hexvals(ex["values"]), rtol=RTOL, atol=1e-12)


def test_known_answers_exact():
    for c in CASES:
        if c["family"] != "cnf":
            continue
        flat = case_flat(c)
        n, t = planfile.to_objects(flat)
        got = float(np.asarray(sliced_execute(n, t).result.values))
        if c["expected"]["known"] is not None:
            assert got == pytest.approx(c["expected"]["known"], rel=1e-12, abs=1e-12), c["name"]
        if c["name"].startswith("cnf_psi") or c["name"] in ("cnf_example4", "cnf_three_free", "cnf_or2"):
            assert got == c["expected"]["known"]  # unweighted: exact
        assert got == pytest.approx(c["expected"]["brute_force"], rel=1e-9, abs=1e-12)


def _rand_tensor(rng, inds):
    shape = [i.domain_size for i in inds]
    return Tensor(tuple(inds), rng.uniform(-2, 2, size=shape) if shape else np.array(rng.uniform(-2, 2)))


def test_contract_pair_random_vs_oracle():
    # test_tensor.py:87-95 pattern with larger ranks so every kernel class runs
    rng = np.random.default_rng(11)
    pool2 = [Index(f"q{k}", 2) for k in range(28)]
    pool3 = [Index(f"t{k}", 3) for k in range(10)]
    for trial in range(60):
        pool = pool3 if trial % 4 == 0 else pool2
        hi = 6 if pool is pool3 else 18
        ia = list(rng.choice(len(pool), int(rng.integers(0, hi)), replace=False))
        ib = list(rng.choice(len(pool), int(rng.integers(0, hi)), replace=False))
        a = _rand_tensor(rng, [pool[k] for k in ia])
        b = _rand_tensor(rng, [pool[k] for k in ib])
        out = contract_pair(a, b)
        sh = [i for i in a.indices if i in b.index_set()]
        want = np.tensordot(a.values, b.values, axes=([a.indices.index(i) for i in sh], [b.indices.index(i) for i in sh]))
        assert list(out.indices) == [i for i in a.indices if i not in b.index_set()] + \
            [i for i in b.indices if i not in a.index_set()]
        assert np.allclose(out.values, want, rtol=1e-12, atol=1e-12), trial


def test_random_networks_vs_oracle_with_slicing():
    rng = random.Random(99)
    for trial in range(30):
        k = rng.randint(2, 9)
        dom = 3 if trial % 3 == 0 else 2
        bonds = [Index(("b", j), rng.randint(2, dom)) for j in range(k - 1)]
        ts = []
        for j in range(k):
            inds = ([bonds[j - 1]] if j else []) + ([bonds[j]] if j < k - 1 else [])
            if rng.random() < 0.3:
                inds.append(Index(("f", j), rng.randint(2, dom)))
            shape = [i.domain_size for i in inds]
            ts.append(Tensor(tuple(inds), np.array([rng.uniform(-1, 1) for _ in range(int(np.prod(shape)))]).reshape(shape)))
        n = TensorNetwork(tuple(ts))
        t = left_deep_tree(n.tensors)
        from paper_2006_15512_b200.flatten import flatten
        flat = flatten(n, t)
        full = oracle.mem_cost(flat)
        budget = max(8, int(full * 0.6))
        try:
            want = oracle.sliced_execute(flat, mem_budget=budget)
        except oracle.BudgetInfeasible:
            with pytest.raises(BudgetInfeasible):
                sliced_execute(n, t, mem_budget=budget)
            continue
        out = sliced_execute(n, t, mem_budget=budget)
        assert [flat.indices.index(i) for i in out.sliced_indices] == want["chosen"]
        assert out.mem_estimate == want["mem_estimate"] and out.peak_observed == want["peak_observed"]
        got = _aligned(out.result, flat.indices, want["indices"])
        assert np.allclose(got, want["values"], rtol=1e-12, atol=1e-12)


def test_plan_mismatch_raised():
    i = Index("i", 2)
    a = Tensor((i,), np.ones(2))
    n = TensorNetwork((a, Tensor((i,), np.ones(2))))
    with pytest.raises(PlanMismatch):
        execute(n, join(leaf(a), leaf(Tensor((i,), np.ones(2)))))


def test_single_leaf_and_rank0():
    s = Tensor((), np.array(2.5))
    n = TensorNetwork((s,))
    assert float(np.asarray(sliced_execute(n, leaf(s)).result.values)) == 2.5
    i = Index("i", 3)
    a = Tensor((i,), np.array([1.0, 2.0, 3.0]))
    assert float(np.asarray(contract_pair(a, a).values)) == 14.0  # test_tensor.py:81-85


def _plan(name):
    flat, meta = planfile.load(os.path.join(PLANS, f"{name}.tcplan.npz"))
    return flat, meta


@pytest.mark.parametrize("name", ["c1a", "c1a_unweighted", "c2"])
def test_benchmark_plans_match_reference_counts(name, golden_counts):
    flat, _ = _plan(name)
    n, t = planfile.to_objects(flat)
    out = sliced_execute(n, t)
    got = float(np.asarray(out.result.values))
    want = golden_counts[name]["count"]
    assert abs(got - want) <= RTOL * abs(want)
    assert out.mem_estimate == int(golden_counts[name]["mem_estimate"])
    assert out.peak_observed == int(golden_counts[name]["peak_observed"])
    if name.endswith("unweighted"):
        assert got == want  # integer count < 2^53: exact


def test_bitwise_determinism_and_slice_partition():
    """Reruns are bitwise identical (test_acceptance.py:357-372), and any block
    partition of the lexicographic slice ids folds to the same bits (the
    multi-device / multi-rank invariant)."""
    flat, _ = _plan("c1a")
    h = _lib.PlanHandle(flat)
    chosen = []
    for _ in range(4):
        chosen.append(h.choose_slice_index(chosen))
    ex = _lib.Exec(h, chosen, 0)
    ex.run(0, 16)
    full, per = ex.fetch(16)
    ex.run(0, 16)
    again, per2 = ex.fetch(16)
    assert np.array_equal(per, per2) and full.tobytes() == again.tobytes()
    parts = []
    for b, e in ((0, 5), (5, 11), (11, 16)):
        ex.run(b, e)
        parts.append(ex.fetch(e - b)[1])
    cat = np.concatenate(parts)
    assert np.array_equal(cat, per)
    acc = cat[0]
    for s in range(1, 16):
        acc = acc + cat[s]
    assert acc.tobytes() == full.tobytes()
    # and the slice sum equals the unsliced count
    n, t = planfile.to_objects(flat)
    un = float(np.asarray(sliced_execute(n, t).result.values))
    assert abs(float(full[0]) - un) <= 1e-12 * abs(un)
    sl = sliced_execute(n, t, slice_indices=[flat.indices[i] for i in chosen])
    assert float(np.asarray(sl.result.values)).hex() == float(full[0]).hex()


def test_slicing_identity_at_full_size():
    """C1b (rank-30 intermediates) sliced 2 ways equals the unsliced count."""
    flat, _ = _plan("c1b")
    n, t = planfile.to_objects(flat)
    un = float(np.asarray(sliced_execute(n, t).result.values))
    h = _lib.PlanHandle(flat)
    c = [h.choose_slice_index([])]
    sl = sliced_execute(n, t, slice_indices=[flat.indices[i] for i in c])
    assert sl.num_slices == 2
    got = float(np.asarray(sl.result.values))
    assert abs(got - un) <= 1e-12 * abs(un)
    gold = json.load(open(os.path.join(GOLDEN, "counts.json")))["c1b"]["count"]
    assert abs(un - gold) <= RTOL * abs(gold)
