"""Pin the CPU oracle (oracle/tc_oracle.c) against fixtures produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import case_flat, hexvals, load_cases
from oracle import oracle

CASES = load_cases()


def _close(got, want, rtol=1e-12, atol=1e-14):
    return np.allclose(got, want, rtol=rtol, atol=atol)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_unsliced_matches_reference(case):
    flat = case_flat(case)
    exp = case["expected"]["unsliced"]
    out = oracle.sliced_execute(flat)
    assert out["indices"] == exp["indices"]  # kept_a ++ kept_b order (tensor.py:108)
    assert _close(out["values"], hexvals(exp["values"]))
    assert out["mem_estimate"] == int(exp["mem_estimate"])
    assert out["peak_observed"] == int(exp["peak_observed"])
    assert out["num_slices"] == exp["num_slices"] == 1


@pytest.mark.parametrize("case", [c for c in CASES if "budgeted" in c["expected"]],
                         ids=[c["name"] for c in CASES if "budgeted" in c["expected"]])
def test_oracle_budgeted_matches_reference(case):
    flat = case_flat(case)
    exp = case["expected"]["budgeted"]
    if "error" in exp:
        with pytest.raises(oracle.BudgetInfeasible):
            oracle.sliced_execute(flat, mem_budget=exp["budget"])
        return
    out = oracle.sliced_execute(flat, mem_budget=exp["budget"])
    assert out["chosen"] == exp["chosen"]  # identical greedy picks (slicing.py:70-79)
    assert out["mem_estimate"] == int(exp["mem_estimate"])
    assert out["peak_observed"] == int(exp["peak_observed"])
    assert out["num_slices"] == exp["num_slices"]
    assert out["indices"] == exp["indices"]
    assert _close(out["values"], hexvals(exp["values"]))


@pytest.mark.parametrize("case", [c for c in CASES if c["family"] == "random_network"],
                         ids=[c["name"] for c in CASES if c["family"] == "random_network"])
def test_oracle_memory_model_and_greedy(case):
    flat = case_flat(case)
    exp = case["expected"]
    for k, v in exp["mem_cost"].items():
        drop = [int(k)] if k else []
        assert oracle.mem_cost(flat, drop) == int(v)
    if "choose" in exp:
        assert oracle.choose_slice_index(flat) == exp["choose"]
    with pytest.raises(oracle.BudgetInfeasible):
        oracle.sliced_execute(flat, mem_budget=1)
    for ex in exp["explicit"]:
        out = oracle.sliced_execute(flat, slice_ids=ex["ids"])
        want = hexvals(ex["values"])
        # align index order (slice sums keep the first part's order)
        assert sorted(out["indices"]) == sorted(ex["indices"])
        if out["indices"] != ex["indices"]:
            shape_o = [int(flat.domain[i]) for i in out["indices"]]
            perm = [out["indices"].index(i) for i in ex["indices"]]
            got = np.transpose(out["values"].reshape(shape_o), perm).reshape(-1)
        else:
            got = out["values"]
        assert _close(got, want, rtol=1e-9, atol=1e-12)


def test_oracle_known_answers():
    for c in CASES:
        if c["family"] != "cnf":
            continue
        out = oracle.sliced_execute(case_flat(c))
        known = c["expected"]["known"]
        bf = c["expected"]["brute_force"]
        got = float(out["values"][0])
        if known is not None:
            assert got == pytest.approx(known, rel=1e-12, abs=1e-12), c["name"]
        assert got == pytest.approx(bf, rel=1e-9, abs=1e-12), c["name"]
