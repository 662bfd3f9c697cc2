"""The drop-in: patch the unmodified reference package so its own public API
(count_formula / count_text, driver.py:217-254) executes on the B200, and
check it against the reference's own oracle (brute_force_count,
formula.py:183-215) and known answers.  Needs the installed reference
(oracle/_ref or baseline/_ref); skipped if absent."""

import os
import random
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ref():
    for p in (os.path.join(ROOT, "oracle", "_ref"), os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "tensorcount")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import tensorcount

            return tensorcount
    pytest.skip("reference not installed")


@pytest.fixture
def patched():
    tc = _ref()
    from paper_2006_15512_b200 import reference_patch

    reference_patch.install(tc)
    yield tc
    reference_patch.uninstall()


EXAMPLE4 = "p cnf 4 4\n1 2 -3 0\n1 3 4 0\n-2 -3 0\n-3 -4 0\n"


def test_worked_example_and_known_answers(patched):
    tc = patched
    assert tc.driver.sliced_execute.__module__ != "tensorcount.slicing"
    assert abs(tc.count_text(EXAMPLE4, alpha=0.0).count - 7.0) <= 1e-12  # test_acceptance.py:85-90
    assert tc.count_text("p cnf 2 1\nw 1 0.25\n1 2 0\n", alpha=0.0).count == pytest.approx(1.25)
    assert tc.count_text("p cnf 3 0\n", alpha=0.0).count == 8.0
    assert tc.count_text("p cnf 2 1\n0\n", alpha=0.0).count == 0.0


def test_budget_forces_slicing(patched):
    tc = patched
    free = tc.count_text(EXAMPLE4, alpha=0.0)
    out = tc.count_text(EXAMPLE4, alpha=0.0, mem_budget=free.mem_estimate - 1)  # test_driver.py:171-177
    assert out.num_slices > 1 and abs(out.count - 7.0) <= 1e-9
    assert out.peak_observed <= out.mem_estimate <= free.mem_estimate - 1


def test_reference_exception_classes(patched):
    tc = patched
    from tensorcount.errors import BudgetInfeasible

    with pytest.raises(BudgetInfeasible):
        tc.count_text(EXAMPLE4, alpha=0.0, mem_budget=1)


def test_random_suite_vs_brute_force(patched):
    tc = patched
    from tensorcount.formula import CnfFormula, WeightFunction, brute_force_count

    rng = random.Random(20240817)
    for k in range(40):  # test_acceptance.py:75-79 pattern
        nv, nc = rng.randint(5, 14), rng.randint(5, 40)
        clauses = []
        for _ in range(nc):
            vs = rng.sample(range(1, nv + 1), 3)
            clauses.append(tuple(v if rng.random() < 0.5 else -v for v in vs))
        f = CnfFormula(nv, tuple(clauses))
        w = WeightFunction({v: (rng.uniform(0, 1), rng.uniform(0, 1)) for v in range(1, nv + 1)})
        got = tc.count_formula(f, w, alpha=0.0, seed=k).count
        assert got == pytest.approx(brute_force_count(f, w), rel=1e-9, abs=1e-12), k


def test_determinism_through_driver(patched):
    tc = patched
    a = tc.count_text(EXAMPLE4, alpha=0.0, seed=3)
    b = tc.count_text(EXAMPLE4, alpha=0.0, seed=3)
    assert a.count == b.count and a.plan_text == b.plan_text  # test_acceptance.py:357-372


def test_random_suite_sliced_vs_brute_force(patched):
    """Real FactorTree networks (tied copy pieces) under budgets that make the
    greedy slice 1-6 bonds, often inside tie classes (implied slices)."""
    tc = patched
    from tensorcount import driver
    from tensorcount.formula import CnfFormula, WeightFunction, brute_force_count

    from paper_2006_15512_b200 import _lib
    from paper_2006_15512_b200.flatten import flatten

    plans = []
    real = driver.sliced_execute

    def capture(n, t, mem_budget=None):  # the planned network of this formula
        plans.append((n, t))
        return real(n, t, mem_budget=mem_budget)

    rng = random.Random(777)
    sliced = 0
    for k in range(60):
        nv, nc = rng.randint(6, 14), rng.randint(8, 40)
        clauses = []
        for _ in range(nc):
            vs = rng.sample(range(1, nv + 1), 3)
            clauses.append(tuple(v if rng.random() < 0.5 else -v for v in vs))
        f = CnfFormula(nv, tuple(clauses))
        w = WeightFunction({v: (rng.uniform(0, 1), rng.uniform(0, 1)) for v in range(1, nv + 1)})
        driver.sliced_execute = capture
        try:
            tc.count_formula(f, w, alpha=0.0, seed=k)
        finally:
            driver.sliced_execute = real
        n, t = plans[-1]
        h = _lib.PlanHandle(flatten(n, t))
        picks = []
        for _ in range(min(6, h.info().num_bonds)):
            picks.append(h.choose_slice_index(picks))
            budget = h.mem_cost(picks)
            out = tc.count_formula(f, w, alpha=0.0, seed=k, mem_budget=budget)
            sliced += out.num_slices > 1
            assert out.count == pytest.approx(brute_force_count(f, w), rel=1e-9, abs=1e-12), (k, len(picks))
            if len(picks) >= 1 + k % 4:
                break
    assert sliced > 60
