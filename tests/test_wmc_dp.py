"""Pin the exact clause-frontier counter (oracle/wmc_dp.c, test
infrastructure) before it anchors the sliced configs: against the reference's
golden counts (tests/golden/counts.json, produced by the unmodified reference)
and against direct enumeration in the style of the reference's own oracle
``brute_force_count`` (formula.py:183-215).  CPU only."""

import itertools
import random

import pytest

from oracle import wmc_dp
from paper_2006_15512_b200.generators import config_dimacs, uniform_3cnf


def _enumerate(text, fix=None):
    n, clauses, weights = wmc_dp.parse(text)
    total = 0.0
    for bits in itertools.product((0, 1), repeat=n):
        if fix and any(bits[v - 1] != b for v, b in fix.items()):
            continue
        if all(any(bits[abs(l) - 1] == (l > 0) for l in c) for c in clauses):
            w = 1.0
            for v in range(1, n + 1):
                w *= weights.get(v, (1.0, 1.0))[bits[v - 1]]
            total += w
    return total


@pytest.mark.parametrize("name", ["c1a", "c1a_unweighted", "c1b", "c2"])
def test_dp_matches_reference_golden_counts(name, golden_counts):
    got, _ = wmc_dp.count(config_dimacs(name))
    want = golden_counts[name]["count"]
    if name.endswith("unweighted"):
        assert got == want  # integer count < 2^53: exact
    else:
        assert abs(got - want) <= 1e-12 * abs(want)


@pytest.mark.parametrize("seed", range(12))
def test_dp_matches_enumeration(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 12)
    text = uniform_3cnf(max(3, n), rng.choice([1.0, 2.0, 3.0, 4.5]), seed)
    fix = {v: rng.randint(0, 1) for v in rng.sample(range(1, 4), rng.randint(0, 2))}
    got, _ = wmc_dp.count(text, fix=fix)
    want = _enumerate(text, fix)
    assert abs(got - want) <= 1e-12 * max(abs(want), 1e-300)


def test_dp_reference_parse_rules():
    # tautologies dropped, duplicate literals removed, 'w v p' -> (1-p, p), empty clause -> 0
    assert wmc_dp.count("p cnf 2 2\n1 -1 0\n2 2 0\nw 2 0.25\n")[0] == pytest.approx(2 * 0.25)
    assert wmc_dp.count("p cnf 2 1\n0\n")[0] == 0.0
    assert wmc_dp.count("p cnf 3 0\n")[0] == 8.0
    assert wmc_dp.count("p cnf 2 1\nw 1 0.25\n1 2 0\n")[0] == pytest.approx(1.25)  # README.md:80-81
    ex4 = "p cnf 4 4\n1 2 -3 0\n1 3 4 0\n-2 -3 0\n-3 -4 0\n"
    assert wmc_dp.count(ex4)[0] == 7.0  # test_acceptance.py:57,85-90
