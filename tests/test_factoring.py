"""Native FactorTree step (paper_2006_15512_b200/factoring.py, csrc/factor.cpp)
against the reference's ``factor_branch_audit`` (factoring.py:270-333).

* golden: 35 reference runs frozen in tests/golden/factor.json
  (make_factor_golden.py) — the same plan text, pieces (index ids, values)
  and widths, rebuilt from the fixture alone (no reference needed);
* live: the unmodified reference side by side on random CNFs, free-index
  networks and the C1a / C2 benchmark formulas (skipped without it);
* the reference's own test files with only the factoring swapped in
  (``TC_REFSUITE_PATCH=factoring``: reference execution, so CPU-only).
"""

import ast
import json
import os
import random
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2006_15512_b200.errors import InvalidDecomposition, NotFactorable, TooManyFreeIndices
from paper_2006_15512_b200.factoring import factor_branch_audit
from paper_2006_15512_b200.network import ContractionTree, TensorNetwork
from paper_2006_15512_b200.tensor import Index, Tensor


def serialize(m, t):
    """serialize_plan (reference network.py:235-258)."""
    num = {id(x): k for k, x in enumerate(m.tensors)}
    nxt, lines, slot = len(m.tensors), [], {}
    for node in t.postorder():
        if node.is_leaf:
            slot[id(node)] = num[id(node.tensor)]
        else:
            slot[id(node)] = nxt
            lines.append(f"contract {slot[id(node.left)]} {slot[id(node.right)]} -> {nxt}")
            nxt += 1
    return "\n".join(lines) + ("\n" if lines else "")


class _Tree:
    """The two views of a networkx tree the factoring reads (nodes, adj)."""

    def __init__(self, nodes, adj):
        self.nodes = nodes
        self.adj = {u: [nodes[w] for w in a] for u, a in zip(nodes, adj)}


class _BD:
    def __init__(self, tree, leaf_map):
        self.tree, self.leaf_map = tree, leaf_map


def _dense(entries, shape):
    v = np.zeros(int(np.prod(shape)) if shape else 1)
    for k, h in entries:
        v[k] = float.fromhex(h)
    return v.reshape(shape)


def _golden():
    with open(os.path.join(GOLDEN, "factor.json")) as fh:
        return json.load(fh)


GOLDEN_CASES = _golden()


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=[c["name"] for c in GOLDEN_CASES])
def test_golden_matches_reference(case):
    indices = [Index(ast.literal_eval(i), d) for i, d in case["indices"]]
    tensors = []
    for t in case["tensors"]:
        inds = tuple(indices[k] for k in t["idx"])
        tensors.append(Tensor(inds, _dense(t["val"], tuple(ix.domain_size for ix in inds))))
    n = TensorNetwork(tuple(tensors))
    nodes = [ast.literal_eval(s) for s in case["bd_nodes"]]
    bd = _BD(_Tree(nodes, case["bd_adj"]), {nodes[u]: indices[i] for u, i in case["bd_leaf_map"]})
    r = factor_branch_audit(n, bd)
    assert (r.branch_width, r.carving_width) == (case["branch_width"], case["carving_width"])
    assert serialize(r.network, r.tree) == case["plan"]
    assert len(r.network.tensors) == len(case["pieces"])
    for p, want in zip(r.network.tensors, case["pieces"]):
        assert [repr(ix.id) for ix in p.indices] == want["ids"]
        assert [ix.domain_size for ix in p.indices] == want["dom"]
        got = p.values.ravel()
        nz = got.nonzero()[0]
        assert [[int(k), float(got[k]).hex()] for k in nz] == want["val"]
    # pieces come from the original tensors (piece_map), every tensor covered
    assert set(map(id, r.piece_map.values())) == set(map(id, n.tensors))


def test_errors_match_reference_messages():
    a, b, c, d = (Index(k, 2) for k in "abcd")
    dense = Tensor((a, b, c), np.arange(8.0).reshape(2, 2, 2))
    n = TensorNetwork((dense, Tensor((a,), np.ones(2)), Tensor((b,), np.ones(2)), Tensor((c,), np.ones(2))))
    # caterpillar over the three bonds a, b, c (reference decomposition.py:426-448)
    nodes = [("leaf", 0), ("leaf", 1), ("leaf", 2), ("spine", 3)]
    bd = _BD(_Tree(nodes, [[3], [3], [3], [0, 1, 2]]), {nodes[0]: a, nodes[1]: b, nodes[2]: c})
    with pytest.raises(NotFactorable, match=r"tensor #0 is neither a diagonal nor an acceptance tensor"):
        factor_branch_audit(n, bd)
    bad = _BD(_Tree(nodes, [[3], [3], [3], [0, 1, 2]]), {nodes[0]: a, nodes[1]: b})
    with pytest.raises(InvalidDecomposition, match="leaves are not a bijection"):
        factor_branch_audit(n, bad)
    free = TensorNetwork(tuple(Tensor((Index(("f", k), 2),), np.ones(2)) for k in range(4)))
    with pytest.raises(TooManyFreeIndices, match="4 free indices, at most 3 allowed"):
        factor_branch_audit(free, None)
    # a width-0 decomposition falls back to the component-wise plan
    i = Index("i", 2)
    two = TensorNetwork((Tensor((i,), np.array([1.0, 2.0])), Tensor((i,), np.array([3.0, 4.0]))))
    r = factor_branch_audit(two, _BD(_Tree([("leaf", 0)], [[]]), {("leaf", 0): i}))
    assert r.network is two and r.carving_width == -1 and isinstance(r.tree, ContractionTree)


# ---------------------------------------------------------------------------
# live comparison with the unmodified reference (this container only)

def _reference():
    for p in (os.path.join(ROOT, "oracle", "_ref"), os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "tensorcount")):
            if p not in sys.path:
                sys.path.insert(1, p)
            try:
                import tensorcount  # noqa: F401
                return True
            except Exception:
                return False
    return False


needs_ref = pytest.mark.skipif(not _reference(), reason="reference not importable")


def rand_dimacs(rng, nv, nc, k):
    lines = [f"p cnf {nv} {nc}"]
    lines += [f"w {v} {rng.uniform(0, 1):.6f} {rng.uniform(0, 1):.6f}" for v in range(1, nv + 1)]
    for _ in range(nc):
        vs = rng.sample(range(1, nv + 1), min(k, nv))
        lines.append(" ".join(str(v if rng.random() < 0.5 else -v) for v in vs) + " 0")
    return "\n".join(lines) + "\n"


def _same(r1, r2):
    from tensorcount.network import serialize_plan

    assert (r1.branch_width, r1.carving_width) == (r2.branch_width, r2.carving_width)
    assert serialize_plan(r1.network, r1.tree) == serialize_plan(r2.network, r2.tree)
    for p1, p2 in zip(r1.network.tensors, r2.network.tensors, strict=True):
        assert [ix.id for ix in p1.indices] == [ix.id for ix in p2.indices]
        assert np.array_equal(p1.values, p2.values)
        assert r1.piece_map[id(p1)] is r2.piece_map[id(p2)]


@needs_ref
def test_live_random_formulas_and_decompositions():
    from tensorcount import factoring as RF
    from tensorcount.decomposition import caterpillar_branch_decomposition, min_fill_tree_decomposition, tree_to_branch
    from tensorcount.formula import parse_dimacs
    from tensorcount.network import structure_graph
    from tensorcount.reduction import reduce_formula

    rng = random.Random(99)
    done = 0
    for trial in range(80):
        nv = rng.randint(2, 14)
        f, w = parse_dimacs(rand_dimacs(rng, nv, rng.randint(1, 3 * nv), rng.randint(1, 4)))
        n = reduce_formula(f, w)
        g = structure_graph(n)
        if not g.edges:
            continue
        for bd in (tree_to_branch(min_fill_tree_decomposition(g, seed=trial), g), caterpillar_branch_decomposition(g)):
            _same(RF.factor_branch_audit(n, bd, g), factor_branch_audit(n, bd, g))
            done += 1
    assert done > 100


@needs_ref
@pytest.mark.parametrize("config", ["c1a", "c2"])
def test_live_benchmark_formulas(config):
    from tensorcount import factoring as RF
    from tensorcount.decomposition import min_fill_tree_decomposition, tree_to_branch
    from tensorcount.formula import parse_dimacs
    from tensorcount.network import structure_graph
    from tensorcount.reduction import reduce_formula

    from paper_2006_15512_b200.generators import config_dimacs

    f, w = parse_dimacs(config_dimacs(config))
    n = reduce_formula(f, w)
    g = structure_graph(n)
    bd = tree_to_branch(min_fill_tree_decomposition(g, seed=0), g)
    _same(RF.factor_branch_audit(n, bd, g), factor_branch_audit(n, bd, g))


@needs_ref
def test_reference_suite_with_native_host_steps():
    """All 208 reference tests with the native planning heuristics,
    tree_to_branch and FactorTree swapped in (execution stays on the
    reference's CPU path)."""
    suite = os.path.join(ROOT, "tests", "reference_suite")
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", TC_REFSUITE_PATCH="host")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--confcutdir", suite,
                        "--rootdir", suite, suite], cwd=suite, env=env, capture_output=True, text=True, timeout=1800)
    m = re.search(r"(\d+) passed", p.stdout)
    assert p.returncode == 0 and m and int(m.group(1)) == 208, p.stdout[-3000:] + p.stderr[-2000:]


@needs_ref
def test_reduction_matches_reference():
    """reduction.py: the same network as the reference's reduce_formula
    (reduction.py:80-101), object for object: index ids and order, values."""
    from tensorcount import tensor as RT
    from tensorcount.formula import CnfFormula, WeightFunction, parse_dimacs
    from tensorcount.network import TensorNetwork as RN
    from tensorcount.reduction import reduce_formula as ref_reduce

    from paper_2006_15512_b200.generators import config_dimacs
    from paper_2006_15512_b200.reduction import reduce_formula

    rng = random.Random(3)
    texts = [config_dimacs("c1a"), "p cnf 3 0\n", "p cnf 2 1\n0\n", "p cnf 0 0\n"]
    texts += [rand_dimacs(rng, rng.randint(1, 12), rng.randint(0, 30), rng.randint(1, 4)) for _ in range(60)]
    forms = [parse_dimacs(t) for t in texts]
    forms.append((CnfFormula(3, ((1, -2), (3,), ())), WeightFunction({1: (0.25, 0.75)})))
    for f, w in forms:
        want = ref_reduce(f, w)
        got = reduce_formula(f, w, RT.Index, RT.Tensor, RN)
        assert len(got.tensors) == len(want.tensors)
        for a, b in zip(got.tensors, want.tensors):
            assert [ix.id for ix in a.indices] == [ix.id for ix in b.indices]
            assert a.values.shape == b.values.shape and np.array_equal(a.values, b.values)


@needs_ref
def test_patched_plan_metadata_matches_reference():
    """max_rank / serialize_plan / time_cost of the patched driver (native plan)
    equal the reference's on C2's plan (network.py:178-201, 235-258)."""
    import subprocess as sp

    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import tensorcount\n"
        "from tensorcount.driver import plan_contraction\n"
        "from tensorcount.formula import parse_dimacs\n"
        "from tensorcount import network as RN\n"
        "from tensorcount import driver as RD\n"
        "from tensorcount.reduction import reduce_formula\n"
        "from paper_2006_15512_b200 import reference_patch\n"
        "from paper_2006_15512_b200.generators import config_dimacs\n"
        "f, w = parse_dimacs(config_dimacs('c2')); n = reduce_formula(f, w)\n"
        "best, _, _ = plan_contraction(n, planner_spec='minfill', alpha=0.0, seed=0)\n"
        "m, t = best.network, best.tree\n"
        "a = (RN.max_rank(m, t), RN.serialize_plan(m, t), RD.time_cost(m, t))\n"
        "reference_patch.install(tensorcount, execution=False)\n"
        "b = (RN.max_rank(m, t), RN.serialize_plan(m, t), RD.time_cost(m, t))\n"
        "assert a == b, (a[0], b[0], a[2], b[2])\n"
        "print('same')\n") % (ROOT, [p for p in sys.path if p.endswith("_ref") or p.endswith("pkg/src")][0])
    out = sp.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "same" in out.stdout, out.stdout + out.stderr
