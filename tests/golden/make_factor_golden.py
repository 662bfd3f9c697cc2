"""Golden fixtures for the native FactorTree step, made by the UNMODIFIED reference.

    python tests/golden/make_factor_golden.py     -> tests/golden/factor.json

Each case holds the reference's INPUT to ``factor_branch_audit``
(``factoring.py:270-333``) — the reduced network (``reduce_formula``, or a
hand-built network with free indices) and a branch decomposition
(``tree_to_branch(min_fill_tree_decomposition(g, seed))`` or
``caterpillar_branch_decomposition``) with its networkx node / adjacency order
and node labels — and its OUTPUT: ``serialize_plan(M, T)`` (``network.py:235-258``),
every piece's index ids and values (float.hex), branch and carving width.
``tests/test_factoring.py`` rebuilds the inputs from this file (no reference
needed on the GPU box) and checks the native result against it.
Needs the reference importable (oracle/_ref or /root/reference/pkg/src).
"""

from __future__ import annotations

import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(p):
        sys.path.insert(1, p)
        break

from tensorcount.decomposition import (  # noqa: E402
    caterpillar_branch_decomposition, min_fill_tree_decomposition, tree_to_branch)
from tensorcount.factoring import factor_branch_audit  # noqa: E402
from tensorcount.formula import parse_dimacs  # noqa: E402
from tensorcount.network import TensorNetwork, serialize_plan, structure_graph  # noqa: E402
from tensorcount.reduction import copy_tensor, reduce_formula  # noqa: E402
from tensorcount.tensor import Index  # noqa: E402

from paper_2006_15512_b200.generators import config_dimacs  # noqa: E402


def rand_dimacs(rng, nv, nc, k):
    lines = [f"p cnf {nv} {nc}"]
    for v in range(1, nv + 1):
        lines.append(f"w {v} {rng.uniform(0, 1):.6f} {rng.uniform(0, 1):.6f}")
    for _ in range(nc):
        vs = rng.sample(range(1, nv + 1), min(k, nv))
        lines.append(" ".join(str(v if rng.random() < 0.5 else -v) for v in vs) + " 0")
    return "\n".join(lines) + "\n"


def free_network(rng):
    """Copy tensors over shared bonds plus up to three free indices."""
    k = rng.randint(2, 6)
    pool = [Index(("e", j), 2) for j in range(k)] * 2 + [Index(("f", j), 2) for j in range(rng.randint(1, 3))]
    rng.shuffle(pool)
    groups, cur = [], []
    for ix in pool:
        if ix in cur or len(cur) >= 3:
            groups.append(cur)
            cur = []
        cur.append(ix)
    groups.append(cur)
    return TensorNetwork(tuple(copy_tensor(tuple(gq), rng.uniform(0.1, 2), rng.uniform(0.1, 2))
                               for gq in groups if gq))


def sparse(values):
    """[flat position, float.hex] of the nonzero entries (row-major)."""
    flat = values.ravel()
    return [[int(k), float(flat[k]).hex()] for k in flat.nonzero()[0]]


def encode(name, n, bd, res):
    ipos, indices = {}, []
    tensors = []
    for t in n.tensors:
        ids = []
        for ix in t.indices:
            if ix not in ipos:
                ipos[ix] = len(indices)
                indices.append(ix)
            ids.append(ipos[ix])
        tensors.append(dict(idx=ids, val=sparse(t.values)))
    nodes = list(bd.tree.nodes)
    npos = {u: k for k, u in enumerate(nodes)}
    return dict(
        name=name,
        indices=[[repr(ix.id), ix.domain_size] for ix in indices],
        tensors=tensors,
        bd_nodes=[repr(u) for u in nodes],
        bd_adj=[[npos[w] for w in bd.tree.adj[u]] for u in nodes],
        bd_leaf_map=[[npos[u], ipos[e]] for u, e in bd.leaf_map.items()],
        plan=serialize_plan(res.network, res.tree),
        pieces=[dict(ids=[repr(ix.id) for ix in p.indices], dom=[ix.domain_size for ix in p.indices],
                     val=sparse(p.values)) for p in res.network.tensors],
        branch_width=res.branch_width,
        carving_width=res.carving_width,
    )


def main():
    rng = random.Random(20261017)
    cases = []
    f, w = parse_dimacs(config_dimacs("c1a"))
    n = reduce_formula(f, w)
    g = structure_graph(n)
    bd = tree_to_branch(min_fill_tree_decomposition(g, seed=0), g)
    cases.append(encode("c1a", n, bd, factor_branch_audit(n, bd, g)))
    while len(cases) < 25:
        nv = rng.randint(2, 10)
        f, w = parse_dimacs(rand_dimacs(rng, nv, rng.randint(1, 3 * nv), rng.randint(1, 4)))
        n = reduce_formula(f, w)
        g = structure_graph(n)
        if not g.edges:
            continue
        seed = len(cases)
        for kind, bd in (("minfill", tree_to_branch(min_fill_tree_decomposition(g, seed=seed), g)),
                         ("caterpillar", caterpillar_branch_decomposition(g))):
            cases.append(encode(f"cnf{len(cases)}-{kind}", n, bd, factor_branch_audit(n, bd, g)))
    while len(cases) < 35:
        n = free_network(rng)
        g = structure_graph(n)
        bd = tree_to_branch(min_fill_tree_decomposition(g, seed=len(cases)), g)
        cases.append(encode(f"free{len(cases)}", n, bd, factor_branch_audit(n, bd, g)))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "factor.json")
    with open(out, "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print(out, len(cases), "cases")


if __name__ == "__main__":
    main()
