"""Golden fixtures for the native planning heuristics, made by the UNMODIFIED reference.

    python tests/golden/make_decomp_golden.py     -> tests/golden/decomp.json

Each case is a multigraph (vertices ``v000000``.., edge ids ``e000000``.. so
that str order is index order) from a reduced random CNF's structure graph
(``reduction.py`` + ``network.structure_graph``, relabelled order-preserving)
and what the reference builds from it with ``fresh_node``'s counter reset to 0:
``min_fill_tree_decomposition`` / ``min_degree_tree_decomposition``
(``decomposition.py:297-340``: node names, node and adjacency order, bags) and
``tree_to_branch`` of it (``:346-411``: tree and leaf map in order).
Needs the reference importable (oracle/_ref or /root/reference/pkg/src).
"""

from __future__ import annotations

import itertools
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

import tensorcount.decomposition as D  # noqa: E402
from tensorcount.formula import parse_dimacs  # noqa: E402
from tensorcount.graphs import Graph  # noqa: E402
from tensorcount.network import structure_graph  # noqa: E402
from tensorcount.reduction import reduce_formula  # noqa: E402


def rand_dimacs(rng, nv, nc, k):
    lines = [f"p cnf {nv} {nc}"]
    lines += [f"w {v} {rng.uniform(0, 1):.6f} {rng.uniform(0, 1):.6f}" for v in range(1, nv + 1)]
    for _ in range(nc):
        vs = rng.sample(range(1, nv + 1), min(k, nv))
        lines.append(" ".join(str(v if rng.random() < 0.5 else -v) for v in vs) + " 0")
    return "\n".join(lines) + "\n"


def relabel(g):
    verts = sorted(g.vertices, key=str)
    vid = {v: f"v{k:06d}" for k, v in enumerate(verts)}
    edges = sorted(g.edges, key=str)
    h = Graph(vertices=set(vid.values()), edges={})
    for k, e in enumerate(edges):
        a, b = tuple(g.endpoints(e))
        h.add_edge(f"e{k:06d}", vid[a], vid[b])
    return h, [sorted((int(vid[a][1:]), int(vid[b][1:]))) for a, b in (tuple(g.endpoints(e)) for e in edges)]


def tree_json(tree):
    nodes = list(tree.nodes)
    pos = {u: k for k, u in enumerate(nodes)}
    return [list(u) for u in nodes], [[pos[w] for w in tree.adj[u]] for u in nodes]


def main():
    rng = random.Random(20261018)
    cases = []
    while len(cases) < 40:
        nv = rng.randint(2, 24)
        f, w = parse_dimacs(rand_dimacs(rng, nv, rng.randint(1, 4 * nv), rng.randint(2, 4)))
        g, edges = relabel(structure_graph(reduce_formula(f, w)))
        if not g.edges:
            continue
        seed = len(cases)
        kind = "minfill" if seed % 2 == 0 else "mindegree"
        build = D.min_fill_tree_decomposition if kind == "minfill" else D.min_degree_tree_decomposition
        D._fresh = itertools.count(0)
        td = build(g, seed)
        td_nodes, td_adj = tree_json(td.tree)
        bags = [sorted(int(x[1:]) for x in td.bags[tuple(u)]) for u in td_nodes]
        bd = D.tree_to_branch(td, g)
        bd_nodes, bd_adj = tree_json(bd.tree)
        pos = {tuple(u): k for k, u in enumerate(bd_nodes)}
        cases.append(dict(nv=len(g.vertices), edges=edges, kind=kind, seed=seed, td_nodes=td_nodes, td_adj=td_adj,
                          bags=bags, bd_nodes=bd_nodes, bd_adj=bd_adj,
                          leaf_map=[[pos[u], int(e[1:])] for u, e in bd.leaf_map.items()]))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "decomp.json")
    with open(out, "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print(out, len(cases), "cases")


if __name__ == "__main__":
    main()
