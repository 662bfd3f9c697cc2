"""Plan the benchmark configurations with the UNMODIFIED reference planner and
freeze them as ``data/plans/<name>.tcplan.npz``.

Pipeline: parse_dimacs → reduce_formula → structure_graph →
min_fill_tree_decomposition(g, seed=0) → tree_to_branch → factor_branch_audit
(reference ``driver.py:79-88``, ``factoring.py:270-333``).  Planning is out of
scope for the B200 stage; it runs here, on the CPU, once.

Usage:  python tools/make_plans.py c1a c2 ...   (needs the reference importable:
oracle/_ref, installed by ``__graft_entry__.build()``, or /root/reference).
"""

from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(p):
        sys.path.insert(1, p)
        break

from tensorcount.decomposition import min_fill_tree_decomposition, tree_to_branch  # noqa: E402
from tensorcount.factoring import factor_branch_audit  # noqa: E402
from tensorcount.formula import parse_dimacs  # noqa: E402
from tensorcount.network import contraction_ops, max_rank, structure_graph  # noqa: E402
from tensorcount.reduction import reduce_formula  # noqa: E402
from tensorcount.slicing import mem_cost  # noqa: E402

from paper_2006_15512_b200 import planfile  # noqa: E402
from paper_2006_15512_b200.flatten import flatten  # noqa: E402
from paper_2006_15512_b200.generators import CONFIGS, config_dimacs  # noqa: E402


def plan_text(text):
    f, w = parse_dimacs(text)
    n = reduce_formula(f, w)
    g = structure_graph(n)
    td = min_fill_tree_decomposition(g, seed=0)
    bd = tree_to_branch(td, g)
    res = factor_branch_audit(n, bd, g)
    return f, res


def main(names):
    os.makedirs(os.path.join(ROOT, "data", "plans"), exist_ok=True)
    for name in names:
        t0 = time.time()
        text = config_dimacs(name)
        f, res = plan_text(text)
        t_plan = time.time() - t0
        m, t = res.network, res.tree
        flat = flatten(m, t)
        meta = dict(
            config=name,
            generator=CONFIGS[name],
            num_vars=f.num_vars,
            num_clauses=len(f.clauses),
            leaves=flat.num_leaves,
            branch_width=res.branch_width,
            max_rank=max_rank(m, t),
            contraction_ops=int(contraction_ops(t)),
            mem_cost_unsliced=str(mem_cost(m, t)),
            planning_seconds=t_plan,
        )
        path = os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz")
        planfile.save(path, flat, meta)
        print(name, meta, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1a", "c1a_unweighted", "c1b", "c2"])
