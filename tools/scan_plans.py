"""Plan candidate benchmark instances with the UNMODIFIED reference planner and
report the statistics that pin a config: max-rank, MACs,
dense mem_cost, and for a greedy slice prefix of length k (the reference's
choose_slice_index, exact C++ port) the per-slice max-rank / mem_cost and the
executed (tie-aware) work per slice.

    python tools/scan_plans.py banded:400:4.0:36:11 banded:400:4.0:44:2 --picks 8 --out /tmp/plans
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from make_plans import plan_text  # noqa: E402

from paper_2006_15512_b200 import _lib, generators, planfile  # noqa: E402
from paper_2006_15512_b200.flatten import flatten  # noqa: E402


def sliced_max_rank(flat, chosen):
    ch = set(chosen)
    L = flat.num_leaves
    sets = [frozenset(flat.leaf_idx[flat.leaf_idx_off[k]:flat.leaf_idx_off[k + 1]].tolist()) - ch for k in range(L)]
    best = max((len(s) for s in sets), default=0)
    for l, r in zip(flat.left.tolist(), flat.right.tolist()):
        s = sets[l] ^ sets[r]
        sets.append(s)
        best = max(best, len(s))
    return best


def gen_text(spec):
    p = spec.split(":")
    if p[0] == "banded":
        return generators.banded_3cnf(int(p[1]), float(p[2]), int(p[3]), int(p[4]))
    if p[0] == "uniform":
        return generators.uniform_3cnf(int(p[1]), float(p[2]), int(p[3]))
    if p[0] == "grid":
        return generators.grid_ising(int(p[1]), int(p[2]))
    raise ValueError(spec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--picks", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    for spec in a.specs:
        t0 = time.time()
        f, res = plan_text(gen_text(spec))
        flat = flatten(res.network, res.tree)
        tp = time.time() - t0
        h = _lib.PlanHandle(flat)
        info = h.info()
        row = dict(spec=spec, plan_s=round(tp, 1), leaves=flat.num_leaves, max_rank=info.max_rank,
                   macs=info.contraction_ops.value(), mem_gib=info.mem_cost.value() / 2 ** 30)
        st0 = h.compile_stats([])
        row["phys_gb"] = st0["phys_bytes"] / 1e9
        chosen = []
        picks = []
        for k in range(a.picks):
            chosen.append(h.choose_slice_index(chosen))
            st = h.compile_stats(chosen)
            picks.append(dict(k=k + 1, rank=sliced_max_rank(flat, chosen), mem_gib=round(h.mem_cost(chosen) / 2 ** 30, 3),
                              phys_gb_slice=round(st["phys_bytes"] / 1e9, 3),
                              phys_gb_total=round(st["phys_bytes"] / 1e9 * 2 ** (k + 1), 1),
                              dense_gb_slice=round(st["alg_bytes"] / 1e9, 2)))
        row["picks"] = picks
        print(json.dumps(row), flush=True)
        if a.out:
            planfile.save(os.path.join(a.out, spec.replace(":", "_") + ".tcplan.npz"), flat,
                          dict(spec=spec, max_rank=info.max_rank, planning_seconds=tp))


if __name__ == "__main__":
    main()
