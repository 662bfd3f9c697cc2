"""Per-launch profile of one slice of a frozen plan (eager replay, CUDA events).

    python tools/profile_plan.py c2 [--slices K] [--top 25] [--json out.json]
"""
import argparse
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_15512_b200 import _lib, planfile  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--slices", type=int, default=0, help="greedy-slice prefix length")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    flat, meta = planfile.load(os.path.join(ROOT, "data", "plans", f"{a.plan}.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    chosen = []
    for _ in range(a.slices):
        chosen.append(h.choose_slice_index(chosen))
    ex = _lib.Exec(h, chosen, 0)
    st = ex.run(0, 1)
    st = ex.run(0, 1)
    prof = ex.profile(0)
    prof = ex.profile(0)
    # node shapes
    L = flat.num_leaves
    sets = [frozenset(flat.leaf_idx[flat.leaf_idx_off[k]:flat.leaf_idx_off[k + 1]].tolist()) - set(chosen)
            for k in range(L)]
    shape = {}
    for k in range(flat.num_nodes):
        A, B = sets[flat.left[k]], sets[flat.right[k]]
        sets.append(A ^ B)
        shape[L + k] = (len(A), len(B), len(A ^ B), len(A & B))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for p in prof:
        g = agg[p["kind"]]
        g[0] += 1
        g[1] += p["ms"]
        g[2] += p["bytes"]
        g[3] += p["flops"]
    tot = sum(p["ms"] for p in prof)
    print(f"plan {a.plan} slices={len(chosen)} graph device_ms={st['device_ms']:.3f} eager_sum_ms={tot:.3f}")
    for k, (n, ms, by, fl) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:9s} n={n:6d} ms={ms:9.3f} ({100 * ms / tot:5.1f}%)  GB/s={by / ms / 1e6 if ms else 0:8.1f}"
              f"  GF/s={fl / ms / 1e6 if ms else 0:9.1f}")
    # critical path of the launch DAG with eager per-launch times
    deps = ex.deps()
    fin = [0.0] * len(prof)
    pred = [-1] * len(prof)
    for i, p in enumerate(prof):
        best, arg = 0.0, -1
        for d in deps[i]:
            if fin[d] > best:
                best, arg = fin[d], d
        fin[i] = best + p["ms"]
        pred[i] = arg
    end = max(range(len(prof)), key=lambda i: fin[i])
    path = []
    while end >= 0:
        path.append(end)
        end = pred[end]
    cp = collections.Counter()
    cpn = collections.Counter()
    for i in path:
        cp[prof[i]["kind"]] += prof[i]["ms"]
        cpn[prof[i]["kind"]] += 1
    print(f"critical path (eager times): {max(fin):.3f} ms over {len(path)} launches:",
          {k: (cpn[k], round(v, 3)) for k, v in cp.items()})
    print("top launches:")
    for p in sorted(prof, key=lambda p: -p["ms"])[: a.top]:
        print(f"  {p['kind']:8s} slot={p['slot']:7d} shape(ra,rb,rc,k)={shape.get(p['slot'])} ms={p['ms']:.4f}"
              f" GB/s={p['bytes'] / p['ms'] / 1e6 if p['ms'] else 0:8.1f} GF/s={p['flops'] / p['ms'] / 1e6 if p['ms'] else 0:8.1f}")
    if a.json:
        json.dump(dict(plan=a.plan, stats=st, prof=prof), open(a.json, "w"))


if __name__ == "__main__":
    main()
