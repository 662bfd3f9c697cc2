"""The whole counting pipeline of one benchmark formula, reference vs native:
``count_formula`` (reference driver.py:217-251: reduce_formula -> plan_contraction
(min-fill tree decomposition -> tree_to_branch -> factor_branch_audit, alpha=0)
-> sliced_execute).

    python tools/pipeline_bench.py c2 --impl native      # planning + FactorTree native, execution on the GPU
    python tools/pipeline_bench.py c2 --impl reference   # the unmodified reference (CPU)
    python tools/pipeline_bench.py c4 --impl native --no-execute

Prints one JSON line: per-stage seconds (reduce, plan, execute), the count,
and a hash of serialize_plan(M, T) (identical plan on both sides).
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "tensorcount")):
        sys.path.insert(1, p)
        break


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--no-execute", action="store_true")
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    import tensorcount

    if a.impl == "native":
        from paper_2006_15512_b200 import reference_patch

        reference_patch.install(tensorcount, execution=not a.no_execute)
    from tensorcount.driver import plan_contraction, sliced_execute
    from tensorcount.formula import parse_dimacs
    from tensorcount.network import serialize_plan
    from tensorcount.reduction import reduce_formula

    from paper_2006_15512_b200.generators import config_dimacs

    text = config_dimacs(a.config)
    rows = []
    for _ in range(a.repeat):
        t0 = time.perf_counter()
        f, w = parse_dimacs(text)
        n = reduce_formula(f, w)
        t1 = time.perf_counter()
        best, nplans, _ = plan_contraction(n, planner_spec="minfill", alpha=0.0, seed=0)
        t2 = time.perf_counter()
        count = None
        if not a.no_execute:
            ex = sliced_execute(best.network, best.tree, mem_budget=None)
            count = float(ex.result.values)
        t3 = time.perf_counter()
        rows.append(dict(reduce_s=t1 - t0, plan_s=t2 - t1, execute_s=(t3 - t2) if not a.no_execute else None))
    plan_hash = hashlib.sha256(serialize_plan(best.network, best.tree).encode()).hexdigest()[:16]
    best_row = min(rows, key=lambda r: r["plan_s"] + (r["execute_s"] or 0.0))
    print(json.dumps(dict(config=a.config, impl=a.impl, **best_row, count=count, plan_sha=plan_hash,
                          leaves=len(best.network.tensors), width=best.record.width, repeats=a.repeat)))


if __name__ == "__main__":
    main()
