"""Run ONE eager pass (prologue + a few slices) of a config's plan (the unit an
ncu capture profiles).  Bench configs use their own slice rule.

    python tools/one_slice.py c4 [--run-slices K]
    python tools/one_slice.py c2 --slices 3        (a plan + greedy prefix length)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2006_15512_b200 import _lib, planfile  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--slices", type=int, default=None, help="greedy-slice prefix length (default: the config's rule)")
    ap.add_argument("--run-slices", type=int, default=1, help="slices in the pass (<= 2: eager launches)")
    a = ap.parse_args()
    if a.slices is None and a.plan in bench.CONFIGS:
        spec = bench.CONFIGS[a.plan]
        flat, _ = bench.load_plan(spec["plan"])
        h, chosen = bench.choose(flat, spec["slices"])
    else:
        flat, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{a.plan}.tcplan.npz"))
        h = _lib.PlanHandle(flat)
        chosen = []
        for _ in range(a.slices or 0):
            chosen.append(h.choose_slice_index(chosen))
    ex = _lib.Exec(h, chosen, 0)
    st = ex.run(0, a.run_slices)  # one pass (prologue + slices), launched eagerly (no graph)
    print(f"{a.plan}: launches {st['gpu_launches']} device_ms {st['device_ms']:.3f}")


if __name__ == "__main__":
    main()
