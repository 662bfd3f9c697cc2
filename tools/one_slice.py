"""Run ONE eager slice of a frozen plan (the unit an ncu capture profiles).

    python tools/one_slice.py c2 [--slices K]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_15512_b200 import _lib, planfile  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--slices", type=int, default=0, help="greedy-slice prefix length")
    a = ap.parse_args()
    flat, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{a.plan}.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    chosen = []
    for _ in range(a.slices):
        chosen.append(h.choose_slice_index(chosen))
    ex = _lib.Exec(h, chosen, 0)
    st = ex.run(0, 1)  # one pass, launched eagerly (no graph)
    print(f"{a.plan}: launches {st['gpu_launches']} device_ms {st['device_ms']:.3f}")


if __name__ == "__main__":
    main()
