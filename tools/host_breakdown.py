"""Host-side costs of one public-API call (no GPU needed for the first three):
native flatten (leaves vs tree), plan_create, host program compile.

    python tools/host_breakdown.py c2
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_15512_b200 import _lib, planfile  # noqa: E402
from paper_2006_15512_b200.flatten import _native, flatten  # noqa: E402
from paper_2006_15512_b200.network import ContractionTree  # noqa: E402


def best(f, k=7):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


def main(name):
    flat0, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))
    n, t = planfile.to_objects(flat0)
    nat = _native()
    lt = ContractionTree(tensor=n.tensors[0])
    fl = flatten(n, t, with_sort_rank=False)
    print(f"{name}: flatten {best(lambda: flatten(n, t, with_sort_rank=False)):.2f} ms "
          f"(leaves {best(lambda: nat.flatten(n.tensors, lt)):.2f}, tree {best(lambda: nat.flatten((n.tensors[0],), t)):.2f})"
          f" | plan_create {best(lambda: _lib.PlanHandle(fl)):.2f} ms"
          f" | compile {best(lambda: _lib.PlanHandle(fl).compile_stats([])):.2f} ms (incl. plan_create)")


if __name__ == "__main__":
    for a in sys.argv[1:] or ["c2"]:
        main(a)
