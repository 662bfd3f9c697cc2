"""Where the end-to-end time of one public-API call goes (bench configs,
their slice rules).

    python tools/e2e_breakdown.py c4 c2
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2006_15512_b200 import _lib, planfile, sliced_execute  # noqa: E402
from paper_2006_15512_b200.flatten import flatten  # noqa: E402


def main(name):
    spec = bench.CONFIGS[name]
    flat0, _ = bench.load_plan(spec["plan"])
    _, chosen = bench.choose(flat0, spec["slices"])
    n, t = planfile.to_objects(flat0)
    sl = [flat0.indices[i] for i in chosen] if chosen else None
    rng = None
    if spec.get("sample"):
        rng = (0, min(spec["sample"], bench.num_slices(flat0, chosen)))
    sliced_execute(n, t, slice_indices=sl, slice_range=rng)  # warm: CUDA context, module load
    for _ in range(3):
        t0 = time.perf_counter()
        fl = flatten(n, t, with_sort_rank=False)
        t1 = time.perf_counter()
        _lib.PlanHandle(fl)
        t2 = time.perf_counter()
        res = sliced_execute(n, t, slice_indices=sl, slice_range=rng)
        t3 = time.perf_counter()
        st = res.stats
        print(f"{name}: e2e {1e3 * (t3 - t2):.1f} ms | flatten {1e3 * (t1 - t0):.1f} plan_create {1e3 * (t2 - t1):.1f} | "
              f"program {st['program_ms']:.1f} setup {st['setup_ms']:.1f} graph {st['graph_ms']:.1f} "
              f"device {st['device_ms']:.1f} | launches {st['gpu_launches']}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c4", "c2"]:
        main(nm)
