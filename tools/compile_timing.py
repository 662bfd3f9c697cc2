"""Host compile time of a config's program (compile_stats: no device work),
best of 5, with the per-phase breakdown of the last run on stderr.

    TC_COMPILE_TIMING=1 python tools/compile_timing.py c4 c2
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import planfile, slicing  # noqa: E402

for name in sys.argv[1:] or ["c4", "c2"]:
    spec = bench.CONFIGS[name]
    flat, _ = bench.load_plan(spec["plan"])
    h, ch = bench.choose(flat, spec["slices"])
    n, t = planfile.to_objects(flat)
    best = {}
    for _ in range(5):
        t0 = time.perf_counter()
        f2, h2 = slicing._plan(n, t, with_sort_rank=False)
        t1 = time.perf_counter()
        h.compile_stats(ch)
        t2 = time.perf_counter()
        for k, v in (("flatten+plan", t1 - t0), ("compile", t2 - t1)):
            best[k] = min(best.get(k, 1e9), v * 1e3)
    print(name, {k: round(v, 2) for k, v in best.items()}, flush=True)
