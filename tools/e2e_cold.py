"""Per-call wall time of the public sliced_execute on a bench config: three
calls after tc_release_cache (the bench's e2e protocol), then three warm.

    python tools/e2e_cold.py c4
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib, planfile, sliced_execute  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = bench.CONFIGS[name]
flat, _ = bench.load_plan(spec["plan"])
_, chosen = bench.choose(flat, spec["slices"])
n, t = planfile.to_objects(flat)
sl = [flat.indices[i] for i in chosen] if chosen else None
sliced_execute(n, t, slice_indices=sl, devices=[0])
for phase in ("after release_cache", "warm"):
    if phase.startswith("after"):
        _lib.release_cache(0)
    for k in range(3):
        t0 = time.perf_counter()
        sliced_execute(n, t, slice_indices=sl, devices=[0])
        print(f"{name} {phase} call {k}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
