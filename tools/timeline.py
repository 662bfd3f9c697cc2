"""Graph-mode timeline of one slice of a config: every launch's start (us from
the graph launch) and duration, sorted by start -> the critical path.

    python tools/timeline.py c2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec = bench.CONFIGS[name]
flat, _ = bench.load_plan(spec["plan"])
h, ch = bench.choose(flat, spec["slices"])
ex = _lib.Exec(h, ch, 0)
ex.run(0, 1)
ex.run(0, 1, repeats=3)
prof, pm = ex.profile_graph(0, 1)
rows = sorted((p["start_us"], p["ms"] * 1e3, p["kind"], p["bytes"] / 1e6, p["inv"]) for p in prof)
print(f"{name}: {len(rows)} launches, pass {pm * 1e3:.1f} us (with event nodes)")
for st, du, k, mb, inv in rows:
    print(f"{st:8d} {du:8.1f} {st + du:9.1f}  {k:8s} {'inv' if inv else '   '} {mb:9.2f} MB")
