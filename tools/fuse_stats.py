"""Chain-link fusion statistics of a config's program (TC_FUSE_DEBUG lines on
stderr; run on a GPU box): candidate links, fused pairs, missing kernel shapes.

    TC_FUSE_DEBUG=1 python tools/fuse_stats.py c4 2> fuse.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = bench.CONFIGS[name]
flat, _ = bench.load_plan(spec["plan"])
h, ch = bench.choose(flat, spec["slices"])
ex = _lib.Exec(h, ch, 0)
st = ex.run(0, 1)
print(name, "launches_prologue", st["launches_prologue"], "launches_per_slice", st["launches_per_slice"])
