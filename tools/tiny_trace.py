"""Per-node clock trace of the first tiny group (block 0 of each tiny launch)
of one eager slice (TC_TINY_TRACE=1, stderr).

    TC_TINY_TRACE=1 python tools/tiny_trace.py c2 2> trace.txt
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
ex.profile(0)
