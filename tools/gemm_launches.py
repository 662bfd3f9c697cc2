"""GEMM launches of a config's per-slice program with their graph-mode time,
flops and bytes, in emission order (pair with TC_GEMM_STATS=1 on stderr).

    TC_GEMM_STATS=1 python tools/gemm_launches.py c3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec = bench.CONFIGS[name]
flat, _ = bench.load_plan(spec["plan"])
h, ch = bench.choose(flat, spec["slices"])
ex = _lib.Exec(h, ch, 0)
ex.run(0, 2)
prof, pm = ex.profile_graph(0, 1)
for p in prof:
    if p["kind"] in ("gemm", "gemm_reduce"):
        print(f"{p['kind']:12s} inv={int(p['inv'])} ms={p['ms']:.4f} GF={p['flops'] / 1e9:.3f} MB={p['bytes'] / 1e6:.1f} "
              f"TF/s={p['flops'] / p['ms'] / 1e9 if p['ms'] else 0:.2f} GB/s={p['bytes'] / p['ms'] / 1e6 if p['ms'] else 0:.0f}",
              flush=True)
