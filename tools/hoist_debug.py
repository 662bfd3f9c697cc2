import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os
sys.path.insert(0, %r)
import numpy as np
from paper_2006_15512_b200 import _lib, planfile
name, picks = sys.argv[1], int(sys.argv[2])
flat, _ = planfile.load(os.path.join(%r, "data", "plans", name + ".tcplan.npz"))
h = _lib.PlanHandle(flat)
ch = []
for _ in range(picks): ch.append(h.choose_slice_index(ch))
ns = 2 ** picks
ex = _lib.Exec(h, ch, 0)
ex.run(0, ns)
f, per = ex.fetch(ns)
st = h.compile_stats(ch)
print(os.environ.get("TC_HOIST"), os.environ.get("TC_HOIST_DBG"), os.environ.get("TC_FUSE"), " ".join(x.hex()[:12] for x in per[:4]), f[0], st["launches_prologue"], st["pinned_bytes"])
''' % (ROOT, ROOT)
for name, picks in [("c2", 4), ("c2", 1), ("c2", 2), ("c1b", 3)]:
    for env in [{"TC_HOIST": "0"}, {}, {"TC_HOIST_DBG": "1"}, {"TC_HOIST_DBG": "2"}, {"TC_HOIST_DBG": "4"}, {"TC_HOIST_DBG": "3"}, {"TC_FUSE": "0"}, {"TC_ARENA_REUSE": "0"}]:
        r = subprocess.run([sys.executable, "-c", code, name, str(picks)], env=dict(os.environ, **env), capture_output=True, text=True)
        print(name, picks, env, r.stdout.strip(), r.stderr[-300:], flush=True)
