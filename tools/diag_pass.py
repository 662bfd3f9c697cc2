"""Device time of a whole pass over a config's slices (graph mode), for A/B runs of
diagnostics builds (TC_LIBTC=...), e.g. one whose k_tiny returns at entry
(-DTC_DIAG_TINY_SKIP): an upper bound on what the tiny stage costs in the pass.

    TC_LIBTC=paper_2006_15512_b200/lib/diag/libtc_tinyskip.so python tools/diag_pass.py c4
"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402

for name in sys.argv[1:]:
    spec = bench.CONFIGS[name]
    flat, _ = bench.load_plan(spec["plan"])
    rule = spec["slices"]
    if os.environ.get("DIAG_PICKS") and rule and rule[0] == "greedy":  # k-pick greedy prefix instead
        rule = ("greedy", int(os.environ["DIAG_PICKS"]))
    h, ch = bench.choose(flat, rule)
    ex = _lib.Exec(h, ch, 0)
    ns = min(ex.num_slices(), int(os.environ.get("DIAG_SLICES", "512")))
    ex.run(0, ns)
    ex.run(0, ns, repeats=2)
    st = ex.run(0, ns, repeats=5)
    B = max(1, st.get("slices_per_block", 1))
    ex_b = (st["phys_bytes_hoisted"] + -(-ns // B) * st["phys_bytes_block"]
            + ns * (st["phys_bytes"] - st["phys_bytes_hoisted"] - st["phys_bytes_block"])) / 1e9
    print(name, os.path.basename(_lib.LIB_PATH), "picks", len(ch), "slices", ns, "ms/pass %.3f" % (st["device_ms"] / 5),
          "executed GB/pass %.1f" % ex_b, "launches/pass", st["gpu_launches"] // 5, flush=True)
