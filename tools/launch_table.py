"""Per-launch graph-mode table of a config's program (bench's slice rule):
kind, hoisted?, executed MB, ms, GB/s -> gpurun_out/launches_<config>.json and
a size-class summary on stdout.

    python tools/launch_table.py c4 [--slices 4]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--slices", type=int, default=4)
    a = ap.parse_args()
    spec = bench.CONFIGS[a.config]
    flat, _ = bench.load_plan(spec["plan"])
    h, ch = bench.choose(flat, spec["slices"])
    ex = _lib.Exec(h, ch, 0)
    ns = max(1, min(a.slices, ex.num_slices()))
    ex.run(0, ns)
    prof, pass_ms = ex.profile_graph(0, ns)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(dict(config=a.config, slices=ns, pass_ms=pass_ms, launches=prof),
              open(os.path.join(ROOT, "gpurun_out", f"launches_{a.config}.json"), "w"))
    import math
    buckets = {}
    for p in prof:
        mult = 1 if p["inv"] else ns
        key = (p["kind"], p["inv"], int(math.log2(max(p["bytes"], 1))) if p["bytes"] else -1)
        b = buckets.setdefault(key, [0, 0.0, 0.0])
        b[0] += mult
        b[1] += p["ms"]
        b[2] += p["bytes"] * mult
    print(f"pass over {ns} slices: {pass_ms:.2f} ms (graph events, sync per slice)")
    tot = sum(b[1] for b in buckets.values())
    for k in sorted(buckets, key=lambda k: -buckets[k][1]):
        n, ms, by = buckets[k]
        print(f"{k[0]:>10} {'inv' if k[1] else 'var'} 2^{k[2]:>2}B  launches {n:6d}  ms {ms:9.3f} ({ms / tot:5.1%})"
              f"  GB/s {by / ms / 1e6 if ms else 0:8.1f}  us/launch {ms / n * 1e3:8.1f}")


if __name__ == "__main__":
    main()
