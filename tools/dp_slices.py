"""Every per-slice value of a sliced config from the exact counter
(oracle/wmc_dp.c) — test-fixture generation, parallel over slices.

    python tools/dp_slices.py c4 [--procs 8]   -> tests/golden/sliced_dp_c4.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

_TEXT = None
_VARS = None


def _init(text, vars_):
    global _TEXT, _VARS
    _TEXT, _VARS = text, vars_


def _one(args):
    from oracle import wmc_dp

    s, eta = args
    fix = {}
    for v, b in zip(_VARS, eta):
        if fix.get(v, b) != b:
            return s, 0.0
        fix[v] = b
    return s, wmc_dp.count(_TEXT, fix=fix)[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--procs", type=int, default=8)
    a = ap.parse_args()
    from make_sliced_golden import SLICE_RULES, bond_var, chosen_ids, eta_of
    from oracle import wmc_dp
    from paper_2006_15512_b200 import planfile
    from paper_2006_15512_b200.generators import config_dimacs

    flat, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{a.config}.tcplan.npz"))
    ch = chosen_ids(flat, SLICE_RULES[a.config])
    text = config_dimacs(a.config)
    n = wmc_dp.parse(text)[0]
    vars_ = [bond_var(flat.indices[i].id, n) for i in ch]
    assert all(v is not None for v in vars_), "a sliced bond is not a variable-copy bond"
    doms = [int(flat.domain[i]) for i in ch]
    ns = 1
    for d in doms:
        ns *= d
    t0 = time.time()
    with Pool(a.procs, initializer=_init, initargs=(text, vars_)) as pool:
        vals = dict(pool.imap_unordered(_one, [(s, eta_of(s, doms)) for s in range(ns)], chunksize=4))
    out = dict(config=a.config, chosen=[repr(flat.indices[i].id) for i in ch], variables=vars_, num_slices=ns,
               values=[vals[s] for s in range(ns)], seconds=time.time() - t0,
               source="oracle/wmc_dp.c with the sliced variables fixed (slice s: first chosen index = MSB)")
    with open(os.path.join(ROOT, "tests", "golden", f"sliced_dp_{a.config}.json"), "w") as f:
        json.dump(out, f)
    nz = sum(1 for v in out["values"] if v != 0.0)
    print(a.config, "slices", ns, "nonzero", nz, "sum", sum(out["values"]), "seconds", out["seconds"])


if __name__ == "__main__":
    main()
