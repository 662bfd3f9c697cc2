"""Golden per-slice values of the sliced benchmark configurations
(tests/golden/sliced.json), from two independent sources:

* ``reference``: the UNMODIFIED reference's own slice code path,
  ``_execute_tracked(*_slice_plan(n, t, eta))`` (pkg/src/tensorcount/
  slicing.py:30-41, 91-109, 139-145), on the first lexicographic slices.
  Feasible where one slice's dense working set fits host RAM (C3: 5 GiB,
  ~400 GB of dense traffic per slice, minutes each).
* ``dp``: the exact clause-frontier counter ``oracle/wmc_dp.c`` (restating
  the reference's count oracle brute_force_count, formula.py:183-215), for the
  whole count and for slices whose sliced bonds are variable-copy bonds
  (``(("b", ordinal), k)`` of the copy tensor of variable ordinal+1, or an
  occurrence index ``(var, clause)``: fixing the bond fixes the variable,
  factoring.py:194-206, reduction.py:80-92).  Used where the reference's dense
  per-slice working set exceeds RAM (C4: 96 GiB, C5: 8 TB of dense traffic).

Slice sets: C4 / C5 = the reference greedy's 8 / 12-pick prefix
(choose_slice_index, slicing.py:70-79, via libtc's exact port, which is pinned
to the reference on every fixture); C3 = libtc's work-aware chooser down to
2^28 entries per intermediate (rank 28; the greedy plateaus at rank 34).
Slice s assigns the first chosen index the most significant digit
(itertools.product order, slicing.py:138-139).

    python tests/golden/make_sliced_golden.py c4 c5        # seconds
    python tests/golden/make_sliced_golden.py c3 --slices 4  # ~1 h on 8 cores
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "sliced.json")

SLICE_RULES = {"c4": ("greedy", 8), "c5": ("greedy", 12), "c3": ("work", 28)}


def chosen_ids(flat, rule):
    from paper_2006_15512_b200 import _lib

    h = _lib.PlanHandle(flat)
    kind, k = rule
    if kind == "greedy":
        ch = []
        for _ in range(k):
            ch.append(h.choose_slice_index(ch))
        return ch
    return h.choose_slices_work(2 ** k)


def eta_of(s, doms):
    out = []
    for d in reversed(doms):
        out.append(s % d)
        s //= d
    return out[::-1]


def bond_var(ix_id, num_vars):
    """CNF variable carried by a copy-tensor bond, or None."""
    a, k = ix_id
    if isinstance(a, tuple) and a[0] == "b":
        return a[1] + 1 if a[1] < num_vars else None  # reduce_formula: variables 1..n first
    if isinstance(a, int):
        return a  # occurrence index (var, clause ordinal)
    return None


def dp_golden(name, flat, ch, samples):
    from oracle import wmc_dp
    from paper_2006_15512_b200.generators import config_dimacs

    text = config_dimacs(name)
    n, _, _ = wmc_dp.parse(text)
    t0 = time.time()
    total, peak = wmc_dp.count(text)
    rec = dict(count=total, count_source="dp", dp_peak_states=peak, dp_seconds=time.time() - t0, slices={})
    vars_ = [bond_var(flat.indices[i].id, n) for i in ch]
    if all(v is not None for v in vars_):
        doms = [int(flat.domain[i]) for i in ch]
        for s in samples:
            eta = eta_of(s, doms)
            fix = {}
            ok = True
            for v, b in zip(vars_, eta):
                if fix.get(v, b) != b:
                    ok = False  # two bonds of one variable with different values: structural zero
                fix[v] = b
            val = wmc_dp.count(text, fix=fix)[0] if ok else 0.0
            rec["slices"][str(s)] = dict(value=val, source="dp", fixed=fix)
    return rec


def ref_golden(flat, ch, samples):
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    sys.path.insert(0, ROOT)
    from bench import _ref_indices, reference_objects
    from tensorcount import slicing as ref_slicing
    from tensorcount.tensor import Assignment

    n, t = reference_objects(flat)
    idx = _ref_indices(n, flat, ch)
    doms = [int(flat.domain[i]) for i in ch]
    out = {}
    for s in samples:
        t0 = time.time()
        m, plan = ref_slicing._slice_plan(n, t, Assignment(zip(idx, eta_of(s, doms))))
        res, peak = ref_slicing._execute_tracked(m, plan)
        out[str(s)] = dict(value=float(res.values.reshape(-1)[0]), source="reference", peak_observed=int(peak),
                           seconds=time.time() - t0)
        print(f"slice {s}: {out[str(s)]}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--slices", type=int, default=4)
    a = ap.parse_args()
    from paper_2006_15512_b200 import planfile

    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in a.configs:
        flat, meta = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))
        rule = SLICE_RULES[name]
        ch = chosen_ids(flat, rule)
        ns = 1
        for i in ch:
            ns *= int(flat.domain[i])
        samples = list(range(min(a.slices, ns)))
        rec = data.get(name, {})
        rec.update(rule=list(rule), chosen=[repr(flat.indices[i].id) for i in ch], num_slices=ns)
        if name in ("c4", "c5"):
            samples += [ns - 1, ns // 2 + 1, 37 % ns]
            rec.update(dp_golden(name, flat, ch, samples))
        else:
            rec.setdefault("slices", {}).update(ref_golden(flat, ch, samples))
        data[name] = rec
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        print(name, json.dumps(rec)[:600], flush=True)


if __name__ == "__main__":
    main()
