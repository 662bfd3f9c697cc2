"""Validate bench.reference_sample_model (the extrapolated CPU baseline of the
sliced configs) against full runs of the unmodified reference on the plans
where the reference runs whole (c1a, c2, c1b).

    python tools/validate_ref_model.py [c1a c2 c1b]  -> profiles/ref_model_validation.json
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main(names):
    out = {}
    for name in names:
        flat, _ = bench.load_plan(name)
        rec = {}
        for cap in (25, 27):
            r = bench.reference_sample_model(flat, [], budget_s=20.0, cap_log2=cap)
            rec[f"model_cap{cap}"] = r
        t0 = time.perf_counter()
        sec, count, times = bench.time_reference_full(flat, 1)
        rec["actual_seconds"] = sec
        for cap in (25, 27):
            rec[f"ratio_model_over_actual_cap{cap}"] = rec[f"model_cap{cap}"]["seconds_per_slice"] / sec
        rec["cores"] = bench.host_cores()
        out[name] = rec
        print(name, json.dumps({k: v for k, v in rec.items() if not k.startswith("model")}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ref_model_validation.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1a", "c2", "c1b"])
