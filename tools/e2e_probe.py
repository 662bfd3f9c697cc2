"""Python-side timing of every stage of one public sliced_execute call
(slicing._run, _lib.PlanHandle.sliced_execute) for a bench config.

    python tools/e2e_probe.py c4
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2006_15512_b200 import _lib, planfile, sliced_execute, slicing  # noqa: E402
from paper_2006_15512_b200.flatten import _native  # noqa: E402


def main(name):
    spec = bench.CONFIGS[name]
    flat0, _ = bench.load_plan(spec["plan"])
    _, chosen = bench.choose(flat0, spec["slices"])
    n, t = planfile.to_objects(flat0)
    sl = [flat0.indices[i] for i in chosen] if chosen else None
    sliced_execute(n, t, slice_indices=sl)
    for _ in range(3):
        T = [time.perf_counter()]
        flat, h = slicing._plan(n, t, with_sort_rank=False)
        T.append(time.perf_counter())
        ids = _native().positions(flat.indices, sl) if sl else None  # as slicing._run
        T.append(time.perf_counter())
        root = h.result_indices(())
        T.append(time.perf_counter())
        vals, idx, ch, st = h.sliced_execute(None, ids, [0])
        T.append(time.perf_counter())
        res = type(n.tensors[0])(tuple(flat.indices[i] for i in idx), np.asarray(vals).reshape(
            tuple(int(flat.domain[i]) for i in idx)))
        T.append(time.perf_counter())
        d = np.diff(T) * 1e3
        print(f"{name}: plan(flatten+create) {d[0]:.1f} ids {d[1]:.1f} result_indices {d[2]:.1f} "
              f"tc_sliced_execute {d[3]:.1f} (device {st['device_ms']:.1f} program {st['program_ms']:.1f} "
              f"setup {st['setup_ms']:.1f} graph {st['graph_ms']:.1f}) tensor {d[4]:.1f} total {sum(d):.1f}", flush=True)
        del res, root


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c4"]:
        main(nm)
