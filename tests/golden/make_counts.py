"""Run the UNMODIFIED reference ``sliced_execute`` (slicing.py:112-146) on the
frozen benchmark plans and record the counts as golden values.

    python tests/golden/make_counts.py c1a c1a_unweighted c2 c1b

Needs the reference importable (oracle/_ref or /root/reference/pkg/src); it
only runs in the build container.  Output: tests/golden/counts.json.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(p):
        sys.path.insert(1, p)
        break

from tensorcount.network import ContractionTree, TensorNetwork  # noqa: E402
from tensorcount.slicing import sliced_execute  # noqa: E402
from tensorcount.tensor import Index, Tensor  # noqa: E402

from paper_2006_15512_b200 import planfile  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "counts.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        flat, meta = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"), index_cls=Index)
        n, t = planfile.to_objects(flat, Tensor, TensorNetwork, ContractionTree)
        t0 = time.time()
        res = sliced_execute(n, t)
        dt = time.time() - t0
        data[name] = dict(
            count=float(res.result.values),
            count_hex=float(res.result.values).hex(),
            mem_estimate=str(res.mem_estimate),
            peak_observed=str(res.peak_observed),
            ref_seconds=dt,
            ref_host_cores=os.cpu_count(),
        )
        print(name, data[name], flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)




def greedy(name, picks):
    """Reference greedy prefix (slicing.py:70-79) on a frozen plan."""
    from tensorcount.slicing import choose_slice_index
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    flat, meta = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"), index_cls=Index)
    n, t = planfile.to_objects(flat, Tensor, TensorNetwork, ContractionTree)
    pos = {ix: k for k, ix in enumerate(flat.indices)}
    chosen = []
    t0 = time.time()
    for _ in range(picks):
        chosen.append(choose_slice_index(n, t, already=frozenset(chosen)))
    data[f"{name}_greedy{picks}"] = dict(ids=[pos[i] for i in chosen], id_reprs=[repr(i.id) for i in chosen],
                                         ref_seconds=time.time() - t0)
    print(data[f"{name}_greedy{picks}"], flush=True)
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["greedy"]:
        greedy(sys.argv[2], int(sys.argv[3]))
    else:
        main(sys.argv[1:])
