"""compute-sanitizer target: one small sliced pass (hoisting, 2 lanes, graph
replay) and one eager pass of plans that exercise k_tiny (elided barriers),
k_stream, k_stream_pair, k_gemm (split-K), k_select, k_rootcopy, k_fold.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TC_LANES", "2")

import numpy as np  # noqa: E402

from paper_2006_15512_b200 import Index, Tensor, _lib, contract_pair, planfile  # noqa: E402


def main():
    for name, picks in (("c1a", 2), ("c1a", 0), ("c2", 0)):
        flat, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))
        h = _lib.PlanHandle(flat)
        ch = []
        for _ in range(picks):
            ch.append(h.choose_slice_index(ch))
        ex = _lib.Exec(h, ch, 0)
        ns = ex.num_slices()
        ex.run(0, ns)               # eager
        ex.run(0, ns, repeats=3)    # graphs (+ lanes when sliced)
        f, _ = ex.fetch()
        print(name, picks, f[0])
    rng = np.random.default_rng(0)
    idx = [Index(k, 2) for k in range(20)]
    a = Tensor(tuple(idx[:14]), rng.uniform(-1, 1, [2] * 14))
    b = Tensor(tuple(idx[6:20]), rng.uniform(-1, 1, [2] * 14))
    c = contract_pair(a, b)  # k_gemm
    print("gemm", float(np.abs(c.values).sum()))


if __name__ == "__main__":
    main()
