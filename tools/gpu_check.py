"""Quick GPU sanity run: small random contractions vs numpy (checker only),
and the frozen benchmark plans vs the reference's golden counts."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_15512_b200 import Index, Tensor, TensorNetwork, contract_pair, planfile, sliced_execute  # noqa
from paper_2006_15512_b200 import _lib  # noqa


def check_pairs():
    rng = np.random.default_rng(0)
    bad = 0
    for trial in range(200):
        dom = 2 if trial % 3 else 3
        pool = [Index(f"i{k}", dom if rng.random() < 0.8 else 2) for k in range(14 if dom == 2 else 8)]
        ra = int(rng.integers(0, 7 if dom == 2 else 5))
        rb = int(rng.integers(0, 7 if dom == 2 else 5))
        ia = list(rng.choice(len(pool), ra, replace=False))
        ib = list(rng.choice(len(pool), rb, replace=False))
        A = Tensor(tuple(pool[k] for k in ia), rng.uniform(-1, 1, size=[pool[k].domain_size for k in ia]))
        B = Tensor(tuple(pool[k] for k in ib), rng.uniform(-1, 1, size=[pool[k].domain_size for k in ib]))
        out = contract_pair(A, B)
        sh = [i for i in A.indices if i in B.index_set()]
        want = np.tensordot(A.values, B.values, axes=([A.indices.index(i) for i in sh], [B.indices.index(i) for i in sh]))
        kept = [i for i in A.indices if i not in B.index_set()] + [i for i in B.indices if i not in A.index_set()]
        assert list(out.indices) == kept, (out.indices, kept)
        if not np.allclose(out.values, want, rtol=1e-12, atol=1e-12):
            bad += 1
            print("MISMATCH", trial, ia, ib)
    print("pairs: bad", bad, flush=True)


def check_big_pair():
    # big x big GEMM-class and big x piece stream-class single contractions
    rng = np.random.default_rng(1)
    idx = [Index(f"x{k}", 2) for k in range(40)]
    cases = [(list(range(0, 16)), list(range(8, 24))),      # gemm m=8,k=8,n=8
             (list(range(0, 20)), [3, 21, 22]),                 # stream s=1 f=2
             (list(range(0, 20)), [5, 9, 30]),                  # stream s=2 f=1
             (list(range(0, 14)), list(range(4, 18))[::-1]),    # gemm, permuted
             ]
    for ia, ib in cases:
        A = Tensor(tuple(idx[k] for k in ia), rng.uniform(-1, 1, size=[2] * len(ia)))
        B = Tensor(tuple(idx[k] for k in ib), rng.uniform(-1, 1, size=[2] * len(ib)))
        from paper_2006_15512_b200.network import join, leaf
        n = TensorNetwork((A, B))
        t = join(leaf(A), leaf(B))
        res = sliced_execute(n, t)
        out = res.result
        sh = [i for i in A.indices if i in B.index_set()]
        want = np.tensordot(A.values, B.values, axes=([A.indices.index(i) for i in sh], [B.indices.index(i) for i in sh]))
        err = np.max(np.abs(out.values - want)) / max(1e-300, np.max(np.abs(want)))
        print("big pair", len(ia), len(ib), "stats", {k: res.stats[k] for k in ("n_stream_nodes", "n_gemm_nodes", "n_generic_nodes", "n_tiny_nodes")}, "relerr", err, flush=True)


def check_plans(names):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "counts.json")))
    for name in names:
        flat, meta = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))
        n, t = planfile.to_objects(flat)
        for rep in range(2):
            t0 = time.time()
            res = sliced_execute(n, t)
            dt = time.time() - t0
            c = float(res.result.values)
            g = gold[name]["count"] if name in gold else float("nan")
            print(name, "count", c, "gold", g, "rel", abs(c - g) / abs(g) if g else None, "e2e_s", round(dt, 4),
                  {k: res.stats[k] for k in ("device_ms", "compile_ms", "gpu_launches", "n_tiny_nodes", "n_stream_nodes",
                                              "n_gemm_nodes", "n_generic_nodes", "device_peak_bytes")}, flush=True)


if __name__ == "__main__":
    print("devices", _lib.lib().tc_device_count())
    check_pairs()
    check_big_pair()
    check_plans(sys.argv[1:] or ["c1a", "c1a_unweighted", "c2", "c1b"])
