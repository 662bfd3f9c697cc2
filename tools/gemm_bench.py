"""Micro-benchmark of libtc's FP64 DMMA GEMM class on one pairwise
contraction vs cuBLAS DGEMM (torch.matmul float64) of the same M, N, K.

    python tools/gemm_bench.py 11:13:13 5:3:17 16:9:8 ...   (m:n:k bits)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_15512_b200 import Index, Tensor, TensorNetwork, join, leaf  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402
from paper_2006_15512_b200.flatten import flatten  # noqa: E402


def one(m, n, k, reps=5):
    import torch

    M = [Index(("m", i), 2) for i in range(m)]
    N = [Index(("n", i), 2) for i in range(n)]
    K = [Index(("k", i), 2) for i in range(k)]
    rng = np.random.default_rng(0)
    a = Tensor(tuple(M + K), rng.uniform(-1, 1, [2] * (m + k)))
    # both operands K-lowest (row-major M x K and N x K), the layouts the
    # compiler's layout pass requests for GEMM operands
    b = Tensor(tuple(N + K), rng.uniform(-1, 1, [2] * (n + k)))
    nw = TensorNetwork((a, b))
    fl = flatten(nw, join(leaf(a), leaf(b)))
    h = _lib.PlanHandle(fl)
    ex = _lib.Exec(h, [], 0)
    ex.run(0, 1, repeats=2)
    st = ex.run(0, 1, repeats=reps)
    ms = st["device_ms"] / reps
    fl_ = 2.0 * 2 ** (m + n + k)
    # correctness spot check on the full result
    folded, _ = ex.fetch()
    A = torch.tensor(a.values.reshape(2 ** m, 2 ** k), device="cuda")
    B = torch.tensor(b.values.reshape(2 ** n, 2 ** k), device="cuda").t().contiguous()
    C = (A @ B).cpu().numpy().reshape(-1)
    err = float(np.max(np.abs(folded - C)) / max(1e-300, np.max(np.abs(C))))
    for _ in range(2):
        A @ B
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        A @ B
    e1.record()
    torch.cuda.synchronize()
    cms = e0.elapsed_time(e1) / reps
    print(f"m={m:2d} n={n:2d} k={k:2d}  ours {ms:8.3f} ms {fl_ / ms / 1e9:7.2f} TF/s   cuBLAS {cms:8.3f} ms "
          f"{fl_ / cms / 1e9:7.2f} TF/s   ratio {cms / ms:5.2f}  relerr {err:.1e}", flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["11:13:13", "16:9:8", "5:3:17", "13:13:13", "14:14:12"]:
        m, n, k = map(int, spec.split(":"))
        one(m, n, k)
