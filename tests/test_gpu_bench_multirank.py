"""The bench's sharded path end to end (self-launch under torchrun, block
partition of the slice ids, gather + lexicographic fold, distributed e2e) with
two ranks sharing the one GPU of the test box (TC_BENCH_SHARE_GPU=1: gloo for
the collectives, since NCCL rejects two ranks on one device).  The folded
count must equal the single-process count bit for bit."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")


def _bench(args, env=None):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, env=dict(os.environ, **(env or {})), cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_two_ranks_fold_to_the_single_rank_bits():
    common = ["--config", "c1b_s3", "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--e2e-steps", "1"]
    one = _bench(common)
    two = _bench(["--gpus", "2", *common], env={"TC_BENCH_SHARE_GPU": "1"})
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "slices/2"
    assert two["count"] == one["count"] and two["e2e_count"] == one["e2e_count"] == one["count"]
    assert two["parity"]["rel_err"] <= 1e-9
