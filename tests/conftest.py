import ast
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

collect_ignore = ["reference_suite"]  # run in isolated subprocesses (test_gpu_reference_suite.py)

GOLDEN = os.path.join(ROOT, "tests", "golden")
PLANS = os.path.join(ROOT, "data", "plans")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libtc's kernels")


def has_gpu():
    try:
        from paper_2006_15512_b200 import _lib

        return _lib.lib().tc_device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def load_cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)["cases"]


def case_flat(case):
    """FlatPlan (mirror Index objects) of a golden case."""
    from paper_2006_15512_b200.flatten import FlatPlan
    from paper_2006_15512_b200.tensor import Index

    p = case["plan"]
    ids = [ast.literal_eval(s) for s in p["ids"]]
    return FlatPlan(
        indices=[Index(i, d) for i, d in zip(ids, p["domain"])],
        domain=np.array(p["domain"], np.int32),
        sort_rank=np.array(p["sort_rank"], np.int32),
        leaf_idx_off=np.array(p["leaf_idx_off"], np.int64),
        leaf_idx=np.array(p["leaf_idx"], np.int32),
        leaf_val_off=np.array(p["leaf_val_off"], np.int64),
        leaf_val=np.array([float.fromhex(x) for x in p["leaf_val"]], np.float64),
        left=np.array(p["left"], np.int32),
        right=np.array(p["right"], np.int32),
        root_slot=int(p["root_slot"]),
    )


def hexvals(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


@pytest.fixture(scope="session")
def golden_cases():
    return load_cases()


@pytest.fixture(scope="session")
def golden_counts():
    with open(os.path.join(GOLDEN, "counts.json")) as f:
        return json.load(f)
