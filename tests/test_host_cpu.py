"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/tc.h declares; libtc's exact memory model / greedy chooser / plan
validation agree with the golden fixtures and the oracle; the plan
interchange format and generators are stable.  No kernel is launched."""

import ctypes
import json
import os
import random
import re

import numpy as np
import pytest

from conftest import GOLDEN, PLANS, ROOT, case_flat, load_cases
from oracle import oracle
from paper_2006_15512_b200 import _lib, planfile
from paper_2006_15512_b200.errors import BudgetInfeasible, IndexOveruse, NoCandidates, PlanMismatch
from paper_2006_15512_b200.flatten import flatten

CASES = load_cases()


def test_library_exports_every_header_symbol():
    import glob
    hdr = "".join(open(h).read() for h in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    declared = set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    so = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(so, name), f"libtc.so does not export {name}"
    # and the Python binding covers all of them
    assert declared == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("case", [c for c in CASES if c["family"] == "random_network"],
                         ids=[c["name"] for c in CASES if c["family"] == "random_network"])
def test_mem_cost_and_choose_match_reference(case):
    flat = case_flat(case)
    h = _lib.PlanHandle(flat)
    for k, v in case["expected"]["mem_cost"].items():
        assert h.mem_cost([int(k)] if k else []) == int(v)
    if "choose" in case["expected"]:
        assert h.choose_slice_index([]) == case["expected"]["choose"]


@pytest.mark.parametrize("case", [c for c in CASES if "budgeted" in c["expected"]],
                         ids=[c["name"] for c in CASES if "budgeted" in c["expected"]])
def test_greedy_slice_set_matches_reference(case):
    flat = case_flat(case)
    h = _lib.PlanHandle(flat)
    exp = case["expected"]["budgeted"]
    chosen = np.zeros(max(1, len(flat.domain)), np.int32)
    n = ctypes.c_int32()
    need = _lib.U128()
    st = _lib.lib().tc_choose_slices(h.h, exp["budget"], chosen.ctypes.data_as(_lib.I32P), len(chosen),
                                     ctypes.byref(n), ctypes.byref(need))
    if "error" in exp:
        assert st == 3
        msg = _lib.lib().tc_last_error().decode()
        assert msg == exp["message"]  # reference wording, slicing.py:124-128
        return
    assert st == 0
    assert chosen[: n.value].tolist() == exp["chosen"]
    assert h.mem_cost(exp["chosen"]) == int(exp["mem_estimate"])


def test_infeasible_message_and_status():
    c = next(c for c in CASES if c["family"] == "random_network")
    flat = case_flat(c)
    h = _lib.PlanHandle(flat)
    inf = c["expected"]["infeasible"]
    chosen = np.zeros(len(flat.domain) + 1, np.int32)
    n = ctypes.c_int32()
    st = _lib.lib().tc_choose_slices(h.h, 1, chosen.ctypes.data_as(_lib.I32P), len(chosen), ctypes.byref(n), None)
    assert st == 3 and _lib.lib().tc_last_error().decode() == inf["message"]
    with pytest.raises(BudgetInfeasible):
        _lib.check(st)


def test_choose_no_candidates():
    from paper_2006_15512_b200 import Index, Tensor, TensorNetwork, left_deep_tree
    i = Index("i", 2)
    n = TensorNetwork((Tensor((i,), np.ones(2)),))
    h = _lib.PlanHandle(flatten(n, left_deep_tree(n.tensors)))
    with pytest.raises(NoCandidates):
        h.choose_slice_index([])


def test_plan_validation_errors():
    from paper_2006_15512_b200 import ContractionTree, Index, Tensor, TensorNetwork, join, leaf
    from paper_2006_15512_b200 import slicing
    i, j = Index("i", 2), Index("j", 2)
    a, b = Tensor((i, j), np.ones((2, 2))), Tensor((j,), np.ones(2))
    n = TensorNetwork((a, b))
    stranger = Tensor((i,), np.ones(2))
    with pytest.raises(PlanMismatch):
        slicing.mem_cost(n, join(leaf(a), leaf(stranger)))
    # an index used three times is rejected by the library as well
    flat = flatten(n, join(leaf(a), leaf(b)))
    flat.leaf_idx = np.array([0, 0, 1], np.int32)  # i twice in one leaf
    with pytest.raises(ValueError):
        _lib.PlanHandle(flat)
    c = Tensor((j,), np.ones(2))
    n3 = TensorNetwork((a, b))
    flat3 = flatten(n3, join(join(leaf(a), leaf(b)), leaf(b)))
    assert flat3.root_slot >= 0
    # j in three leaves -> IndexOveruse (network.py:42-43)
    flat3 = flatten(TensorNetwork((a, b, Tensor((i,), np.ones(2)))),
                    join(leaf(a), leaf(b)))
    flat3.leaf_idx = np.array([0, 1, 1, 1], np.int32)
    with pytest.raises(IndexOveruse):
        _lib.PlanHandle(flat3)
    del c


def test_result_indices_reference_order():
    for c in CASES:
        flat = case_flat(c)
        h = _lib.PlanHandle(flat)
        assert h.result_indices([]) == c["expected"]["unsliced"]["indices"], c["name"]


def test_random_mem_cost_vs_oracle():
    rng = random.Random(3)
    for c in [c for c in CASES if c["family"] in ("random_network", "cnf")]:
        flat = case_flat(c)
        h = _lib.PlanHandle(flat)
        occ = np.bincount(flat.leaf_idx, minlength=len(flat.domain))
        bonds = np.nonzero(occ == 2)[0].tolist()
        for _ in range(4):
            drop = rng.sample(bonds, rng.randint(0, len(bonds))) if bonds else []
            assert h.mem_cost(drop) == oracle.mem_cost(flat, drop)


@pytest.mark.parametrize("name", ["c1a", "c2", "c1b", "c3", "c4", "c5"])
def test_frozen_plans_memory_model(name):
    path = os.path.join(PLANS, f"{name}.tcplan.npz")
    flat, meta = planfile.load(path)
    h = _lib.PlanHandle(flat)
    info = h.info()
    assert info.mem_cost.value() == int(meta["mem_cost_unsliced"])  # reference mem_cost at planning time
    assert info.max_rank == meta["max_rank"]
    assert info.contraction_ops.value() == meta["contraction_ops"]


def test_greedy_prefix_matches_reference_on_c1a():
    counts = json.load(open(os.path.join(GOLDEN, "counts.json")))
    key = next((k for k in counts if k.startswith("c1a_greedy")), None)
    if key is None:
        pytest.skip("reference greedy prefix not recorded")
    flat, _ = planfile.load(os.path.join(PLANS, "c1a.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    chosen = []
    for _ in counts[key]["ids"]:
        chosen.append(h.choose_slice_index(chosen))
    assert chosen == counts[key]["ids"]
    assert [repr(flat.indices[i].id) for i in chosen] == counts[key]["id_reprs"]


def test_planfile_roundtrip(tmp_path):
    c = next(c for c in CASES if c["name"] == "cnf_example4")
    flat = case_flat(c)
    p = tmp_path / "x.tcplan.npz"
    planfile.save(str(p), flat, {"k": 1})
    back, meta = planfile.load(str(p))
    assert meta == {"k": 1}
    for f in ("domain", "sort_rank", "leaf_idx_off", "leaf_idx", "leaf_val_off", "leaf_val", "left", "right"):
        assert np.array_equal(getattr(back, f), getattr(flat, f))
    assert [ix.id for ix in back.indices] == [ix.id for ix in flat.indices]
    n, t = planfile.to_objects(back)
    again = flatten(n, t)
    assert np.array_equal(again.left, flat.left) and again.root_slot == flat.root_slot


def test_generators_deterministic():
    from paper_2006_15512_b200.generators import banded_3cnf, grid_ising, uniform_3cnf
    assert uniform_3cnf(30, 3.0, 1) == uniform_3cnf(30, 3.0, 1)
    assert banded_3cnf(200, 3.5, 29, 1).count("\n") == 1 + 700 + 200
    g = grid_ising(4, 1)
    assert g.startswith("p cnf 40 96")


def _flat_equal(x, y):
    for f in ("domain", "sort_rank", "leaf_idx_off", "leaf_idx", "leaf_val_off", "leaf_val", "left", "right"):
        assert np.array_equal(getattr(x, f), getattr(y, f)), f
    assert x.root_slot == y.root_slot
    assert [ix.id for ix in x.indices] == [ix.id for ix in y.indices]


def test_native_flatten_matches_python_spec():
    from paper_2006_15512_b200.flatten import _native, flatten_py
    assert _native() is not None, "host extension _tcflat not built"
    for c in CASES[:40]:
        n, t = planfile.to_objects(case_flat(c))
        _flat_equal(flatten(n, t), flatten_py(n, t))
    n, t = planfile.to_objects(planfile.load(os.path.join(PLANS, "c1a.tcplan.npz"))[0])
    _flat_equal(flatten(n, t), flatten_py(n, t))


def test_native_flatten_views_dtypes_and_mismatch():
    from paper_2006_15512_b200 import Index, Tensor, TensorNetwork
    from paper_2006_15512_b200.flatten import flatten_py
    from paper_2006_15512_b200.network import join, leaf
    i, j, k = Index("i", 2), Index("j", 3), Index(("k", 1), 2)
    base = np.arange(12.0).reshape(2, 3, 2)
    a = Tensor((i, j), base[:, :, 1])          # non-contiguous view
    b = Tensor((Index("j", 3), k), np.ones((3, 2), dtype=np.float32).T.T)  # equal-by-id, distinct object
    s = Tensor((), np.array(2.5))
    n = TensorNetwork((a, b, s))
    t = join(join(leaf(a), leaf(b)), leaf(s))
    x, y = flatten(n, t), flatten_py(n, t)
    _flat_equal(x, y)
    assert list(x.leaf_val[:6]) == [1.0, 3.0, 5.0, 7.0, 9.0, 11.0]
    other = Tensor((i,), np.ones(2))
    bad = flatten(n, join(join(leaf(a), leaf(other)), leaf(s)))
    assert (bad.left < 0).any() or (bad.right < 0).any()


def test_tie_compression_stats_on_benchmark_plan():
    """Copy-tensor pieces are stored over tie blocks: the executed work of the
    C2 plan is a small fraction of the dense per-node work; the dense path
    (TC_NO_TIES=1) keeps dense variables and the same reference accounting."""
    flat, _ = planfile.load(os.path.join(PLANS, "c2.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    tied = h.compile_stats([])
    os.environ["TC_NO_TIES"] = "1"
    try:
        dense = h.compile_stats([])
    finally:
        del os.environ["TC_NO_TIES"]
    assert tied["n_tied_leaves"] > 10000 and dense["n_tied_leaves"] == 0
    assert tied["alg_bytes"] == dense["alg_bytes"] and tied["alg_flops"] == dense["alg_flops"]
    assert tied["mem_estimate"] == dense["mem_estimate"] and tied["peak_observed"] == dense["peak_observed"]
    assert tied["phys_bytes"] * 10 < dense["phys_bytes"]
    assert tied["phys_flops"] * 100 < dense["phys_flops"]
    assert tied["device_peak_bytes"] * 10 < dense["device_peak_bytes"]


def test_benchmark_formula_satisfiability():
    """Every benchmark formula is satisfiable (reject seeds whose
    count is 0).  C4's seeds 1-10 (banded(400, 4.0, 36)) and C5's seeds 1-5
    (banded(400, 4.0, 34)) are UNSAT; the configs use the first SAT seed."""
    z3 = pytest.importorskip("z3")
    from paper_2006_15512_b200.generators import config_dimacs

    def sat(text):
        s = z3.Solver()
        xs = {}
        for line in text.splitlines():
            if not line or line[0] in "cpw":
                continue
            lits = [int(x) for x in line.split()[:-1]]
            if lits:
                s.add(z3.Or([xs.setdefault(abs(l), z3.Bool(f"x{abs(l)}")) if l > 0
                             else z3.Not(xs.setdefault(abs(l), z3.Bool(f"x{abs(l)}"))) for l in lits]))
        return s.check() == z3.sat

    from paper_2006_15512_b200.generators import CONFIGS, banded_3cnf

    for name in ("c2", "c3", "c4", "c5"):
        assert sat(config_dimacs(name)), name
    for name in ("c4", "c5"):
        c = CONFIGS[name]
        assert not any(sat(banded_3cnf(c["n"], c["ratio"], c["window"], s)) for s in range(1, c["seed"])), name


def test_native_flatten_merges_equal_ids_in_first_appearance_order():
    from paper_2006_15512_b200 import Index, Tensor, TensorNetwork
    from paper_2006_15512_b200.flatten import flatten_py
    from paper_2006_15512_b200.network import join, leaf
    i1, i2 = Index(("a", 1), 2), Index(("a", 1), 2)
    j = Index("j", 3)
    k1, k2 = Index("k", 2), Index("k", 2)
    f = Index("free", 2)
    a = Tensor((i1, j), np.arange(6.0))
    b = Tensor((j, i2, k1), np.arange(12.0))
    c = Tensor((k2, f), np.arange(4.0))
    n = TensorNetwork((a, b, c))
    t = join(join(leaf(a), leaf(b)), leaf(c))
    x = flatten(n, t)
    _flat_equal(x, flatten_py(n, t))
    assert [q.id for q in x.indices] == [("a", 1), "j", "k", "free"]
    assert x.leaf_idx.tolist() == [0, 1, 1, 0, 2, 2, 3]


def test_hoisting_compile_on_cpu(monkeypatch):
    """Slice-invariant hoisting (compile only): on C4's 2^8-slice plan the
    prologue holds most of the executed bytes, the reference accounting is
    unchanged, and TC_HOIST=0 (read per call) restores per-slice re-execution."""
    flat, _ = planfile.load(os.path.join(PLANS, "c4.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(8):
        ch.append(h.choose_slice_index(ch))
    on = h.compile_stats(ch)
    monkeypatch.setenv("TC_HOIST", "0")
    off = h.compile_stats(ch)
    assert on["phys_bytes"] == off["phys_bytes"] and off["phys_bytes_hoisted"] == 0
    assert on["mem_estimate"] == off["mem_estimate"] and on["peak_observed"] == off["peak_observed"]
    assert on["phys_bytes_hoisted"] > 0.5 * on["phys_bytes"]
    assert on["launches_prologue"] > 0 and on["pinned_bytes"] > 0 and off["launches_prologue"] == 0
    # unsliced plans are never hoisted
    assert h.compile_stats([])["launches_prologue"] == 0


def test_slice_blocks_compile_on_cpu(monkeypatch):
    """The block tier (C4, 8 greedy picks): per-slice nodes that do not depend
    on the last chosen index run once per block of 2 slices; the reference
    accounting and the executed work per slice are unchanged, TC_BLOCK=0
    (read per call) runs them per slice."""
    flat, _ = planfile.load(os.path.join(PLANS, "c4.tcplan.npz"))
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(8):
        ch.append(h.choose_slice_index(ch))
    on = h.compile_stats(ch)
    monkeypatch.setenv("TC_SLICE_ORDER", "0")
    lex = h.compile_stats(ch)
    monkeypatch.setenv("TC_BLOCK", "0")
    off = h.compile_stats(ch)
    # the slice order makes 3 of the 8 chosen indices fast (blocks of 8); the
    # lexicographic order only the last (blocks of 2)
    assert on["slices_per_block"] == 8 and lex["slices_per_block"] == 2 and off["slices_per_block"] == 1
    assert on["launches_block"] > 0 and off["launches_block"] == 0 and off["phys_bytes_block"] == 0
    assert 0 < on["phys_bytes_block"] < on["phys_bytes"] - on["phys_bytes_hoisted"]
    assert on["phys_bytes"] == off["phys_bytes"] and on["phys_bytes_hoisted"] == off["phys_bytes_hoisted"]
    assert on["mem_estimate"] == off["mem_estimate"] and on["peak_observed"] == off["peak_observed"]
    # (a tiny level may split into a block and a per-slice launch: one step more)
    assert 0 <= on["launches_block"] + on["launches_per_slice"] - off["launches_per_slice"] <= 4


def test_budget_semantics_match_reference_loop():
    """sliced_execute's budget loop is ``while mem_cost(chosen) > mem_budget``
    (slicing.py:120-128) for any real budget: inf / nan / a budget beyond int64
    never slice when the plan fits, a non-integral budget slices like its
    floor, and an unreachable one raises BudgetInfeasible with the reference's
    wording."""
    case = next(c for c in CASES if "budgeted" in c["expected"] and "error" not in c["expected"]["budgeted"])
    flat = case_flat(case)
    h = _lib.PlanHandle(flat)
    full = h.mem_cost([])
    assert h._budget_slices(float("inf")) == ([], _lib.INT64_MIN)
    assert h._budget_slices(float("nan")) == ([], _lib.INT64_MIN)
    assert h._budget_slices(2 ** 80) == ([], _lib.INT64_MIN)
    assert h._budget_slices(full) == ([], _lib.INT64_MIN)
    b = case["expected"]["budgeted"]["budget"]
    assert h._budget_slices(b) == (None, b)  # libtc's greedy (pinned by test_greedy_slice_set_matches_reference)
    ch, _ = h._budget_slices(b + 0.5)
    assert ch == case["expected"]["budgeted"]["chosen"]
    with pytest.raises(BudgetInfeasible, match=r"cannot fit in -0.5 bytes even fully sliced \(needs \d+\)"):
        h._budget_slices(-0.5)


def test_native_index_positions_identity_then_id():
    from paper_2006_15512_b200.flatten import _native
    from paper_2006_15512_b200.tensor import Index

    nat = _native()
    idx = [Index(("v", k), 2) for k in range(50)]
    twin = Index(("v", 7), 2)  # equal by id, another object
    got = nat.positions(idx, [idx[3], twin, Index("absent", 2), idx[3], idx[49]])
    assert got == [3, 7, -1, 3, 49]
    assert nat.positions([], [twin]) == [-1] and nat.positions(idx, []) == []
