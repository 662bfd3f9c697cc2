"""GPU tests of the sliced benchmark configurations and of slice-invariant
hoisting.

* C4 / C5 (SAT-pinned, BASELINE configs[3]/[4]): the slice set is the
  reference greedy's 8 / 12-pick prefix (slicing.py:70-79, libtc's exact port);
  every per-slice value the GPU computes is compared with the exact
  clause-frontier counter (oracle/wmc_dp.c, restating brute_force_count,
  formula.py:183-215) with the sliced variables fixed
  (tests/golden/sliced_dp_*.json), and the folded count with its whole-formula
  count (tests/golden/sliced.json).  Rel. tolerance 1e-9 (north_star).
* C3 (grid 30x30 sliced to rank 28): slices 0-3 against the UNMODIFIED
  reference's own slice path _execute_tracked(*_slice_plan(n, t, eta))
  (slicing.py:30-41, 91-109, 139-145), tests/golden/sliced.json.
* Hoisting (compile.cpp): per-slice results bit-identical with TC_HOIST=0.
* Multi-device slice partition: devices=[0, 0] (peer gather) and, with two
  GPUs, devices=[0, 1] (NCCL all-reduce) give the bits of devices=[0].
"""

import json
import os

import numpy as np
import pytest

from paper_2006_15512_b200 import _lib, planfile, sliced_execute

pytestmark = pytest.mark.gpu

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
GOLD = os.path.join(ROOT, "tests", "golden")
RTOL = 1e-9


def _plan(name):
    return planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))[0]


def _golden(name):
    p = os.path.join(GOLD, "sliced.json")
    return json.load(open(p)).get(name) if os.path.exists(p) else None


def _chosen(flat, gold):
    ids = {repr(ix.id): k for k, ix in enumerate(flat.indices)}
    return [ids[s] for s in gold["chosen"]]


def _per_slice(flat, chosen, b, e, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        h = _lib.PlanHandle(flat)
        ex = _lib.Exec(h, chosen, 0)
        ex.run(b, e)
        folded, per = ex.fetch(e - b)
        return per.reshape(e - b, -1)[:, 0], folded[0], ex
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _close(got, want):
    got, want = np.asarray(got), np.asarray(want)
    scale = np.maximum(np.abs(want), 1e-300)
    return bool(np.all((np.abs(got - want) <= RTOL * scale) | ((got == 0) & (want == 0))))


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_greedy_prefix_is_the_golden_slice_set(name):
    flat = _plan(name)
    gold = _golden(name)
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(len(gold["chosen"])):
        ch.append(h.choose_slice_index(ch))
    assert ch == _chosen(flat, gold)


def test_c4_every_slice_matches_exact_counter():
    """C4: 2^8 slices, each against the exact counter; the slice sum against
    the whole-formula count; the count is non-zero (SAT-pinned seed)."""
    flat = _plan("c4")
    gold = _golden("c4")
    p = os.path.join(GOLD, "sliced_dp_c4.json")
    if not os.path.exists(p):
        pytest.skip("sliced_dp_c4.json not generated")
    dp = json.load(open(p))
    ch = _chosen(flat, gold)
    per, folded, ex = _per_slice(flat, ch, 0, 256)
    assert _close(per, dp["values"])
    assert gold["count"] > 0 and abs(folded - gold["count"]) <= RTOL * gold["count"]
    assert sum(1 for v in dp["values"] if v != 0.0) >= 1


def test_c5_slices_match_exact_counter():
    """C5: 2^12 slices of per-slice max-rank 30.  Slices 0-3, the last one and
    every slice the exact counter finds non-zero, one launch range each."""
    flat = _plan("c5")
    gold = _golden("c5")
    p = os.path.join(GOLD, "sliced_dp_c5.json")
    if not os.path.exists(p):
        pytest.skip("sliced_dp_c5.json not generated")
    dp = json.load(open(p))["values"]
    ch = _chosen(flat, gold)
    h = _lib.PlanHandle(flat)
    ex = _lib.Exec(h, ch, 0)
    picks = sorted({0, 1, 2, 3, len(dp) - 1} | {s for s, v in enumerate(dp) if v != 0.0})
    assert len(picks) > 5  # non-zero slices exist
    for s in picks[:64]:
        ex.run(s, s + 1)
        folded, _ = ex.fetch()
        assert _close([folded[0]], [dp[s]]), s
    assert gold["count"] > 0 and abs(sum(dp) - gold["count"]) <= 1e-9 * gold["count"]


def test_c3_first_slices_match_reference():
    flat = _plan("c3")
    gold = _golden("c3")
    if not gold or not gold.get("slices"):
        pytest.skip("C3 reference slices not generated")
    h = _lib.PlanHandle(flat)
    ch = h.choose_slices_work(2 ** 28)
    assert ch == _chosen(flat, gold)
    ex = _lib.Exec(h, ch, 0)
    for s, rec in sorted(gold["slices"].items(), key=lambda kv: int(kv[0])):
        s = int(s)
        ex.run(s, s + 1)
        folded, _ = ex.fetch()
        assert _close([folded[0]], [rec["value"]]), (s, folded[0], rec["value"])


@pytest.mark.parametrize("name,picks", [("c1b", 3), ("c2", 4), ("c1a", 5), ("c3", -28)])
def test_hoisting_is_bitwise_identical(name, picks):
    """(C3: the work-aware rank-28 slice set, the first 8 of its 2^30 slices;
    thousands of split tiny groups, forced roots read across hoisting.)"""
    flat = _plan(name)
    h = _lib.PlanHandle(flat)
    ch = []
    if picks < 0:
        ch = h.choose_slices_work(2 ** -picks)
        picks = 3
    for _ in range(picks if not ch else 0):
        ch.append(h.choose_slice_index(ch))
    ns = 2 ** picks
    on, fon, exon = _per_slice(flat, ch, 0, ns)
    off, foff, exoff = _per_slice(flat, ch, 0, ns, env={"TC_HOIST": "0"})
    assert on.tobytes() == off.tobytes() and fon == foff
    st_on = h.compile_stats(ch)
    assert st_on["launches_prologue"] > 0 and st_on["phys_bytes_hoisted"] > 0
    # graph replay (repeats > 2 builds the graphs) gives the same bits
    exon.run(0, ns, repeats=3)
    f2, p2 = exon.fetch(ns)
    assert p2.reshape(ns, -1)[:, 0].tobytes() == on.tobytes()


@pytest.mark.parametrize("name,picks", [("c1b", 3), ("c2", 4), ("c1a", 5), ("c3", -28)])
def test_slice_blocks_are_bitwise_identical(name, picks):
    """Block tier (nodes not depending on the last chosen index run once per
    block of consecutive slices) vs TC_BLOCK=0 (every variant node per slice):
    the same bits for a whole pass, a pass starting and ending mid-block (the
    block graph then runs before every slice), one-shot and graph replay."""
    flat = _plan(name)
    h = _lib.PlanHandle(flat)
    ch = []
    if picks < 0:
        ch = h.choose_slices_work(2 ** -picks)
        picks = 3
    for _ in range(picks if not ch else 0):
        ch.append(h.choose_slice_index(ch))
    ns = 2 ** picks
    st = h.compile_stats(ch)
    for b, e in ((0, ns), (1, ns - 1)):
        on, fon, exon = _per_slice(flat, ch, b, e)
        off, foff, _ = _per_slice(flat, ch, b, e, env={"TC_BLOCK": "0"})
        assert on.tobytes() == off.tobytes() and fon == foff, (b, e)
        exon.run(b, e, repeats=3)
        f2, p2 = exon.fetch(e - b)
        assert p2.reshape(e - b, -1)[:, 0].tobytes() == on.tobytes() and f2[0] == fon
    if st["launches_block"]:
        assert st["slices_per_block"] % int(flat.domain[ch[-1]]) == 0


@pytest.mark.parametrize("name,ranges", [("c4", ((0, 32), (3, 21), (64, 128))), ("c5", ((3584, 4096), (3584, 3600)))])
def test_slice_order_is_bitwise_identical(name, ranges):
    """A permuted slice order (C4: 3 fast indices, blocks of 8; C5: 5 fast
    indices, blocks of 32) against the lexicographic order (TC_SLICE_ORDER=0)
    and against per-slice execution (TC_BLOCK=0): the same bits in every
    lexicographic row, for ranges the order maps onto themselves (blocks) and
    for ranges it does not (the lexicographic walk)."""
    flat = _plan(name)
    ch = _chosen(flat, _golden(name))
    st = _lib.PlanHandle(flat).compile_stats(ch)
    assert st["slices_per_block"] > 2
    for b, e in ranges:
        on, fon, _ = _per_slice(flat, ch, b, e)
        lex, flex, _ = _per_slice(flat, ch, b, e, env={"TC_SLICE_ORDER": "0"})
        off, foff, _ = _per_slice(flat, ch, b, e, env={"TC_BLOCK": "0"})
        assert on.tobytes() == lex.tobytes() == off.tobytes() and fon == flex == foff, (b, e)


def test_c4_slice_blocks_cut_work():
    flat = _plan("c4")
    ch = _chosen(flat, _golden("c4"))
    st = _lib.PlanHandle(flat).compile_stats(ch)
    B = st["slices_per_block"]
    inv, blk = st["phys_bytes_hoisted"], st["phys_bytes_block"]
    per_pass = inv + 256 // B * blk + 256 * (st["phys_bytes"] - inv - blk)
    assert B >= 2 and blk > 0.2 * (st["phys_bytes"] - inv)
    assert per_pass < 0.9 * (inv + 256 * (st["phys_bytes"] - inv))


def test_c4_hoisting_cuts_work():
    flat = _plan("c4")
    ch = _chosen(flat, _golden("c4"))
    st = _lib.PlanHandle(flat).compile_stats(ch)
    per_pass_hoisted = st["phys_bytes_hoisted"] + 256 * (st["phys_bytes"] - st["phys_bytes_hoisted"])
    assert per_pass_hoisted < 0.3 * 256 * st["phys_bytes"]


def test_multi_device_partition_same_device_twice():
    """Two workers on one GPU: block partition of the slice ids, peer gather,
    lexicographic fold -> the bits of the single-device run."""
    flat = _plan("c1b")
    n, t = planfile.to_objects(flat)
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(3):
        ch.append(h.choose_slice_index(ch))
    sl = [flat.indices[i] for i in ch]
    one = sliced_execute(n, t, slice_indices=sl, devices=[0])
    two = sliced_execute(n, t, slice_indices=sl, devices=[0, 0])
    assert np.asarray(one.result.values).tobytes() == np.asarray(two.result.values).tobytes()
    assert two.num_slices == 8


@pytest.mark.skipif(_lib.lib().tc_device_count() < 2 if os.path.exists(_lib.LIB_PATH) else True,
                    reason="needs two GPUs")
def test_multi_device_nccl_bitwise():
    flat = _plan("c1b")
    n, t = planfile.to_objects(flat)
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(3):
        ch.append(h.choose_slice_index(ch))
    sl = [flat.indices[i] for i in ch]
    one = sliced_execute(n, t, slice_indices=sl, devices=[0])
    two = sliced_execute(n, t, slice_indices=sl, devices=[0, 1])
    assert np.asarray(one.result.values).tobytes() == np.asarray(two.result.values).tobytes()


def test_nonfinite_leaf_runs_dense_like_the_reference():
    """A non-finite leaf next to structural zeros: the reference contracts an
    identity piece with the Inf-holding delta densely, so 0*Inf = NaN enters
    the sum (tensor.py:96-108).  Tie compression / relabel aliasing would skip
    that term; libtc runs plans with non-finite leaves on dense variables, so
    it produces the reference's NaN/Inf pattern (the oracle restates the
    reference's pairwise order)."""
    from oracle import oracle
    from paper_2006_15512_b200 import Index, Tensor, TensorNetwork, join, leaf
    from paper_2006_15512_b200.flatten import flatten

    i, j, k, m = (Index(c, 2) for c in "ijkm")
    ident = Tensor((i, j), np.eye(2))
    delta = np.zeros((2, 2, 2))
    delta[0, 0, 0], delta[1, 1, 1] = np.inf, 0.5
    d = Tensor((j, k, m), delta)
    w = Tensor((k,), np.array([1.0, 2.0]))
    a = Tensor((i,), np.array([0.25, 3.0]))
    n = TensorNetwork((a, ident, d, w))
    t = join(join(leaf(ident), leaf(d)), join(leaf(a), leaf(w)))
    got = np.asarray(sliced_execute(n, t).result.values, dtype=np.float64).reshape(-1)
    want = np.asarray(oracle.sliced_execute(flatten(n, t))["values"], dtype=np.float64).reshape(-1)
    assert np.isnan(want).any()  # the reference's 0 * Inf
    assert np.array_equal(np.isnan(got), np.isnan(want)) and np.array_equal(np.isinf(got), np.isinf(want))
    fin = np.isfinite(want)
    assert np.allclose(got[fin], want[fin], rtol=1e-12)


def test_distributed_sliced_execute_single_rank_nccl():
    """distributed.sliced_execute in a 1-rank NCCL group equals sliced_execute bit for bit."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2006_15512_b200 import distributed

    flat = _plan("c1b")
    n, t = planfile.to_objects(flat)
    h = _lib.PlanHandle(flat)
    ch = []
    for _ in range(3):
        ch.append(h.choose_slice_index(ch))
    sl = [flat.indices[i] for i in ch]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        got = distributed.sliced_execute(n, t, slice_indices=sl, device=0)
        part = distributed.sliced_execute(n, t, slice_indices=sl, device=0, slice_range=(2, 5))
    finally:
        dist.destroy_process_group()
    want = sliced_execute(n, t, slice_indices=sl, devices=[0])
    assert np.asarray(got.result.values).tobytes() == np.asarray(want.result.values).tobytes()
    assert got.num_slices == 8 and part.num_slices == 3
    blk = sliced_execute(n, t, slice_indices=sl, devices=[0], slice_range=(2, 5))
    assert np.asarray(part.result.values).tobytes() == np.asarray(blk.result.values).tobytes()


def _per_slice_subprocess(env, name, picks):
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np\n"
            "from paper_2006_15512_b200 import _lib, planfile\n"
            "f, _ = planfile.load(%r + '/data/plans/%s.tcplan.npz')\n"
            "h = _lib.PlanHandle(f); ch = []\n"
            "for _ in range(%d): ch.append(h.choose_slice_index(ch))\n"
            "ex = _lib.Exec(h, ch, 0); ns = ex.num_slices()\n"
            "ex.run(0, ns, repeats=3)\n"
            "fo, per = ex.fetch(ns)\n"
            "print(per.tobytes().hex(), fo.tobytes().hex())\n") % (ROOT, ROOT, name, picks)
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return res.stdout.split()


@pytest.mark.parametrize("name,picks", [("c1b", 3), ("c2", 4)])
def test_slice_lanes_are_bitwise_identical(name, picks):
    """Concurrent slice lanes (TC_LANES, read once per process) change only
    which stream runs a slice: every per-slice value and the fold are the
    same bits as one lane."""
    one = _per_slice_subprocess({"TC_LANES": "1"}, name, picks)
    for k in ("3", "4", "8"):
        assert _per_slice_subprocess({"TC_LANES": k}, name, picks) == one, k
