"""GPU tests of tie-aware execution (compile.cpp "physical variables").

FactorTree's copy-tensor pieces are generalised diagonals; libtc stores such
leaves over their tie blocks and propagates ties through the tree (union-find,
push-down to where two tied indices meet).  These tests build random networks
rich in identity / delta / weighted-diagonal pieces -- with free indices tied at
the root, diagonal reads of internal operands, batch variables, explicit slices
through tied leaves -- and check the result against a dense numpy einsum of the
whole network and against libtc's own dense path (TC_NO_TIES=1, read per call).
"""

import os
import random
import string

import numpy as np
import pytest

from paper_2006_15512_b200 import Index, Tensor, TensorNetwork, join, leaf, planfile, sliced_execute
from paper_2006_15512_b200 import _lib

pytestmark = pytest.mark.gpu


def _delta(inds, w=None):
    r = len(inds)
    v = np.zeros([2] * r)
    v[(0,) * r] = 1.0 if w is None else w[0]
    v[(1,) * r] = 1.0 if w is None else w[1]
    return Tensor(tuple(inds), v)


def _random_tied_network(rng, n_tensors):
    """Tensors of rank 1-3 over dim-2 indices, each index in <= 2 tensors;
    about half are identity / delta / weighted-diagonal pieces."""
    stubs = []
    specs = []
    for t in range(n_tensors):
        r = rng.choice([1, 2, 2, 3, 3, 3])
        specs.append(r)
        stubs += [t] * r
    rng.shuffle(stubs)
    inds = [[] for _ in range(n_tensors)]
    k = 0
    while stubs:
        a = stubs.pop()
        partner = next((j for j, b in enumerate(stubs) if b != a), None)
        ix = Index(("x", k), 2)
        k += 1
        inds[a].append(ix)
        if partner is not None and rng.random() < 0.9:
            inds[stubs.pop(partner)].append(ix)
    ts = []
    for t in range(n_tensors):
        ii = inds[t]
        kind = rng.random()
        if len(ii) >= 2 and kind < 0.35:
            ts.append(_delta(ii))
        elif len(ii) >= 2 and kind < 0.5:
            ts.append(_delta(ii, (rng.uniform(0.2, 1), rng.uniform(0.2, 1))))
        else:
            shape = [2] * len(ii)
            ts.append(Tensor(tuple(ii), np.array([rng.uniform(-1, 1) for _ in range(2 ** len(ii))]).reshape(shape)))
    return TensorNetwork(tuple(ts))


def _random_tree(rng, tensors):
    nodes = [leaf(t) for t in tensors]
    while len(nodes) > 1:
        i, j = sorted(rng.sample(range(len(nodes)), 2))
        b = nodes.pop(j)
        a = nodes.pop(i)
        nodes.append(join(a, b) if rng.random() < 0.5 else join(b, a))
    return nodes[0]


def _einsum(n, order):
    letters = {}
    pool = iter(string.ascii_letters)
    ops, subs = [], []
    for t in n.tensors:
        s = ""
        for ix in t.indices:
            if ix.id not in letters:
                letters[ix.id] = next(pool)
            s += letters[ix.id]
        subs.append(s)
        ops.append(np.asarray(t.values))
    out = "".join(letters[ix.id] for ix in order)
    return np.einsum(",".join(subs) + "->" + out, *ops, optimize=True)


def _run(n, t, **kw):
    r = sliced_execute(n, t, **kw)
    return r, np.asarray(r.result.values)


def _dense(n, t, **kw):
    os.environ["TC_NO_TIES"] = "1"
    try:
        return _run(n, t, **kw)
    finally:
        del os.environ["TC_NO_TIES"]


@pytest.mark.parametrize("seed", range(40))
def test_random_tied_networks_match_dense(seed):
    rng = random.Random(1000 + seed)
    n = _random_tied_network(rng, rng.randint(6, 16))
    t = _random_tree(rng, list(n.tensors))
    out, got = _run(n, t)
    want = _einsum(n, out.result.indices)
    assert got.shape == want.shape
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    d, dv = _dense(n, t)
    assert list(d.result.indices) == list(out.result.indices)
    assert np.allclose(got, dv, rtol=1e-12, atol=1e-13)
    assert out.mem_estimate == d.mem_estimate and out.peak_observed == d.peak_observed
    # an explicit slice through bonds (possibly inside tied blocks)
    bonds = sorted({ix.id for ix in n.bond_indices}, key=repr)
    if bonds:
        pick = [Index(b, 2) for b in rng.sample(bonds, min(2, len(bonds)))]
        s, sv = _run(n, t, slice_indices=pick)
        assert s.num_slices == 2 ** len(pick)
        assert np.allclose(sv, got, rtol=1e-12, atol=1e-12)


def test_root_with_tied_free_indices():
    """The root keeps two indices tied by a delta piece: the dense result has
    structural zeros off the diagonal (root_map expansion)."""
    rng = np.random.default_rng(3)
    i, j, k, l = (Index(c, 2) for c in "ijkl")
    a = Tensor((i, j), rng.uniform(-1, 1, (2, 2)))
    d = _delta((j, k, l))  # k and l stay free, tied
    n = TensorNetwork((a, d))
    out, got = _run(n, join(leaf(a), leaf(d)))
    assert [ix.id for ix in out.result.indices] == ["i", "k", "l"]
    want = np.einsum("ij,jkl->ikl", a.values, d.values)
    assert np.array_equal(got, want)
    assert got[:, 0, 1].tolist() == [0.0, 0.0] and got[:, 1, 0].tolist() == [0.0, 0.0]


def test_diagonal_read_and_pushdown():
    """delta(s1, s2, f) contracts two separate indices of an internal operand:
    the tie is pushed down to where s1 and s2 meet."""
    rng = np.random.default_rng(5)
    idx = [Index(("q", c), 2) for c in range(14)]
    a = Tensor(tuple(idx[0:7]), rng.uniform(-1, 1, [2] * 7))
    b = Tensor(tuple(idx[7:14]), rng.uniform(-1, 1, [2] * 7))
    f = Index("f", 2)
    d = _delta((idx[3], idx[10], f))
    n = TensorNetwork((a, b, d))
    t = join(join(leaf(a), leaf(b)), leaf(d))
    out, got = _run(n, t)
    want = _einsum(n, out.result.indices)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["c1a", "c2"])
def test_benchmark_plan_dense_path_agrees(name):
    flat, _ = planfile.load(os.path.join(os.path.dirname(__file__), "..", "data", "plans", f"{name}.tcplan.npz"))
    n, t = planfile.to_objects(flat)
    tied, tv = _run(n, t)
    dense, dv = _dense(n, t)
    assert abs(float(tv) - float(dv)) <= 1e-12 * abs(float(dv))
    st = _lib.PlanHandle(flat).compile_stats([])
    assert st["n_tied_leaves"] > 0 and st["phys_bytes"] < st["alg_bytes"]


def test_c4_unsliced_fits_and_matches_exact_count():
    """C4 (2.5 TiB dense mem_cost) runs unsliced on one B200 through the tied
    tensors; the count matches the exact counter (tests/golden/sliced.json)."""
    import json

    flat, _ = planfile.load(os.path.join(os.path.dirname(__file__), "..", "data", "plans", "c4.tcplan.npz"))
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sliced.json")))["c4"]["count"]
    n, t = planfile.to_objects(flat)
    out, v = _run(n, t)
    assert gold > 0 and abs(float(v) - gold) <= 1e-9 * gold
    assert out.mem_estimate > 1000 * 2 ** 30 and out.stats["device_peak_bytes"] < 40 * 2 ** 30


def test_absurd_slice_counts_raise_instead_of_crashing():
    """2^62 slices: the per-slice result buffer cannot exist; the call must
    fail with MemoryError (TC_OOM), not crash or hang."""
    flat, _ = planfile.load(os.path.join(os.path.dirname(__file__), "..", "data", "plans", "c1a.tcplan.npz"))
    n, t = planfile.to_objects(flat)
    bonds = sorted(n.bond_indices, key=lambda ix: repr(ix.id))[:62]
    with pytest.raises(MemoryError):
        sliced_execute(n, t, slice_indices=bonds)


def _run_plans_subprocess(env_over):
    import subprocess
    import sys

    root = os.path.join(os.path.dirname(__file__), "..")
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np\n"
            "from paper_2006_15512_b200 import planfile, sliced_execute\n"
            "for name in ('c1a', 'c2', 'c1b'):\n"
            "    f, _ = planfile.load(%r + '/data/plans/' + name + '.tcplan.npz')\n"
            "    n, t = planfile.to_objects(f)\n"
            "    r = sliced_execute(n, t)\n"
            "    print(name, float(np.asarray(r.result.values)).hex(), r.stats['gpu_launches'])\n") % (root, root)
    env = dict(os.environ, **env_over)
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return {ln.split()[0]: (float.fromhex(ln.split()[1]), int(ln.split()[2])) for ln in res.stdout.strip().splitlines()}


def test_chain_link_fusion_is_bitwise_identical():
    """k_stream_pair computes each fused chain link with the operations and
    order of the two separate steps: the counts are bit-identical to a run
    with fusion disabled (TC_FUSE=0, read once per process -> subprocess).
    """
    on = _run_plans_subprocess({"TC_FUSE": "1"})
    off = _run_plans_subprocess({"TC_FUSE": "0"})
    for name in ("c1a", "c2", "c1b"):
        assert on[name][0] == off[name][0], name  # same bits
    assert on["c2"][1] < off["c2"][1]  # fewer launches when fused


def _chain_network(seed):
    """A rank-17 tensor contracted in turn with 14 small pieces (summing 1-2
    of its indices, adding 0-2 new ones; some pieces are weighted deltas,
    whose ties make later steps batch steps)."""
    rng = np.random.default_rng(100 + seed)
    pyr = random.Random(200 + seed)
    cur = [Index(("b", i), 2) for i in range(17)]
    big = Tensor(tuple(cur), rng.uniform(-1, 1, [2] * 17))
    tree = leaf(big)
    tensors = [big]
    fresh = 0
    for step in range(14):
        summed = pyr.sample(cur, pyr.choice([1, 1, 2]))
        new = [Index(("n", fresh + j), 2) for j in range(pyr.choice([0, 1, 1, 2]) if len(cur) > 15 else pyr.choice([1, 2]))]
        fresh += len(new)
        kept = [ix for ix in cur if ix not in summed]
        inds = summed + new
        if pyr.random() < 0.3 and len(inds) >= 2:
            piece = _delta(inds, (rng.uniform(0.2, 1), rng.uniform(0.2, 1)))
        else:
            piece = Tensor(tuple(inds), rng.uniform(-1, 1, [2] * len(inds)))
        tensors.append(piece)
        tree = join(tree, leaf(piece)) if pyr.random() < 0.5 else join(leaf(piece), tree)
        cur = kept + new
    return TensorNetwork(tuple(tensors)), tree


def _check_chain(seed):
    n, tree = _chain_network(seed)
    out, got = _run(n, tree)
    want = _einsum(n, out.result.indices)
    assert got.shape == want.shape
    assert np.allclose(got, want, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("seed", range(6))
def test_stream_chains(seed):
    """Stream-kernel chains (k_stream, fused pairs) against a dense einsum."""
    _check_chain(seed)


def _big_chain_network(seed, rank=24, steps=8):
    """A rank-24 tensor (128 MB) through a chain of small pieces: launches of
    >= 2^12 chunks (grid-stride 'persistent' stream kernels, fused pairs)."""
    rng = np.random.default_rng(300 + seed)
    pyr = random.Random(400 + seed)
    cur = [Index(("B", i), 2) for i in range(rank)]
    big = Tensor(tuple(cur), rng.uniform(-1, 1, [2] * rank))
    tree = leaf(big)
    tensors = [big]
    for step in range(steps):
        summed = pyr.sample(cur, pyr.choice([1, 2]))
        new = [Index(("N", seed, step, j), 2) for j in range(len(summed))]
        kept = [ix for ix in cur if ix not in summed]
        piece = Tensor(tuple(summed + new), rng.uniform(-1, 1, [2] * (2 * len(summed))))
        tensors.append(piece)
        tree = join(tree, leaf(piece))
        cur = kept + new
    return TensorNetwork(tuple(tensors)), tree


def test_large_stream_launches_modes_bitwise():
    """Grid-stride (TC_STREAM_PERSIST, default from 2^12 chunks) vs per-CTA
    chunk blocks (TC_STREAM_PERSIST=0), fused vs unfused (TC_FUSE): the same
    bits for a 128 MB chain (env read once per process -> subprocesses)."""
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import numpy as np, test_gpu_ties as T\n"
            "n, t = T._big_chain_network(0)\n"
            "out, v = T._run(n, t)\n"
            "print(np.asarray(v).tobytes().hex()[:4096], float(np.abs(np.asarray(v)).sum()))\n") % (os.path.join(here, ".."), here)
    outs = []
    for env in ({}, {"TC_STREAM_PERSIST": "0"}, {"TC_FUSE": "0"}, {"TC_STREAM_PERSIST": "0", "TC_FUSE": "0"}):
        res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                             timeout=900)
        assert res.returncode == 0, res.stderr[-3000:]
        outs.append(res.stdout.strip())
    assert len(set(outs)) == 1, outs
