"""World-size-2 gloo test of the multi-rank slice path (CPU): block
partition of the lexicographic slice ids, the zero-padded all-reduce is exact,
and the lexicographic fold of the gathered vector equals the single-process
Algorithm 3 sum bit for bit.  Per-slice parts come from the CPU oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_15512_b200.distributed import gather_slices, slice_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, flat_path, chosen, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2006_15512_b200 import planfile

    flat, _ = planfile.load(flat_path)
    ns = 1
    for i in chosen:
        ns *= int(flat.domain[i])
    b, e = slice_block(ns, world, rank)
    parts = []
    for s in range(b, e):
        # one slice = the network with the sliced indices fixed to the
        # mixed-radix digits of s (first chosen slowest); oracle restatement
        sub = _slice_flat(flat, chosen, s)
        parts.append(oracle.sliced_execute(sub)["values"])
    local = torch.tensor(np.array(parts).reshape(len(parts), -1) if parts else np.zeros((0, 1)), dtype=torch.float64)
    full = gather_slices(local, b, ns)
    acc = full[0].clone()
    for s in range(1, ns):
        acc = acc + full[s]
    if rank == 0:
        out_q.put((full.numpy().copy(), acc.numpy().copy()))
    dist.destroy_process_group()


def _slice_flat(flat, chosen, s):
    """FlatPlan with each chosen index fixed (K5 semantics, tensor.py:118-125)."""
    import copy
    digits = {}
    for i in reversed(chosen):
        d = int(flat.domain[i])
        digits[i] = s % d
        s //= d
    out = copy.copy(flat)
    new_idx, new_off, new_val, new_voff = [], [0], [], [0]
    for l in range(flat.num_leaves):
        ids = flat.leaf_idx[flat.leaf_idx_off[l]:flat.leaf_idx_off[l + 1]].tolist()
        vals = flat.leaf_val[flat.leaf_val_off[l]:flat.leaf_val_off[l + 1]]
        shape = [int(flat.domain[i]) for i in ids]
        v = vals.reshape(shape) if shape else vals.reshape(())
        sel = tuple(digits[i] if i in digits else slice(None) for i in ids)
        v = v[sel] if ids else v
        keep = [i for i in ids if i not in digits]
        new_idx += keep
        new_off.append(len(new_idx))
        new_val += list(np.asarray(v).reshape(-1))
        new_voff.append(len(new_val))
    out.leaf_idx = np.array(new_idx, np.int32)
    out.leaf_idx_off = np.array(new_off, np.int64)
    out.leaf_val = np.array(new_val, np.float64)
    out.leaf_val_off = np.array(new_voff, np.int64)
    return out


def test_slice_block_partition():
    for ns in (1, 7, 256, 4096):
        for g in (1, 2, 4, 8):
            blocks = [slice_block(ns, g, r) for r in range(g)]
            covered = [s for b, e in blocks for s in range(b, e)]
            assert covered == list(range(ns))


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process(tmp_path):
    from conftest import GOLDEN, case_flat, load_cases
    from oracle import oracle
    from paper_2006_15512_b200 import planfile

    case = next(c for c in load_cases() if c["name"] == "random_network_3")
    flat = case_flat(case)
    path = str(tmp_path / "p.tcplan.npz")
    planfile.save(path, flat)
    occ = np.bincount(flat.leaf_idx, minlength=len(flat.domain))
    bonds = [int(i) for i in np.nonzero(occ == 2)[0]][:2]
    want = oracle.sliced_execute(flat, slice_ids=bonds)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, path, bonds, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, acc = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert full.shape[0] == want["num_slices"]
    # bitwise: same fold order as Algorithm 3 in the oracle
    assert acc.tobytes() == np.asarray(want["values"]).tobytes()
