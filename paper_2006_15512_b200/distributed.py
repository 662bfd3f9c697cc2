"""Multi-process slice scheduling (one process per GPU, torch.distributed).

Slices are independent (Thm 5; same tree per slice,
slicing.py:30-41), so rank g executes the contiguous block of lexicographic
slice ids ``slice_block(NS, G, g)`` (first sliced index slowest,
slicing.py:138-139).  The only collective is ONE all-reduce (sum) of a
zero-padded [NS, R] FP64 vector in which every position has exactly one
non-zero contributor, so the reduction is exact (x + 0 = x) under any NCCL
algorithm; every rank then folds the vector left-to-right in lexicographic
order — the reference's ``add`` order (slicing.py:144) — so the count is
bitwise identical for G = 1, 2, 4, 8.

For unsliced plans (C1, C2) the path does not shard: ``--gpus N`` runs N
independent replicas (no collective) — see DESIGN.md.
"""

from __future__ import annotations


def slice_block(num_slices: int, world: int, rank: int):
    per = -(-num_slices // world)
    b = min(num_slices, rank * per)
    return b, min(num_slices, b + per)


def gather_slices(local, begin: int, num_slices: int, group=None):
    """Zero-padded all-reduce of this rank's per-slice block [n_local, R]
    (a torch tensor on the rank's device, or CPU for gloo) -> [NS, R]."""
    import torch
    import torch.distributed as dist

    R = local.shape[1] if local.dim() == 2 else 1
    # gloo (CPU tests, ranks sharing a GPU) reduces host tensors
    dev = "cpu" if dist.get_backend(group) == "gloo" else local.device
    full = torch.zeros((num_slices, R), dtype=torch.float64, device=dev)
    if local.numel():
        full[begin:begin + local.shape[0]] = local.reshape(-1, R).to(dev)
    dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full.to(local.device)


def fold(full):
    """Lexicographic left fold on the device that holds ``full`` (libtc's
    deterministic k_fold for CUDA tensors)."""
    import torch

    if full.is_cuda:
        from . import _lib

        out = torch.empty(full.shape[1], dtype=torch.float64, device=full.device)
        torch.cuda.synchronize(full.device)
        _lib.fold_device(full.data_ptr(), full.shape[1], full.shape[0], out.data_ptr(), full.device.index)
        return out
    raise ValueError("fold() runs on the GPU; CPU tensors are test-only")


def sliced_execute(n, t, mem_budget=None, *, slice_indices=None, device=None, group=None, slice_range=None):
    """Algorithm 3 across the ranks of a torch.distributed group (one process
    per GPU): every rank plans the same slice set, executes its block of the
    lexicographic slice ids on its own GPU, and the blocks meet in ONE
    zero-padded all-reduce followed by the lexicographic fold — bitwise the
    single-device result.  ``slice_range=(b, e)`` restricts the job to slices
    b..e-1 (split over the ranks in the same way).  Returns the reference's
    SlicedExecution fields (``num_slices`` = slices executed by all ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _lib
    from .slicing import SlicedExecution, _ids, _plan

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.cuda.current_device() if device is None else int(device)
    flat, h = _plan(n, t, with_sort_rank=mem_budget is not None and slice_indices is None)
    if slice_indices is not None:
        chosen = _ids(flat, slice_indices)
    elif mem_budget is not None:
        chosen = h.choose_slices(mem_budget)
    else:
        chosen = []
    ex = _lib.Exec(h, chosen, dev)
    ns = ex.num_slices()
    lo, hi = (int(x) for x in slice_range) if slice_range is not None else (0, ns)
    b, e = slice_block(hi - lo, world, rank)
    b, e = lo + b, lo + e
    st = ex.run(b, e) if e > b else None
    R = ex.result_size()
    # the copy runs on libtc's stream: the buffer must have no pending write on
    # torch's stream (a zero fill there could land after the copy)
    local = torch.empty((e - b, R), dtype=torch.float64, device=torch.device("cuda", dev))
    if e > b:
        torch.cuda.current_stream(dev).synchronize()
        ex.copy_results(local.data_ptr())
    full = gather_slices(local, b - lo, hi - lo, group=group)
    out = fold(full).cpu().numpy()
    idx = h.result_indices(chosen)
    tensor_cls = type(n.tensors[0])
    shape = tuple(int(flat.domain[i]) for i in idx)
    res = tensor_cls(tuple(flat.indices[i] for i in idx), np.asarray(out, dtype=np.float64).reshape(shape))
    st = st or {}
    return SlicedExecution(result=res, sliced_indices=[flat.indices[i] for i in chosen],
                           mem_estimate=st.get("mem_estimate", h.mem_cost(chosen)),
                           peak_observed=st.get("peak_observed", 0), num_slices=hi - lo, stats=st)
