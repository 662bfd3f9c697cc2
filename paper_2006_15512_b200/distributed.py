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
    full = torch.zeros((num_slices, R), dtype=torch.float64, device=local.device)
    if local.numel():
        full[begin:begin + local.shape[0]] = local.reshape(-1, R)
    dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


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
