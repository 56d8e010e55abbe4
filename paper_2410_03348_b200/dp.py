"""Data-parallel plumbing for the hot path (one process per GPU, torch.distributed).

The symbolic path shards along the batch with no data-path collective: every tag
kernel is per-sample independent, and symbol plans are a pure function of the symbol
lists, so each rank builds identical plans itself (``plan_fingerprint`` lets a run assert
that).  The only collective in training is DDP's gradient all-reduce of the perception
network (NCCL over NVLink on B200; gloo in the CPU tests), after ``loss.backward()``.
``loss_nll`` is a batch mean, so the mean of equal-size shard gradients equals the
global-batch gradient.  Timing is the max over ranks of device-measured time.
"""

from __future__ import annotations

import hashlib

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_range", "plan_fingerprint", "assert_plans_replicated", "max_over_ranks", "rank_world"]


def rank_world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(global_batch: int, rank: int, world: int):
    """Contiguous [start, stop) rows of the global batch owned by ``rank`` (equal sizes
    when divisible; the first ``global_batch % world`` ranks get one extra row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def plan_fingerprint(plan) -> str:
    """Stable digest of a SymbolPlan (output symbols, kept combinations, output index)."""
    h = hashlib.sha1()
    h.update(repr(plan.out_symbols).encode())
    h.update(np.ascontiguousarray(plan.combos).tobytes())
    h.update(np.ascontiguousarray(plan.out_idx).tobytes())
    h.update(repr(plan.sizes).encode())
    return h.hexdigest()


def assert_plans_replicated(plans, group=None):
    """All ranks built bit-identical plans (raises on divergence, e.g. rank-local sampling)."""
    mine = [plan_fingerprint(p) for p in plans]
    if not (dist.is_available() and dist.is_initialized()):
        return mine
    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    for r, other in enumerate(gathered):
        if other != mine:
            raise RuntimeError(f"symbol plans diverge between this rank and rank {r}")
    return mine


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. device-timed milliseconds) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
