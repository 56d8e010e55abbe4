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

__all__ = ["shard_range", "plan_fingerprint", "assert_plans_replicated", "max_over_ranks", "rank_world",
           "FlatGradReducer"]


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


class FlatGradReducer:
    """The training step's one collective: the perception gradients averaged over ranks.

    Every parameter's ``.grad`` is a view into ONE flat fp32 buffer, so ``loss.backward()``
    accumulates straight into it and the average is a single ``all_reduce`` (NCCL over
    NVLink on B200, gloo in the CPU tests) — no per-parameter launches and no bucket
    copies.  ``zero_`` / ``backward`` / ``all_reduce_`` / ``optimizer.step()`` are all
    capturable, so a whole data-parallel train step (collective included) replays as one
    CUDA graph.  ``loss_nll`` is a batch mean, so the mean of equal-shard gradients is the
    global-batch gradient.
    """

    def __init__(self, params, group=None):
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no trainable parameters")
        dev = self.params[0].device
        n = sum(p.numel() for p in self.params)
        self.flat = torch.zeros(n, device=dev, dtype=torch.float32)
        off = 0
        for p in self.params:
            if p.dtype != torch.float32:
                raise ValueError("FlatGradReducer keeps fp32 master gradients; parameters must be fp32")
            p.grad = self.flat[off: off + p.numel()].view_as(p)
            off += p.numel()
        self.group = group

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * self.flat.element_size()

    def zero_(self):
        self.flat.zero_()

    def all_reduce_(self):
        """Average the flat gradient over the group's ranks (no-op on one process)."""
        if dist.is_available() and dist.is_initialized():
            world = dist.get_world_size(self.group)
            if world > 1:
                dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
                self.flat.mul_(1.0 / world)
        for p, off in zip(self.params, self._offsets()):
            # autograd may have replaced a view .grad with a fresh tensor (e.g. set_to_none)
            if p.grad is None or p.grad.data_ptr() != self.flat[off:].data_ptr():
                raise RuntimeError("a parameter's .grad no longer aliases the flat buffer; "
                                   "use reducer.zero_() instead of optimizer.zero_grad()")

    def _offsets(self):
        off = 0
        for p in self.params:
            yield off
            off += p.numel()
