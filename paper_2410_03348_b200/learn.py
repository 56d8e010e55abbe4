"""Training-side callers of the hot path: the reference loss convention and a LeNet
perception model for data-parallel training over NCCL.

``loss_nll`` follows learn.py:92-119 exactly, including its gradient convention: both
floors are ``clamp`` with a pass-through backward (tensor.py:275-287), which plain
``torch.clamp`` would mask.
"""

from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

__all__ = ["PassClamp", "loss_nll", "loss_nll_torch", "LeNet", "Mlp"]


class PassClamp(torch.autograd.Function):
    """clamp(x, lo, hi) whose backward is the identity everywhere (tensor.py:275-287)."""

    @staticmethod
    def forward(ctx, x, lo, hi):
        return x.clamp(lo, hi)

    @staticmethod
    def backward(ctx, g):
        return g, None, None


def loss_nll(probs: torch.Tensor, targets) -> torch.Tensor:
    """Mean negative log-likelihood of normalised program outputs (learn.py:92-119).

    ``probs`` is ``get_probs(out)`` (batch, n); ``targets`` holds the output-symbol index
    per sample, -1 for "no mass" (None in the reference), which contributes the floor's
    log penalty.  Runs as one fused sm_100a kernel forward and one backward (fp64 inside,
    float64 scalar loss).
    """
    from . import ops

    b, n = probs.shape
    targets = _check_targets(targets, b, n)
    targets = targets.to(device=probs.device, dtype=torch.int64).contiguous()
    if probs.dtype != torch.float32:
        probs = probs.float()
    pnb = probs.t()
    chain = ops.known_chain(pnb)
    if chain is not None:  # the output of a fused Sum-N chain: one fused backward
        n0, kf, B, base, filters, states, rowsum, _ = chain
        return ops.ChainNllLoss.apply((n0, kf, B, states, rowsum), pnb.detach(), targets, base, *filters)
    return ops.NllLoss.apply(pnb, targets)


def _check_targets(targets, b: int, n: int) -> torch.Tensor:
    """The reference's target contract (learn.py:102-112): ``len(targets) == b``
    (ValueError) and every target None or in [0, n) (IndexError).  Host targets are
    checked here; device targets are checked with one reduction unless a CUDA graph is
    being captured — the kernels additionally turn any target outside [-1, n) into a NaN
    loss and gradient instead of reading out of bounds."""
    if not isinstance(targets, torch.Tensor):
        targets = list(targets)
        if len(targets) != b:
            raise ValueError(f"{len(targets)} targets for batch of {b}")
        for t in targets:
            if t is not None and not 0 <= t < n:
                raise IndexError(f"target index {t} out of range for {n} symbols")
        return torch.as_tensor([(-1 if t is None else int(t)) for t in targets], dtype=torch.int64)
    if targets.ndim != 1 or targets.shape[0] != b:
        raise ValueError(f"{targets.shape[0] if targets.ndim else 1} targets for batch of {b}")
    if targets.is_floating_point() or targets.is_complex():
        raise ValueError(f"targets must be integer symbol indices, got {targets.dtype}")
    if targets.is_cuda:
        if torch.cuda.is_current_stream_capturing():
            return targets
        if getattr(targets, "_sg_checked", None) == (targets._version, n):  # already range-checked
            return targets
    bad = (targets < -1) | (targets >= n)
    if bool(bad.any()):
        t = int(targets[bad][0])
        raise IndexError(f"target index {t} out of range for {n} symbols")
    if targets.is_cuda:
        targets._sg_checked = (targets._version, n)
    return targets


def loss_nll_torch(probs: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    """The same loss composed from torch ops (reference check for the fused kernel)."""
    b, n = probs.shape
    p = probs.double()
    rowsum = p.sum(dim=1, keepdim=True)
    norm = p / (rowsum + 1e-8)
    floored = PassClamp.apply(norm, 1e-12, float("inf"))
    valid = targets >= 0
    idx = targets.clamp(min=0).long().view(b, 1)
    picked = floored.gather(1, idx).view(b) * valid.to(p.dtype)
    total = torch.log(PassClamp.apply(picked, 1e-12, float("inf"))).sum()
    return total * (-1.0 / b)


class LeNet(nn.Module):
    """LeNet-5 style digit/token classifier for 28x28 inputs, softmax output."""

    def __init__(self, n_classes: int = 10):
        super().__init__()
        self.conv1 = nn.Conv2d(1, 6, 5, padding=2)
        self.conv2 = nn.Conv2d(6, 16, 5)
        self.fc1 = nn.Linear(16 * 5 * 5, 120)
        self.fc2 = nn.Linear(120, 84)
        self.fc3 = nn.Linear(84, n_classes)

    def forward(self, x):
        x = F.max_pool2d(F.relu(self.conv1(x)), 2)
        x = F.max_pool2d(F.relu(self.conv2(x)), 2)
        x = x.flatten(1)
        x = F.relu(self.fc1(x))
        x = F.relu(self.fc2(x))
        return F.softmax(self.fc3(x), dim=1)


class Mlp(nn.Module):
    """The reference's perception model (learn.py:36-70): 784 -> 128 ReLU -> C softmax,
    with its initialisation (normal(0, 1/sqrt(fan_in)) weights, zero biases)."""

    def __init__(self, in_dim: int = 784, hidden: int = 128, n_classes: int = 10, seed: int = 0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.fc1 = nn.Linear(in_dim, hidden)
        self.fc2 = nn.Linear(hidden, n_classes)
        with torch.no_grad():
            self.fc1.weight.copy_(torch.randn(hidden, in_dim, generator=g) / in_dim**0.5)
            self.fc2.weight.copy_(torch.randn(n_classes, hidden, generator=g) / hidden**0.5)
            self.fc1.bias.zero_()
            self.fc2.bias.zero_()

    def forward(self, x):
        return F.softmax(self.fc2(F.relu(self.fc1(x))), dim=-1)
