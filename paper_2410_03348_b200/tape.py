"""Reference-compatible ``GradientTape`` on top of torch autograd (tensor.py:141-199).

The reference ships its own reverse-mode tape; here gradients are plain torch autograd.
The shim keeps the calling convention of programs written against the reference:
``tape.leaf(data)`` creates a differentiable device tensor and ``tape.backward(loss)``
returns ``{leaf: grad}`` (zeros for leaves that do not reach the loss).
"""

from __future__ import annotations

import numpy as np
import torch


class DomainError(ValueError):
    """Raised when an input lies outside an operation's domain."""


class GradientTape:
    def __init__(self, device=None, dtype=torch.float64):
        self._leaves = []
        self.device = device
        self.dtype = dtype

    def leaf(self, data) -> torch.Tensor:
        dev = self.device
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        if isinstance(data, torch.Tensor):
            t = data.detach().to(device=dev, dtype=self.dtype).clone()
        else:
            arr = np.asarray(data, dtype=np.float64)
            t = torch.as_tensor(arr, device=dev, dtype=self.dtype)
        if not bool(torch.isfinite(t).all()):
            raise DomainError("gradient-tape leaves must be finite")
        t.requires_grad_(True)
        self._leaves.append(t)
        return t

    def backward(self, loss: torch.Tensor) -> dict:
        if loss.numel() != 1:
            raise ValueError(f"backward requires a scalar loss, got shape {tuple(loss.shape)}")
        leaves = [t for t in self._leaves]
        if not leaves:
            return {}
        grads = torch.autograd.grad(loss.reshape(()), leaves, allow_unused=True)
        return {t: (torch.zeros_like(t) if g is None else g) for t, g in zip(leaves, grads)}
