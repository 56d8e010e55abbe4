"""Whole-step CUDA-graph capture for fixed-shape programs (public API).

A neurosymbolic training step runs the same program on every batch: the symbol lists,
hence the memoised plans, and all tensor shapes are fixed.  ``GraphedStep`` captures the
step — every ``apply`` / ``filter`` / ``union`` kernel, the loss and the backward — in
one CUDA graph after an eager warm-up (which builds and uploads the plans), so each later
call costs one graph launch plus the copies of the new inputs into the captured buffers
(from pinned host memory they are asynchronous H2D copies on the same stream).

This is the B200 replacement for per-op host dispatch: CUDA graphs, not a tracing
compiler.  The step function must be pure in its tensor inputs and may not read tensor
values on the host (no ``.item()``, no ``forward_probs`` inside the step).
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

__all__ = ["GraphedStep"]


class GraphedStep:
    """Capture ``step_fn(*inputs) -> outputs`` once; ``__call__`` replays it on new inputs.

    ``example_inputs`` are device tensors with the shapes/dtypes of every future call;
    inputs that require grad are re-created as leaves so the step can differentiate
    w.r.t. them (e.g. ``torch.autograd.grad(loss, inputs)``).  Returned outputs are the
    captured static tensors (overwritten by the next call).
    """

    _ALIGN = 256  # bytes; every input starts on an aligned offset of the arena

    def __init__(self, step_fn: Callable, example_inputs: Sequence[torch.Tensor], warmup: int = 3):
        if not example_inputs:
            raise ValueError("GraphedStep needs at least one example input")
        self.device = example_inputs[0].device
        if self.device.type != "cuda":
            raise ValueError("GraphedStep captures CUDA work; inputs must live on a CUDA device")
        # all static inputs live in ONE device arena, so inputs staged in the matching
        # pinned host arena (pinned_inputs()) arrive with a single H2D copy per step
        self._layout = []
        off = 0
        for x in example_inputs:
            nbytes = x.numel() * x.element_size()
            self._layout.append((off, x.shape, x.dtype, nbytes))
            off += -(-nbytes // self._ALIGN) * self._ALIGN
        self._arena_bytes = max(off, self._ALIGN)
        self._arena = torch.empty(self._arena_bytes, device=self.device, dtype=torch.uint8)
        self.static_inputs = []
        for x, (o, shape, dtype, nbytes) in zip(example_inputs, self._layout):
            s = self._arena[o:o + nbytes].view(dtype).view(shape)
            s.copy_(x.detach())
            if x.requires_grad:
                s.requires_grad_(True)
            self.static_inputs.append(s)
        self._host_arena = None
        self._host_views = None
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                step_fn(*self.static_inputs)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            out = step_fn(*self.static_inputs)
        self.static_outputs = out
        torch.cuda.synchronize(self.device)

    def pinned_inputs(self):
        """Pinned host tensors, one per input, laid out like the device arena: fill them and
        pass them back to ``__call__`` to upload the whole step with one async H2D copy."""
        if self._host_arena is None:
            self._host_arena = torch.empty(self._arena_bytes, dtype=torch.uint8).pin_memory()
            self._host_views = [self._host_arena[o:o + n].view(dt).view(shape)
                                for (o, shape, dt, n) in self._layout]
        return list(self._host_views)

    def __call__(self, *inputs: torch.Tensor):
        if len(inputs) != len(self.static_inputs):
            raise ValueError(f"expected {len(self.static_inputs)} inputs, got {len(inputs)}")
        with torch.no_grad():
            hv = self._host_views
            if hv is not None and all(x is h for x, h in zip(inputs, hv)):
                self._arena.copy_(self._host_arena, non_blocking=True)
            else:
                for s, x in zip(self.static_inputs, inputs):
                    if x is not s:
                        s.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.static_outputs
