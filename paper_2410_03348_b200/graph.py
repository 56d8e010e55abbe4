"""Whole-step CUDA-graph capture for fixed-shape programs (public API).

A neurosymbolic training step runs the same program on every batch: the symbol lists,
hence the memoised plans, and all tensor shapes are fixed.  ``GraphedStep`` captures the
step — every ``apply`` / ``filter`` / ``union`` kernel, the loss and the backward — in
one CUDA graph after an eager warm-up (which builds and uploads the plans), so each later
call costs one graph launch plus the copies of the new inputs into the captured buffers.

All static inputs of a capture live in one device arena, and ``pinned_inputs()`` hands
out pinned host views laid out like it, so a step's inputs go up in ONE async H2D copy.
With ``slots=2`` two captures alternate and ``submit`` streams the next step's inputs on
a copy stream while the current step computes: the host<->device traffic of step k+1
overlaps the kernels of step k, and the results are read back without stalling the GPU.

This is the B200 replacement for per-op host dispatch: CUDA graphs, not a tracing
compiler.  The step function must be pure in its tensor inputs and may not read tensor
values on the host (no ``.item()``, no ``forward_probs`` inside the step).
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

__all__ = ["GraphedStep"]


class _Slot:
    """One capture: device input arena, its pinned host twin, the graph, its outputs."""

    def __init__(self, layout, arena_bytes, example_inputs, device):
        self.arena = torch.empty(arena_bytes, device=device, dtype=torch.uint8)
        self.inputs = []
        for x, (o, shape, dtype, nbytes) in zip(example_inputs, layout):
            s = self.arena[o:o + nbytes].view(dtype).view(shape)
            s.copy_(x.detach())
            if x.requires_grad:
                s.requires_grad_(True)
            self.inputs.append(s)
        self.layout = layout
        self.host_arena = None
        self.host_views = None
        self.graph = None
        self.outputs = None
        self.copied = torch.cuda.Event()  # H2D of this slot's inputs finished
        self.done = torch.cuda.Event()    # the replay reading this slot's arena finished
        self.used = False

    def pinned(self):
        if self.host_arena is None:
            self.host_arena = torch.empty(self.arena.numel(), dtype=torch.uint8).pin_memory()
            self.host_views = [self.host_arena[o:o + n].view(dt).view(shape) for (o, shape, dt, n) in self.layout]
        return self.host_views


class GraphedStep:
    """Capture ``step_fn(*inputs) -> outputs`` once per slot; replay it on new inputs.

    ``example_inputs`` are device tensors with the shapes/dtypes of every future call;
    inputs that require grad are re-created as leaves so the step can differentiate
    w.r.t. them (e.g. ``torch.autograd.grad(loss, inputs)``).  Returned outputs are the
    captured static tensors of the slot (overwritten by that slot's next replay).
    """

    _ALIGN = 256  # bytes; every input starts on an aligned offset of the arena

    def __init__(self, step_fn: Callable, example_inputs: Sequence[torch.Tensor], warmup: int = 3, slots: int = 1):
        if not example_inputs:
            raise ValueError("GraphedStep needs at least one example input")
        if slots < 1:
            raise ValueError("slots must be >= 1")
        self.device = example_inputs[0].device
        if self.device.type != "cuda":
            raise ValueError("GraphedStep captures CUDA work; inputs must live on a CUDA device")
        layout, off = [], 0
        for x in example_inputs:
            nbytes = x.numel() * x.element_size()
            layout.append((off, x.shape, x.dtype, nbytes))
            off += -(-nbytes // self._ALIGN) * self._ALIGN
        self._slots = [_Slot(layout, max(off, self._ALIGN), example_inputs, self.device) for _ in range(slots)]
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                step_fn(*self._slots[0].inputs)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        for s in self._slots:
            s.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(s.graph, capture_error_mode="thread_local"):
                s.outputs = step_fn(*s.inputs)
        torch.cuda.synchronize(self.device)
        self._copy_stream = torch.cuda.Stream(self.device)
        self._next = 0

    # ---- backwards-compatible single-slot view
    @property
    def static_inputs(self):
        return self._slots[0].inputs

    @property
    def static_outputs(self):
        return self._slots[0].outputs

    @property
    def graph(self):
        return self._slots[0].graph

    def pinned_inputs(self, slot: int = 0):
        """Pinned host tensors, one per input, laid out like the slot's device arena: fill
        them and pass them back (``__call__``) or call ``submit(slot)`` to upload the whole
        step with one async H2D copy.  Waits until the slot's previous upload has left the
        host buffer, so the views are safe to overwrite."""
        s = self._slots[slot]
        if s.used:
            s.copied.synchronize()
        return list(s.pinned())

    def __call__(self, *inputs: torch.Tensor):
        """Synchronous-order replay of slot 0 on the current stream (copies, then graph)."""
        s = self._slots[0]
        if len(inputs) != len(s.inputs):
            raise ValueError(f"expected {len(s.inputs)} inputs, got {len(inputs)}")
        with torch.no_grad():
            hv = s.host_views
            if hv is not None and all(x is h for x, h in zip(inputs, hv)):
                s.arena.copy_(s.host_arena, non_blocking=True)
            else:
                for d, x in zip(s.inputs, inputs):
                    if x is not d:
                        d.copy_(x, non_blocking=True)
        s.graph.replay()
        return s.outputs

    def next_slot(self) -> int:
        """The slot the next ``submit()`` without an explicit slot will use."""
        return self._next

    def submit(self, slot: int | None = None):
        """Pipelined step: upload the slot's pinned inputs on the copy stream (after the
        slot's previous replay has consumed its arena), then replay the slot's graph on the
        current stream once the upload landed.  Returns the slot's outputs; they are ready
        when the current stream reaches this point (e.g. after a non_blocking D2H + event)."""
        if slot is None:
            slot = self._next
            self._next = (self._next + 1) % len(self._slots)
        s = self._slots[slot]
        if s.host_arena is None:
            raise ValueError("submit() uploads the slot's pinned_inputs(); fill them first")
        compute = torch.cuda.current_stream(self.device)
        cs = self._copy_stream
        if s.used:
            cs.wait_event(s.done)
        with torch.cuda.stream(cs):
            s.arena.copy_(s.host_arena, non_blocking=True)
            s.copied.record(cs)
        compute.wait_event(s.copied)
        s.graph.replay()
        s.done.record(compute)
        s.used = True
        return s.outputs
