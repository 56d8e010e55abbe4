"""Device-resident fixpoint driver for closures (programs.py:177-196).

A closure iterates ``derived <- union(derived, apply_if(f, cond, derived, facts))`` until
the symbol set stops growing.  The stopping test reads SYMBOLS only, which the host owns:
the number of iterations and every plan are a pure function of the fact symbol list, so
a closure never needs a device->host transfer, and its whole tag computation — every
iteration's fused apply and union kernels, ``get_probs`` and (optionally) the loss and
the backward — is one fixed launch sequence.

``closure`` is the eager driver (memoised plans; the reference loop's semantics).
``GraphedClosure`` captures the closure for a fixed fact symbol list as one CUDA graph
per slot (``graph.GraphedStep``) and replays it on new fact probabilities: one graph
launch per batch instead of ``iterations x (apply + union)`` host dispatches.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

from .distribution import Distribution, ProgramContext, apply_if, get_probs, make_distribution, union
from .graph import GraphedStep

__all__ = ["closure", "closure_iterations", "GraphedClosure"]


def closure(f: Callable, cond: Callable | None, facts: Distribution, derived: Distribution | None = None,
            max_iters: int | None = None) -> Distribution:
    """Least fixpoint of ``derived = union(derived, apply_if(f, cond, derived, facts))``
    starting from ``derived`` (default: the facts), as programs.py:177-196.  The symbol
    comparison is a host set test; no tag value leaves the device."""
    derived = facts if derived is None else derived
    it = 0
    while True:
        new = apply_if(f, cond, derived, facts)
        merged = union(derived, new)
        it += 1
        if set(merged.symbols) == set(derived.symbols):
            return merged
        if max_iters is not None and it >= max_iters:
            raise RuntimeError(f"closure did not converge in {max_iters} iterations")
        derived = merged


def closure_iterations(f: Callable, cond: Callable | None, symbols: Sequence) -> int:
    """Number of apply+union rounds the closure of ``symbols`` runs (host-only: uses the
    memoised plans of the same symbol lists, no tags)."""
    from .plan import build_plan

    facts = tuple(symbols)
    derived = facts
    it = 0
    while True:
        plan = build_plan(f, cond, [derived, facts])
        seen = set(derived)
        grown = derived + tuple(s for s in plan.out_symbols if s not in seen)
        it += 1
        if set(grown) == seen:
            return it
        derived = grown


class GraphedClosure:
    """One CUDA graph per slot for ``closure(f, cond, facts)`` over a fixed fact list.

    ``provenance`` is a zero-argument factory (a fresh provenance per context, e.g.
    ``lambda: DtkpAm(5)``); ``example_probs`` is a device ``(B, n_facts)`` tensor.  With
    ``loss_fn(probs) -> scalar`` the capture also runs the loss and its backward and
    returns ``(loss, d loss / d probs)``; otherwise it returns ``probs``.  The output
    symbols are fixed by the fact list and available as ``.symbols``.
    """

    def __init__(self, f: Callable, cond: Callable | None, fact_symbols: Sequence, provenance: Callable,
                 example_probs: torch.Tensor, loss_fn: Callable | None = None, slots: int = 1, warmup: int = 3):
        self.fact_symbols = tuple(fact_symbols)
        self.symbols = None
        grad = loss_fn is not None

        def step(probs):
            ctx = ProgramContext(provenance(), device=probs.device)
            out = closure(f, cond, make_distribution(ctx, probs, self.fact_symbols))
            self.symbols = out.symbols
            p = get_probs(out)
            if not grad:
                return p
            loss = loss_fn(p)
            (g,) = torch.autograd.grad(loss, [probs])
            return loss, g

        x = example_probs.detach()
        if grad:
            x = x.requires_grad_(True)
        self._step = GraphedStep(step, [x], warmup=warmup, slots=slots)

    def __call__(self, probs: torch.Tensor):
        """Copy ``probs`` into the capture and replay it (current stream)."""
        return self._step(probs)

    @property
    def graphed_step(self) -> GraphedStep:
        return self._step
