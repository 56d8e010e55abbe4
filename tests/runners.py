"""Run a golden workload on the CPU oracle or on the CUDA path, with identical inputs."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import golden_cases as G

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz")
    out = {k: z[k] for k in z.files}
    out["symbols"] = json.loads(str(out["symbols"]))
    return out


class OracleAPI:
    """The oracle mini-runtime under the reference API names (test infrastructure)."""

    from paper_2410_03348_b200.plan import UNDEFINED  # the marker the shared symbol functions return

    @staticmethod
    def apply(f, *d):
        from oracle import programs as OP

        return OP.apply(f, *d)

    @staticmethod
    def apply_if(f, cond, *d):
        from oracle import programs as OP

        return OP.apply_if(f, cond, *d)

    @staticmethod
    def union(a, b):
        from oracle import programs as OP

        return OP.union(a, b)

    @staticmethod
    def sample_symbols(d, m, seed=None, strategy="top"):
        from oracle import programs as OP

        return OP.sample_symbols(d, m, seed=seed, strategy=strategy)

    @staticmethod
    def stack(parts):
        from oracle import programs as OP

        return OP.stack(parts)


class OracleP:
    from paper_2410_03348_b200.programs import Coord

    @staticmethod
    def sum_n(ctx, d):
        from oracle import programs as OP

        return OP.sum_n(d)

    @staticmethod
    def hwf(ctx, d, length):
        from oracle import programs as OP

        return OP.hwf(ctx, d, length)

    @staticmethod
    def path_closure(ctx, edges):
        from oracle import programs as OP
        from paper_2410_03348_b200.programs import _ends_match, _join_ends

        return OP.closure(edges, edges, _join_ends, _ends_match)


def run_oracle(name, inputs=None):
    from oracle import programs as OP

    prov, k, prog, syms_fn, _, _ = G.CASES[name]
    inputs = G.case_inputs(name) if inputs is None else inputs
    ctx = OP.OContext(prov, k, undefined=OracleAPI.UNDEFINED)
    dists = [OP.make_distribution(ctx, x, s) for x, s in zip(inputs, syms_fn(OracleP))]
    out = prog(OracleAPI, OracleP, ctx, dists)
    probs = OP.get_probs(out)
    w = G.loss_weights(name, probs.shape)
    grads = OP.grad_inputs(out, w)
    res = {"symbols": [repr(s) for s in out.symbols], "probs": probs, "grads": grads, "w": w}
    if prov == "dtkp":
        from oracle import algebra as A

        m, p = A.pad_width(out.tag, ctx.width)
        res["member"], res["present"] = m, p
    return res


def run_gpu(name, inputs=None, device="cuda"):
    import torch

    import paper_2410_03348_b200 as sg
    from paper_2410_03348_b200 import programs as P

    prov, k, prog, syms_fn, _, _ = G.CASES[name]
    inputs = G.case_inputs(name) if inputs is None else inputs
    ctx = sg.ProgramContext(sg.provenance_from_name(prov, k or 1), device=device)
    leaves = [torch.tensor(x, device=device, dtype=torch.float32, requires_grad=True) for x in inputs]
    dists = [sg.make_distribution(ctx, lf, s) for lf, s in zip(leaves, syms_fn(P))]
    out = prog(sg, P, ctx, dists)
    probs = sg.get_probs(out)
    w = G.loss_weights(name, tuple(probs.shape))
    loss = (probs.double() * torch.as_tensor(w, device=device)).sum()
    loss.backward()
    res = {
        "symbols": [repr(s) for s in out.symbols],
        "probs": probs.detach().double().cpu().numpy(),
        "grads": [lf.grad.double().cpu().numpy() if lf.grad is not None else np.zeros(lf.shape) for lf in leaves],
        "w": w,
    }
    if prov == "dtkp":
        res["member"] = out.tags.member
        res["present"] = out.tags.present
    return res


def assert_close_rel(got, ref, rtol, floor_frac=1e-6, what=""):
    """|got - ref| <= rtol * |ref| + floor_frac * max|ref| (BASELINE tolerance + abs floor)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} != {ref.shape}"
    scale = np.max(np.abs(ref)) if ref.size else 0.0
    err = np.abs(got - ref)
    bound = rtol * np.abs(ref) + floor_frac * scale + 1e-30
    bad = err > bound
    assert not bad.any(), (
        f"{what}: {int(bad.sum())}/{bad.size} entries out of tolerance; worst rel "
        f"{float((err / np.maximum(np.abs(ref), 1e-30)).max()):.3e}"
    )
