"""GPU parity on randomly generated programs (seeded, reproducible).

Each case draws a provenance (DAMP, or DTKP-AM with k = 1..5), a batch, 2-4 input
distributions with random symbol lists, and a random sequence of `apply` (arity 1-3,
a family of black-box symbol functions, some returning UNDEFINED), `apply_if`, `filter`
and `union` calls; the same program then runs on the CUDA path (through the public API)
and on the CPU oracle, and must agree: symbols and order exactly, DTKP proof membership
and row order bit-exactly, fp32 probabilities and gradients within 1e-5 relative (+ the
1e-6·max absolute floor of SURVEY §8c).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from runners import OracleAPI, assert_close_rel

pytestmark = pytest.mark.gpu

N_CASES = 160


def _rows(rng, B, n):
    r = rng.uniform(0.05, 1.0, size=(B, n))
    return (r / r.sum(axis=1, keepdims=True)).astype(np.float32)


def _make_fn(kind, m, undefined):
    """Deterministic black-box symbol functions over int symbols (no str hashing)."""
    if kind == "sum":
        return lambda *xs: sum(xs) % m
    if kind == "plain":  # f = sum: the Toeplitz paths when the operands are position-aligned
        return lambda *xs: sum(xs)
    if kind == "prod":
        return lambda *xs: int(np.prod(xs)) % m
    if kind == "max":
        return lambda *xs: max(xs)
    if kind == "lin":
        return lambda *xs: sum((i + 2) * x for i, x in enumerate(xs)) % m
    if kind == "undef":
        return lambda *xs: undefined if sum(xs) % 4 == 1 else (xs[0] * 3 + sum(xs)) % m
    raise ValueError(kind)


def _program(seed):
    """A random program description: (prov, k, B, input sizes, ops)."""
    rng = np.random.default_rng(seed)
    prov = "damp" if seed % 2 == 0 else "dtkp"
    k = int(rng.integers(1, 6)) if prov == "dtkp" else None
    B = int(rng.choice([1, 3, 37, 64]))
    n_in = int(rng.integers(2, 5))
    top = 9 if prov == "dtkp" or seed % 4 else 41  # some DAMP cases with long lists (long Toeplitz)
    sizes = [int(rng.integers(1, top)) for _ in range(n_in)]
    ops = []
    n_dists = n_in
    for _ in range(int(rng.integers(2, 6))):
        op = rng.choice(["apply", "apply", "apply_if", "filter", "union"])
        if op in ("apply", "apply_if"):
            arity = int(rng.integers(1, 4)) if op == "apply" else 2
            args = [int(rng.integers(0, n_dists)) for _ in range(arity)]
            kind = str(rng.choice(["sum", "plain", "prod", "max", "lin", "undef"]))
            m = int(rng.integers(3, 12))
            ops.append((op, args, kind, m))
        elif op == "filter":
            ops.append((op, [int(rng.integers(0, n_dists))], int(rng.integers(2, 4)), None))
        else:
            ops.append((op, [int(rng.integers(0, n_dists)), int(rng.integers(0, n_dists))], None, None))
        n_dists += 1
    return prov, k, B, sizes, ops


def _run(api, dists, ops, undefined):
    ds = list(dists)
    for op, args, kind, m in ops:
        xs = [ds[i] for i in args]
        if op == "apply":
            out = api.apply(_make_fn(kind, m, undefined), *xs)
        elif op == "apply_if":
            out = api.apply_if(_make_fn(kind, m, undefined), lambda a, b: (a + b) % 3 != 0, *xs)
        elif op == "filter":
            out = xs[0].filter(lambda s, q=kind: s % q != 0)
        else:
            out = api.union(xs[0], xs[1])
        ds.append(out)
    return ds[-1]


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_program_vs_oracle(cuda, seed):
    import paper_2410_03348_b200 as sg
    from oracle import programs as OP

    prov, k, B, sizes, ops = _program(seed)
    rng = np.random.default_rng(1000 + seed)
    inputs = [_rows(rng, B, n) for n in sizes]
    symbols = [list(range(n)) for n in sizes]

    octx = OP.OContext(prov, k, undefined=OracleAPI.UNDEFINED)
    oout = _run(OracleAPI, [OP.make_distribution(octx, x.astype(np.float64), s) for x, s in zip(inputs, symbols)],
                ops, sg.UNDEFINED)

    ctx = sg.ProgramContext(sg.provenance_from_name(prov, k or 1), device=cuda)
    leaves = [torch.tensor(x, device=cuda, requires_grad=True) for x in inputs]
    out = _run(sg, [sg.make_distribution(ctx, lf, s) for lf, s in zip(leaves, symbols)], ops, sg.UNDEFINED)

    assert [repr(s) for s in out.symbols] == [repr(s) for s in oout.symbols]
    if len(oout.symbols) == 0:
        return
    oprobs = OP.get_probs(oout)
    probs = sg.get_probs(out)
    assert_close_rel(probs.detach().double().cpu().numpy(), oprobs, 1e-5, 1e-6, what=f"seed {seed} probs")
    if prov == "dtkp":
        from oracle import algebra as A

        m, p = A.pad_width(oout.tag, octx.width)
        np.testing.assert_array_equal(out.tags.member, m)
        np.testing.assert_array_equal(out.tags.present, p)
    w = np.random.default_rng(2000 + seed).uniform(-1, 1, size=oprobs.shape)
    ograds = OP.grad_inputs(oout, w)
    (probs.double() * torch.as_tensor(w, device=cuda)).sum().backward()
    for i, (lf, og) in enumerate(zip(leaves, ograds)):
        got = lf.grad.double().cpu().numpy() if lf.grad is not None else np.zeros(og.shape)
        assert_close_rel(got, og, 1e-5, 1e-6, what=f"seed {seed} grad {i}")
