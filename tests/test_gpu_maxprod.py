"""GPU parity of the max-product ("max/DAMP") variant: sg_maxprod_fwd / sg_maxprod_bwd
through the public API and the decomposed provenance operators, against the oracle
(oracle/algebra.py max_*, itself pinned to fixtures made from the reference's Tensor
primitives).  Values within 1e-5 relative; first-argmax gradient routing exact."""

import numpy as np
import pytest
import torch

from oracle import algebra as A

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def _rows(rng, B, n):
    r = rng.uniform(0.05, 1.0, size=(B, n))
    return (r / r.sum(axis=1, keepdims=True)).astype(np.float32).astype(np.float64)


def _close(got, ref, what, floor=1e-7):
    got = np.asarray(got, dtype=np.float64)
    tol = RTOL * np.abs(ref) + floor * max(1.0, float(np.abs(ref).max(initial=0.0)))
    bad = np.abs(got - ref) > tol
    assert not bad.any(), f"{what}: {int(bad.sum())} mismatches, max err {float(np.abs(got - ref).max())}"


@pytest.mark.parametrize("arity,size,B", [(2, 37, 64), (3, 7, 40), (2, 10, 300), (1, 12, 33)])
def test_max_apply_sum_vs_oracle(cuda, arity, size, B):
    import paper_2410_03348_b200 as sg

    rng = np.random.default_rng(arity * 100 + size)
    xs = [_rows(rng, B, size) for _ in range(arity)]
    ctx = sg.ProgramContext(sg.DampMax(), device="cuda")
    leaves = [torch.tensor(x, device="cuda", dtype=torch.float32, requires_grad=True) for x in xs]
    ds = [sg.make_distribution(ctx, lf, list(range(size))) for lf in leaves]
    f = (lambda *a: sum(a) % 17) if arity > 1 else (lambda a: a % 5)
    out = sg.apply(f, *ds)
    probs = sg.get_probs(out)
    w = rng.uniform(-1, 1, size=tuple(probs.shape))
    (probs.double() * torch.as_tensor(w, device="cuda")).sum().backward()
    syms, combos, out_idx = A.map_shuffle(f, None, [list(range(size))] * arity, object())
    assert [int(s) for s in out.symbols] == list(syms)
    ref, arg = A.max_apply(xs, combos, out_idx, len(syms))
    _close(probs.detach().cpu().numpy(), ref, "max probs")
    for lf, g in zip(leaves, A.max_apply_grad(xs, combos, arg, w)):
        _close(lf.grad.double().cpu().numpy(), g, "max grads", floor=1e-6)


def test_max_ties_route_to_first_record(cuda):
    """Uniform inputs make every product of an output equal: the gradient must go to the
    earliest combination only (tensor.py:319-325)."""
    import paper_2410_03348_b200 as sg

    B, n = 4, 6
    x = torch.full((B, n), 1.0 / n, device="cuda", requires_grad=True)
    y = torch.full((B, n), 1.0 / n, device="cuda", requires_grad=True)
    ctx = sg.ProgramContext(sg.DampMax(), device="cuda")
    out = sg.apply(lambda a, b: a + b, sg.make_distribution(ctx, x, list(range(n))),
                   sg.make_distribution(ctx, y, list(range(n))))
    probs = sg.get_probs(out)
    probs.sum().backward()
    xs = [np.full((B, n), 1.0 / n)] * 2
    syms, combos, out_idx = A.map_shuffle(lambda a, b: a + b, None, [list(range(n))] * 2, object())
    _, arg = A.max_apply([np.float32(v).astype(np.float64) for v in xs], combos, out_idx, len(syms))
    gx, gy = A.max_apply_grad([x.detach().double().cpu().numpy(), y.detach().double().cpu().numpy()], combos, arg,
                              np.ones((B, len(syms))))
    _close(x.grad.double().cpu().numpy(), gx, "tie grads x")
    _close(y.grad.double().cpu().numpy(), gy, "tie grads y")
    # output s = a + b first derives from (max(0, s - 5), ...): x row min(s, 5) gets no other
    assert (x.grad[:, 0] > 0).all() and (y.grad[:, n - 1] > 0).all()


def test_max_decomposed_operators(cuda):
    from paper_2410_03348_b200 import provenance as PV

    prov = PV.DampMax()
    rng = np.random.default_rng(5)
    B = 48
    a_np, b_np = _rows(rng, B, 7), _rows(rng, B, 7)
    a = PV.DampTags(torch.tensor(a_np, device="cuda", dtype=torch.float32))
    b = PV.DampTags(torch.tensor(b_np, device="cuda", dtype=torch.float32))
    _close(prov.conj(a, b).value.cpu().numpy(), a_np * b_np, "conj")
    _close(prov.disj(a, b).value.cpu().numpy(), np.clip(np.maximum(a_np, b_np), 0, 1), "disj")
    groups = [[0, 3, 5], [1], [], [2, 4, 6, 0]]
    got = prov.group_disj(a, groups).value.cpu().numpy()
    ref = np.stack([a_np[:, g].max(axis=1) if g else np.zeros(B) for g in groups], axis=1)
    _close(got, ref, "group_disj")
    _close(prov.gather(a, [6, 0, 6]).value.cpu().numpy(), a_np[:, [6, 0, 6]], "gather")


def _max_sum_chain(xs, fuse, targets=None, w=None):
    import paper_2410_03348_b200 as sg
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.learn import loss_nll

    old = sg.DampMax.fuse_chains
    sg.DampMax.fuse_chains = fuse
    try:
        ctx = sg.ProgramContext(sg.DampMax(), device="cuda")
        leaves = [torch.tensor(x, device="cuda", dtype=torch.float32, requires_grad=True) for x in xs]
        out = P.sum_n(ctx, [sg.make_distribution(ctx, lf, list(range(x.shape[1]))) for lf, x in zip(leaves, xs)])
        probs = sg.get_probs(out)
        if targets is not None:
            loss = loss_nll(probs, torch.as_tensor(targets, device="cuda"))
        else:
            loss = (probs.double() * torch.as_tensor(w, device="cuda")).sum()
        loss.backward()
        return out, probs.detach().double().cpu().numpy(), [lf.grad.double().cpu().numpy() for lf in leaves]
    finally:
        sg.DampMax.fuse_chains = old


@pytest.mark.parametrize("n,B", [(15, 1000), (4, 33), (9, 257), (15, 16384)])
def test_max_chain_bit_identical_to_per_apply_kernels(cuda, n, B):
    """The fused max chain (sg_maxchain_*) equals the per-apply sg_maxprod path bit for bit
    (same products, first-argmax routing, fmaf order), loss included."""
    rng = np.random.default_rng(n * 7 + B)
    xs = [_rows(rng, B, 10) for _ in range(n)]
    t = rng.integers(0, 9 * n + 1, size=B)
    out_f, p_f, g_f = _max_sum_chain(xs, True, targets=t)
    out_u, p_u, g_u = _max_sum_chain(xs, False, targets=t)
    assert out_f.symbols == out_u.symbols
    np.testing.assert_array_equal(p_f, p_u)
    for a, b in zip(g_f, g_u):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("uniform", [False, True])
def test_max_chain_vs_oracle(cuda, uniform):
    """Sum-6 under the max variant vs the oracle; uniform inputs make every record of an
    output tie, so every gradient must follow the first-argmax rule exactly."""
    from oracle import programs as OP
    from paper_2410_03348_b200.plan import UNDEFINED

    rng = np.random.default_rng(11)
    B, n = 37, 6
    xs = [np.full((B, 10), 0.1) if uniform else _rows(rng, B, 10) for _ in range(n)]
    xs = [x.astype(np.float32).astype(np.float64) for x in xs]
    w = rng.uniform(-1, 1, size=(B, 9 * n + 1))
    _, probs, grads = _max_sum_chain(xs, True, w=w)
    ctx = OP.OContext("max", None, undefined=UNDEFINED)
    out = OP.sum_n([OP.make_distribution(ctx, x, list(range(10))) for x in xs])
    _close(probs, OP.get_probs(out), "max chain probs")
    for g, r in zip(grads, OP.grad_inputs(out, w)):
        _close(g, r, "max chain grads", floor=1e-6)
