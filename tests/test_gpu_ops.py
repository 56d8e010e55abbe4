"""GPU: decomposed provenance operators, the drop-in dedup_topk kernel, the fused loss,
worked examples, edge cases and full-size property checks — all against the oracle."""

import numpy as np
import pytest
import torch

import golden_cases as G
from runners import GOLDEN, assert_close_rel

pytestmark = pytest.mark.gpu


def sg():
    import paper_2410_03348_b200 as m

    return m


# ------------------------------------------------------------------ dedup_topk drop-in
def test_dedup_topk_kernel_bit_exact_on_reference_fuzz(cuda):
    from paper_2410_03348_b200 import ops

    z = np.load(GOLDEN / "dedup_topk_fuzz.npz")
    for c in range(int(z["n_cases"])):
        m = torch.as_tensor(z[f"c{c}_member"], device=cuda)
        p = torch.as_tensor(z[f"c{c}_present"], device=cuda)
        pr = torch.as_tensor(z[f"c{c}_p"], device=cuda)
        om, op = ops.dedup_topk(m, p, pr, int(z[f"c{c}_k"]))
        np.testing.assert_array_equal(om.cpu().numpy(), z[f"c{c}_om"])
        np.testing.assert_array_equal(op.cpu().numpy(), z[f"c{c}_op"])


def test_dedup_topk_kernel_matches_oracle_random(cuda):
    from oracle.algebra import dedup_topk as odt
    from paper_2410_03348_b200 import ops

    rng = np.random.default_rng(3)
    for _ in range(40):
        M, R, I, k = int(rng.integers(1, 300)), int(rng.integers(1, 20)), int(rng.integers(0, 300)), int(rng.integers(1, 9))
        member = (rng.uniform(size=(M, R, I)) < 0.3).astype(np.uint8)
        present = (rng.uniform(size=(M, R)) < 0.8).astype(np.uint8)
        p = np.round(rng.uniform(0.0, 1.0, size=(M, I)), 1)
        om, op = ops.dedup_topk(torch.as_tensor(member, device=cuda), torch.as_tensor(present, device=cuda),
                                torch.as_tensor(p, device=cuda), k)
        rm, rp = odt(member, present, p, k)
        np.testing.assert_array_equal(om.cpu().numpy(), rm)
        np.testing.assert_array_equal(op.cpu().numpy(), rp)


def test_dedup_topk_semantics(cuda):
    from paper_2410_03348_b200 import ops

    def run(member, present, p, k):
        om, op = ops.dedup_topk(torch.as_tensor(np.array(member, np.uint8), device=cuda),
                                torch.as_tensor(np.array(present, np.uint8), device=cuda),
                                torch.as_tensor(np.array(p, np.float64), device=cuda), k)
        return om.cpu().numpy(), op.cpu().numpy()

    m, pr = run([[[1, 0], [0, 1], [0, 0]]], [[1, 1, 1]], [[0.2, 0.8]], 3)
    np.testing.assert_array_equal(m[0], [[0, 0], [0, 1], [1, 0]])
    m, pr = run([[[1, 0], [1, 0], [0, 1]]], [[1, 1, 1]], [[0.5, 0.5]], 3)
    assert pr[0].tolist() == [1, 1, 0]
    m, _ = run([[[0, 1], [1, 0]]], [[1, 1]], [[0.5, 0.5]], 1)
    np.testing.assert_array_equal(m[0, 0], [0, 1])
    m, pr = run([[[1, 0], [0, 1]]], [[0, 1]], [[0.9, 0.1]], 2)
    assert pr[0].tolist() == [1, 0]
    m, pr = run(np.eye(4)[None], [[1, 1, 1, 1]], [[0.9, 0.8, 0.7, 0.6]], 2)
    np.testing.assert_array_equal(m[0], [[1, 0, 0, 0], [0, 1, 0, 0]])
    m, pr = run(np.zeros((1, 3, 0)), [[1, 1, 1]], np.zeros((1, 0)), 2)
    assert pr[0].tolist() == [1, 0]


# ------------------------------------------------------------------ worked examples
D1_ROW = [0.00, 0.90, 0.02, 0.012, 0.012, 0.012, 0.012, 0.012, 0.01, 0.01]
D2_ROW = [0.78, 0.09, 0.02, 0.02, 0.02, 0.02, 0.02, 0.01, 0.01, 0.01]


def probs_of(d):
    return {s: p for s, p in zip(d.symbols, d.forward_probs()[0])}


def test_worked_examples(cuda):
    S = sg()
    ctx = S.ProgramContext(S.Damp())
    d1 = S.make_distribution(ctx, [D1_ROW], range(10))
    d2 = S.make_distribution(ctx, [D2_ROW], range(10))
    out = S.apply(lambda x, y: x + y, d1, d2)
    assert probs_of(out)[1] == pytest.approx(0.702, abs=1e-6)
    even = d1.filter(lambda x: x % 2 == 0)
    got = probs_of(even)
    assert set(even.symbols) == {0, 2, 4, 6, 8}
    assert got[0] == 0.0 and got[2] == pytest.approx(0.02, abs=1e-7) and got[8] == pytest.approx(0.01, abs=1e-7)
    ctx = S.ProgramContext(S.Damp())
    a = S.make_distribution(ctx, [[0.01, 0.24]], [0, 1])
    b = S.make_distribution(ctx, [[0.63, 0.37]], [0, 4])
    u = probs_of(S.union(a, b))
    assert u == pytest.approx({0: 0.64, 1: 0.24, 4: 0.37}, abs=1e-6)
    ctx = S.ProgramContext(S.Damp())
    third = [[1 / 3] * 3]
    da = S.make_distribution(ctx, third, [0, 1, 2])
    db = S.make_distribution(ctx, third, [0, 1, 2])
    out = S.apply(lambda x, y: x + y, da, db)
    assert out.symbols == (0, 1, 2, 3, 4)
    np.testing.assert_allclose(out.forward_probs()[0], np.array([1, 2, 3, 2, 1]) / 9.0, atol=1e-6)


def test_get_probs_gradient_to_leaves(cuda):
    S = sg()
    ctx = S.ProgramContext(S.Damp())
    row = ctx.tape.leaf([[0.2, 0.8]])
    d = S.make_distribution(ctx, row, [0, 1])
    out = S.apply(lambda x: x + 1, d)
    loss = S.get_probs(out).sum()
    grads = ctx.tape.backward(loss)
    np.testing.assert_allclose(grads[row].cpu().numpy(), [[1.0, 1.0]])


def test_dtkp_operator_kats(cuda):
    """test_provenance.py:92-158 known answers on the device operators."""
    S = sg()
    reg = S.InputRegistry()
    prov = S.DtkpAm(4)
    base = prov.input_tags(reg, [("x", 0), ("x", 1)], torch.tensor([[0.8, 0.3]], dtype=torch.float64))
    ta, tb = prov.gather(base, [0]), prov.gather(base, [1])
    out = prov.conj(ta, tb)
    assert out.proof_sets()[0] == {frozenset({0, 1})}
    assert prov.forward_probs(out)[0, 0] == pytest.approx(0.24, abs=1e-7)
    prov1 = S.DtkpAm(1)
    reg1 = S.InputRegistry()
    base1 = prov1.input_tags(reg1, [("x", 0), ("x", 1)], torch.tensor([[0.8, 0.3]], dtype=torch.float64))
    assert prov1.disj(prov1.gather(base1, [0]), prov1.gather(base1, [1])).proof_sets()[0] == {frozenset({0})}
    reg2 = S.InputRegistry()
    prov2 = S.DtkpAm(4)
    prov2.input_tags(reg2, [("x", i) for i in range(3)], torch.tensor([[0.9, 0.8, 0.06]], dtype=torch.float64))
    t = prov2.tags_from_proofs(reg2, [{0, 1}, {2}])
    assert prov2.forward_probs(t)[0, 0] == pytest.approx(0.78, abs=1e-6)
    reg3 = S.InputRegistry()
    prov3 = S.DtkpAm(4)
    prov3.input_tags(reg3, [("x", i) for i in range(2)], torch.tensor([[0.9, 0.9]], dtype=torch.float64))
    t = prov3.tags_from_proofs(reg3, [{0}, {1}, {0, 1}])
    assert prov3.forward_probs(t)[0, 0] == 1.0
    assert prov3.forward_probs(prov3.zero(reg3))[0, 0] == 0.0
    assert prov3.forward_probs(prov3.one(reg3))[0, 0] == 1.0


def test_equality_toy_contrasts_provenances(cuda):
    """test_acceptance.py:86-110: DTKP (k >= n) gives exactly 1, DAMP gives sum p^2."""
    S = sg()
    from paper_2410_03348_b200.programs import equality_toy

    rng = np.random.default_rng(0)
    for _ in range(10):
        n = int(rng.integers(2, 7))
        k = int(rng.integers(n, n + 3))
        row = rng.uniform(0.05, 1.0, size=n)
        row /= row.sum()
        ctx = S.ProgramContext(S.DtkpAm(min(k, 8)))
        out = equality_toy(ctx, S.make_distribution(ctx, row.reshape(1, -1), list(range(n))))
        assert probs_of(out)[True] == pytest.approx(1.0, abs=1e-6)
        ctx = S.ProgramContext(S.Damp())
        out = equality_toy(ctx, S.make_distribution(ctx, row.reshape(1, -1), list(range(n))))
        r32 = row.astype(np.float32).astype(np.float64)
        assert probs_of(out)[True] == pytest.approx(float((r32 ** 2).sum()), abs=1e-6)


# ------------------------------------------------------------------ decomposed operators
def test_damp_decomposed_ops_match_numpy(cuda):
    S = sg()
    rng = np.random.default_rng(4)
    prov = S.Damp()
    a_np = rng.uniform(size=(7, 5)).astype(np.float32)
    b_np = rng.uniform(size=(7, 5)).astype(np.float32)
    a = torch.tensor(a_np, device=cuda, requires_grad=True)
    b = torch.tensor(b_np, device=cuda, requires_grad=True)
    ta, tb = S.DampTags(a), S.DampTags(b)
    c = prov.conj(ta, tb)
    np.testing.assert_allclose(c.value.detach().cpu().numpy(), a_np * b_np, rtol=1e-6)
    d = prov.disj(ta, tb)
    np.testing.assert_allclose(d.value.detach().cpu().numpy(), np.clip(a_np + b_np, 0, 1), rtol=1e-6)
    g = prov.group_disj(ta, [[0, 2], [1], [3, 4, 0]])
    ref = np.clip(np.stack([a_np[:, 0] + a_np[:, 2], a_np[:, 1], a_np[:, 3] + a_np[:, 4] + a_np[:, 0]], 1), 0, 1)
    np.testing.assert_allclose(g.value.detach().cpu().numpy(), ref, rtol=1e-6)
    gat = prov.gather(ta, [4, 4, 1])
    np.testing.assert_array_equal(gat.value.detach().cpu().numpy(), a_np[:, [4, 4, 1]])
    (gat.value.sum() + g.value.sum()).backward()
    expect = np.zeros_like(a_np)
    expect[:, 4] += 2
    expect[:, 1] += 1
    for col, times in {0: 2, 1: 1, 2: 1, 3: 1, 4: 1}.items():
        expect[:, col] += times
    np.testing.assert_allclose(a.grad.cpu().numpy(), expect, rtol=1e-6)


def test_dtkp_decomposed_ops_match_oracle(cuda):
    S = sg()
    from oracle import algebra as A

    rng = np.random.default_rng(5)
    for k in (1, 2, 3, 5, 8):
        reg = S.InputRegistry()
        prov = S.DtkpAm(k)
        p = np.round(rng.uniform(0.05, 0.95, size=(3, 9)), 1).astype(np.float32).astype(np.float64)
        base = prov.input_tags(reg, [("x", i) for i in range(9)], torch.tensor(p))
        obase = A.dtkp_input_tags(0, 9, 9, 3, k)
        cur, ocur = prov.gather(base, [0, 1, 2]), A.dtkp_gather(obase, [0, 1, 2])
        for step in range(8):
            idx = rng.integers(0, 9, size=3)
            oth, ooth = prov.gather(base, idx), A.dtkp_gather(obase, idx)
            op = step % 3
            if op == 0:
                cur, ocur = prov.conj(cur, oth), A.dtkp_conj(ocur, ooth, p, k)
            elif op == 1:
                cur, ocur = prov.disj(cur, oth), A.dtkp_disj(ocur, ooth, p, k)
            else:
                groups = [[0, 2], [1], [2, 1, 0]]
                cur, ocur = prov.group_disj(cur, groups), A.dtkp_group_disj(ocur, groups, p, k)
            np.testing.assert_array_equal(cur.member, ocur[0])
            np.testing.assert_array_equal(cur.present, ocur[1])
        np.testing.assert_allclose(prov.forward_probs(cur), A.dtkp_probs(ocur, p), rtol=1e-6)


# ------------------------------------------------------------------ fused loss
def test_fused_nll_matches_torch_composition(cuda):
    from paper_2410_03348_b200.learn import loss_nll, loss_nll_torch

    rng = np.random.default_rng(6)
    p_np = rng.uniform(0.0, 0.3, size=(257, 41)).astype(np.float32)
    p_np[3, :] = 0.0
    t_np = rng.integers(0, 41, size=257)
    t_np[5] = -1
    p1 = torch.tensor(p_np, device=cuda, requires_grad=True)
    p2 = torch.tensor(p_np, device=cuda, requires_grad=True)
    t = torch.as_tensor(t_np, device=cuda)
    l1 = loss_nll(p1, t)
    l2 = loss_nll_torch(p2, t)
    assert float(l1) == pytest.approx(float(l2), rel=1e-12)
    l1.backward()
    l2.backward()
    assert_close_rel(p1.grad.cpu().numpy(), p2.grad.cpu().numpy(), 1e-5, 1e-7, what="nll grad")


# ------------------------------------------------------------------ edge cases
def test_edge_cases(cuda):
    S = sg()
    ctx = S.ProgramContext(S.Damp())
    d = S.make_distribution(ctx, [[0.5, 0.5]], [0, 1])
    assert S.apply(lambda s: S.UNDEFINED if s == 0 else s, d).symbols == (1,)
    empty = d.filter(lambda s: False)
    assert len(S.apply(lambda x, y: x + y, d, empty)) == 0
    assert S.union(d, empty) is d and S.union(empty, d) is d
    assert len(S.apply_if(lambda x: x, lambda x: False, d)) == 0
    assert len(S.apply(lambda x: S.UNDEFINED, d)) == 0
    with pytest.raises(S.SymbolFunctionError) as err:
        S.apply(lambda x, y: x / y, d, d)
    assert err.value.symbols == (0, 0)
    other = S.make_distribution(S.ProgramContext(S.Damp()), [[1.0]], [0])
    with pytest.raises(S.ContextError):
        S.apply(lambda x, y: x + y, d, other)
    d4 = S.make_distribution(ctx, [[0.25] * 4], [3, 1, 2, 0])
    assert S.apply(lambda s: s % 2, d4).symbols == (1, 0)
    S.get_probs(d)
    with pytest.raises(Exception, match="frozen"):
        S.make_distribution(ctx, [[1.0]], [2])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_input_dtypes_and_noncontiguous_views(cuda, dtype):
    S = sg()
    rng = np.random.default_rng(8)
    base = rng.uniform(0.05, 1.0, size=(10, 33)).astype(np.float32)
    x = torch.tensor(base, device=cuda).to(dtype).t()  # (33, 10) non-contiguous view
    y = torch.tensor(rng.uniform(0.05, 1.0, size=(33, 7)).astype(np.float32), device=cuda).to(dtype)
    ctx = S.ProgramContext(S.Damp())
    out = S.apply(lambda a, b: (a * b) % 11, S.make_distribution(ctx, x, range(10)),
                  S.make_distribution(ctx, y, range(7)))
    from oracle import algebra as A

    syms, combos, idx = A.map_shuffle(lambda a, b: (a * b) % 11, None, [list(range(10)), list(range(7))], S.UNDEFINED)
    ref = A.damp_apply([x.float().cpu().double().numpy(), y.float().cpu().double().numpy()], combos, idx, len(syms))
    assert out.symbols == syms
    assert_close_rel(out.forward_probs(), ref, 1e-5, 1e-7)


def test_batch_one_broadcast_and_reuse(cuda):
    from runners import run_gpu, run_oracle

    got, ref = run_gpu("damp_bcast_reuse"), run_oracle("damp_bcast_reuse")
    for g, r in zip(got["grads"], ref["grads"]):
        assert g.shape == r.shape
        assert_close_rel(g, r, 1e-5, 1e-6)


# ------------------------------------------------------------------ generic path at size
@pytest.mark.parametrize("arity,size,B,fn", [
    (2, 1000, 128, "prod"),   # |S|=1000: operands exceed the shared tile (global path), long segments split
    (2, 100, 512, "mod"),
    (3, 30, 256, "lin3"),     # arity 3, not a plain sum: generic segments of up to ~900 combos
    (1, 5000, 96, "mod3"),    # one input, 3 outputs: segments split across items + fix-up
])
def test_generic_apply_vs_oracle(cuda, arity, size, B, fn):
    S = sg()
    from oracle import algebra as A

    f = {"prod": lambda x, y: x * y, "mod": lambda x, y: (x * 7 + y) % 13, "sum": lambda *xs: sum(xs),
         "lin3": lambda x, y, z: x + 2 * y + z, "mod3": lambda x: x % 3}[fn]
    rng = np.random.default_rng(size + arity)
    xs = [G.rows(rng, B, size) for _ in range(arity)]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    out = S.apply(f, *[S.make_distribution(ctx, lf, range(size)) for lf in leaves])
    syms, combos, idx = A.map_shuffle(f, None, [list(range(size))] * arity, S.UNDEFINED)
    assert out.symbols == syms
    ref = A.damp_apply(xs, combos, idx, len(syms))
    got = S.get_probs(out)
    assert_close_rel(got.detach().cpu().numpy(), ref, 1e-5, 1e-7, what="probs")
    w = rng.uniform(-1, 1, size=ref.shape)
    (got.double() * torch.as_tensor(w, device=cuda)).sum().backward()
    for lf, gr in zip(leaves, A.damp_apply_grad(xs, combos, idx, w)):
        assert_close_rel(lf.grad.cpu().numpy(), gr, 1e-5, 1e-6, what="grad")


@pytest.mark.parametrize("sizes,B", [((12, 5, 30), 70), ((100, 100, 100), 33), ((3, 1, 2), 5), ((40, 40, 40), 1)])
def test_three_way_sum_vs_oracle(cuda, sizes, B):
    """f = a + b + c: the plan runs it as two chained convolutions (conv == 3); forward and
    the four-convolution backward against the oracle's 3-way enumeration."""
    S = sg()
    from oracle import algebra as A
    from paper_2410_03348_b200.plan import build_plan

    f = lambda x, y, z: x + y + z  # noqa: E731
    lists = [list(range(n)) for n in sizes]
    assert build_plan(f, None, [tuple(x) for x in lists]).kernel_plan().conv == 3
    rng = np.random.default_rng(sum(sizes))
    xs = [G.rows(rng, B, n) for n in sizes]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    out = S.apply(f, *[S.make_distribution(ctx, lf, lst) for lf, lst in zip(leaves, lists)])
    syms, combos, idx = A.map_shuffle(f, None, lists, S.UNDEFINED)
    assert out.symbols == syms
    ref = A.damp_apply(xs, combos, idx, len(syms))
    got = S.get_probs(out)
    assert_close_rel(got.detach().cpu().numpy(), ref, 1e-5, 1e-7, what="probs")
    w = rng.uniform(-1, 1, size=ref.shape).astype(np.float32)
    torch.autograd.backward(got, torch.as_tensor(w, device=cuda))
    for lf, gr in zip(leaves, A.damp_apply_grad(xs, combos, idx, w.astype(np.float64))):
        assert_close_rel(lf.grad.cpu().numpy(), gr, 1e-5, 1e-6, what="grad")


@pytest.mark.parametrize("na,nb,B", [(1000, 1000, 64), (17, 300, 33), (300, 17, 65), (40, 64, 1), (100, 100, 257)])
def test_long_toeplitz_vs_oracle(cuda, na, nb, B):
    """f = sum over two long lists (both > 16 symbols): the k_lconv direct-convolution path
    (forward and both correlation backwards), against the oracle."""
    S = sg()
    from oracle import algebra as A

    f = lambda x, y: x + y  # noqa: E731
    rng = np.random.default_rng(na * 7 + nb)
    xs = [G.rows(rng, B, na), G.rows(rng, B, nb)]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    out = S.apply(f, S.make_distribution(ctx, leaves[0], range(na)), S.make_distribution(ctx, leaves[1], range(nb)))
    from paper_2410_03348_b200.plan import build_plan

    assert build_plan(f, None, [tuple(range(na)), tuple(range(nb))]).kernel_plan().conv == 2
    syms, combos, idx = A.map_shuffle(f, None, [list(range(na)), list(range(nb))], S.UNDEFINED)
    assert out.symbols == syms
    ref = A.damp_apply(xs, combos, idx, len(syms))
    got = S.get_probs(out)
    assert_close_rel(got.detach().cpu().numpy(), ref, 1e-5, 1e-7, what="probs")
    w = rng.uniform(-1, 1, size=ref.shape)
    torch.autograd.backward(got, torch.as_tensor(w, device=cuda, dtype=torch.float32))
    for lf, gr in zip(leaves, A.damp_apply_grad(xs, combos, idx, w.astype(np.float32).astype(np.float64))):
        assert_close_rel(lf.grad.cpu().numpy(), gr, 1e-5, 1e-6, what="grad")


# ------------------------------------------------------------------ full-size properties
def test_sum15_full_batch_properties(cuda):
    """BASELINE config 2 at B=16384: mass conservation on every sample, and per-sample
    batch independence — 48 sampled rows equal the oracle run on those rows alone."""
    S = sg()
    from oracle import programs as OP
    from paper_2410_03348_b200 import programs as P

    B, n = 16384, 15
    rng = np.random.default_rng(9)
    xs = [G.rows(rng, B, 10) for _ in range(n)]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    out = P.sum_n(ctx, [S.make_distribution(ctx, lf, range(10)) for lf in leaves])
    assert out.symbols == tuple(range(136))
    probs = S.get_probs(out)
    mass = probs.detach().double().sum(dim=1).cpu().numpy()
    np.testing.assert_allclose(mass, 1.0, atol=2e-5)
    w = rng.uniform(-1, 1, size=(B, 136))
    (probs.double() * torch.as_tensor(w, device=cuda)).sum().backward()
    rows = np.sort(rng.choice(B, size=48, replace=False))
    octx = OP.OContext("damp", None, undefined=S.UNDEFINED)
    od = [OP.make_distribution(octx, x[rows], list(range(10))) for x in xs]
    oout = OP.sum_n(od)
    assert_close_rel(probs.detach().cpu().numpy()[rows], OP.get_probs(oout), 1e-5, 1e-7, what="probs")
    ogr = OP.grad_inputs(oout, w[rows])
    for lf, gr in zip(leaves, ogr):
        assert_close_rel(lf.grad.cpu().numpy()[rows], gr, 1e-5, 1e-6, what="grad")


# ------------------------------------------------------------------ fused Toeplitz chains
@pytest.mark.parametrize("n_digits,B", [(3, 100), (15, 4096), (33, 64), (5, 77), (40, 33), (15, 1)])
def test_fused_chain_equals_per_apply_kernels(cuda, n_digits, B):
    """sum_n through the fused chain kernels vs the per-apply Toeplitz kernels: forward
    bit-identical, gradients within fp32 rounding; intermediates can still be read."""
    S = sg()
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.provenance import Damp

    rng = np.random.default_rng(n_digits)
    xs = [G.rows(rng, B, 10) for _ in range(n_digits)]
    w = rng.uniform(-1, 1, size=(B, 9 * n_digits + 1))

    def run(fuse):
        old = Damp.fuse_chains
        Damp.fuse_chains = fuse
        try:
            ctx = S.ProgramContext(S.Damp())
            leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
            out = P.sum_n(ctx, [S.make_distribution(ctx, lf, range(10)) for lf in leaves])
            if fuse and n_digits > 2:
                assert out.tags.pending  # nothing launched until the values are needed
            probs = S.get_probs(out)
            (probs.double() * torch.as_tensor(w, device=cuda)).sum().backward()
            return probs.detach().cpu().numpy(), [lf.grad.cpu().numpy() for lf in leaves]
        finally:
            Damp.fuse_chains = old

    p1, g1 = run(True)
    p0, g0 = run(False)
    np.testing.assert_array_equal(p1, p0)
    for a, b in zip(g1, g0):
        assert_close_rel(a, b, 1e-5, 1e-6)


def test_fused_chain_intermediate_and_reuse(cuda):
    S = sg()
    rng = np.random.default_rng(1)
    B = 70
    xs = [G.rows(rng, B, 10) for _ in range(5)]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    d = [S.make_distribution(ctx, lf, range(10)) for lf in leaves]
    mid = S.apply(lambda a, b: a + b, S.apply(lambda a, b: a + b, d[0], d[1]), d[2])
    end = S.apply(lambda a, b: a + b, S.apply(lambda a, b: a + b, mid, d[3]), d[4])
    branch = S.apply(lambda a, b: a + b, mid, d[0])  # the same pending prefix used twice
    loss = S.get_probs(end).sum() + 2.0 * S.get_probs(mid).sum() + S.get_probs(branch)[:, 3].sum()
    loss.backward()
    from oracle import programs as OP

    octx = OP.OContext("damp", None, undefined=S.UNDEFINED)
    od = [OP.make_distribution(octx, x, list(range(10))) for x in xs]
    f = lambda a, b: a + b  # noqa: E731
    omid = OP.apply(f, OP.apply(f, od[0], od[1]), od[2])
    oend = OP.apply(f, OP.apply(f, omid, od[3]), od[4])
    obr = OP.apply(f, omid, od[0])
    ge = OP.grad_inputs(oend, np.ones((B, len(oend.symbols))))
    gm = OP.grad_inputs(omid, 2.0 * np.ones((B, len(omid.symbols))))
    wb = np.zeros((B, len(obr.symbols)))
    wb[:, 3] = 1.0
    gb = OP.grad_inputs(obr, wb)
    for i, lf in enumerate(leaves):
        assert_close_rel(lf.grad.cpu().numpy(), ge[i] + gm[i] + gb[i], 1e-5, 1e-6, what=f"leaf {i}")


# ------------------------------------------------------------------ whole-step CUDA graph
def test_graphed_step_matches_eager(cuda):
    """GraphedStep (public API) replays Sum-4 + loss + backward on new inputs, both through
    per-input copies and through its pinned arena (one H2D copy); results equal eager."""
    S = sg()
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.graph import GraphedStep
    from paper_2410_03348_b200.learn import loss_nll

    B, nd = 96, 4

    def step(*a):
        xs, t = list(a[:nd]), a[nd]
        ctx = S.ProgramContext(S.Damp(), device=cuda)
        out = P.sum_n(ctx, [S.make_distribution(ctx, x, range(10)) for x in xs])
        loss = loss_nll(S.get_probs(out), t)
        return (loss, *torch.autograd.grad(loss, xs))

    rng = np.random.default_rng(5)

    def batch():
        xs = [torch.tensor(G.rows(rng, B, 10), dtype=torch.float32) for _ in range(nd)]
        return xs, torch.tensor(rng.integers(0, 9 * nd + 1, size=B), dtype=torch.int64)

    xs0, t0 = batch()
    g = GraphedStep(step, [x.to(cuda).requires_grad_(True) for x in xs0] + [t0.to(cuda)])
    for use_arena in (False, True):
        xs, t = batch()
        if use_arena:
            host = g.pinned_inputs()
            for h, x in zip(host, xs + [t]):
                h.copy_(x)
            got = g(*host)
        else:
            got = g(*[x.pin_memory() for x in xs], t.pin_memory())
        got = [o.detach().cpu().clone() for o in got]
        want = step(*[x.to(cuda).requires_grad_(True) for x in xs], t.to(cuda))
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a.numpy(), b.detach().cpu().numpy())


def test_graphed_step_pipelined_slots(cuda):
    """GraphedStep(slots=2).submit: alternating captures with the next step's upload on a
    copy stream give the same losses as eager calls on the same inputs."""
    S = sg()
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.graph import GraphedStep
    from paper_2410_03348_b200.learn import loss_nll

    B, nd = 64, 3

    def step(*a):
        xs, t = list(a[:nd]), a[nd]
        ctx = S.ProgramContext(S.Damp(), device=cuda)
        loss = loss_nll(S.get_probs(P.sum_n(ctx, [S.make_distribution(ctx, x, range(10)) for x in xs])), t)
        return (loss, *torch.autograd.grad(loss, xs))

    rng = np.random.default_rng(9)
    batches = []
    for _ in range(5):
        xs = [torch.tensor(G.rows(rng, B, 10), dtype=torch.float32) for _ in range(nd)]
        batches.append(xs + [torch.tensor(rng.integers(0, 9 * nd + 1, size=B), dtype=torch.int64)])
    g = GraphedStep(step, [x.to(cuda).requires_grad_(x.dtype == torch.float32) for x in batches[0]], slots=2)
    got = []
    for bt in batches:
        slot = g.next_slot()
        for h, x in zip(g.pinned_inputs(slot), bt):
            h.copy_(x)
        out = g.submit()
        got.append(out[0].detach().clone())
    torch.cuda.synchronize()
    for bt, loss in zip(batches, got):
        want = step(*[x.to(cuda).requires_grad_(x.dtype == torch.float32) for x in bt])[0]
        assert float(loss) == float(want)


def test_sum15_step_launches_three_native_kernels(cuda):
    """The whole Sum-15 step (15 distributions, 14 applies, get_probs, loss_nll, backward)
    is three kernels of libsgb200 — fused chain fwd, loss fwd, and the chain bwd with the
    loss gradient generated inside it — counted by the library itself (sg_launch_count),
    with no torch kernels in between."""
    S = sg()
    from paper_2410_03348_b200 import _native as N
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.learn import loss_nll

    rng = np.random.default_rng(3)
    B = 16384  # BASELINE configs[1]; the batch alone fills the GPU, so the loss is one pass
    xs = [torch.tensor(G.rows(rng, B, 10), device=cuda, requires_grad=True) for _ in range(15)]
    t = torch.tensor(rng.integers(0, 136, size=B), device=cuda)
    one = torch.ones((), device=cuda, dtype=torch.float64)

    def step():
        ctx = S.ProgramContext(S.Damp(), device=cuda)
        loss = loss_nll(S.get_probs(P.sum_n(ctx, [S.make_distribution(ctx, x, range(10)) for x in xs])), t)
        return torch.autograd.grad(loss, xs, grad_outputs=one)

    step()  # plans built and uploaded
    torch.cuda.synchronize()
    n0 = N.launch_count()
    step()
    torch.cuda.synchronize()
    assert N.launch_count() - n0 == 3


def test_chain_rowsum_feeds_the_loss(cuda):
    """The fused chain forward's fp64 row sums (a side output) let loss_nll skip its row
    pass; the loss and gradients equal the general path's, and an in-place change of the
    probabilities invalidates the shortcut."""
    S = sg()
    from paper_2410_03348_b200 import ops
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.learn import loss_nll

    rng = np.random.default_rng(4)
    B = 777
    xs = [torch.tensor(G.rows(rng, B, 10), device=cuda, requires_grad=True) for _ in range(6)]
    t = torch.tensor(rng.integers(-1, 46, size=B), device=cuda)

    def run(detour):
        ctx = S.ProgramContext(S.Damp(), device=cuda)
        probs = S.get_probs(P.sum_n(ctx, [S.make_distribution(ctx, x, range(10)) for x in xs]))
        assert ops.known_rowsum(probs.t()) is not None
        if detour:
            probs = probs * 1.0  # a different tensor: the loss computes its own row sums
            assert ops.known_rowsum(probs.t()) is None
        loss = loss_nll(probs, t)
        return float(loss), [g.cpu().numpy() for g in torch.autograd.grad(loss, xs)]

    l_fused, g_fused = run(False)
    l_gen, g_gen = run(True)
    assert l_fused == pytest.approx(l_gen, rel=1e-12)
    for a, b in zip(g_fused, g_gen):
        assert_close_rel(a, b, 1e-9, 1e-12)
    ctx = S.ProgramContext(S.Damp(), device=cuda)
    out = P.sum_n(ctx, [S.make_distribution(ctx, x.detach(), range(10)) for x in xs])
    probs = S.get_probs(out)
    probs.mul_(0.5)
    assert ops.known_rowsum(probs.t()) is None


@pytest.mark.parametrize("fn,size", [("prod", 10), ("lin", 17), ("undef", 12)])
def test_generic_apply_resident_one_pass_backward(cuda, fn, size):
    """Large-batch arity-2 generic applies run on the plan-resident kernel (forward and the
    per-input backward problems, the upstream gradient read in place as the (B, n) block a
    torch loss produces): vs the oracle."""
    S = sg()
    from oracle import algebra as A
    f = {"prod": lambda x, y: x * y, "lin": lambda x, y: (x + 3 * y) % 17,
         "undef": lambda x, y: S.UNDEFINED if (x + y) % 5 == 0 else (x * y) % 23}[fn]
    B = 2 * 64 * 148 + 77  # >= 2 sample groups of 64 per SM: the resident kernel
    rng = np.random.default_rng(size)
    xs = [G.rows(rng, B, size) for _ in range(2)]
    ctx = S.ProgramContext(S.Damp())
    leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
    out = S.apply(f, *[S.make_distribution(ctx, lf, range(size)) for lf in leaves])
    syms, combos, idx = A.map_shuffle(f, None, [list(range(size))] * 2, S.UNDEFINED)
    assert out.symbols == syms
    ref = A.damp_apply(xs, combos, idx, len(syms))
    got = S.get_probs(out)
    assert_close_rel(got.detach().cpu().numpy(), ref, 1e-5, 1e-7, what="probs")
    w = rng.uniform(-1, 1, size=ref.shape).astype(np.float32)
    torch.autograd.backward(got, torch.as_tensor(w, device=cuda))
    for lf, gr in zip(leaves, A.damp_apply_grad(xs, combos, idx, w.astype(np.float64))):
        assert_close_rel(lf.grad.cpu().numpy(), gr, 1e-5, 1e-6, what="grad")


@pytest.mark.parametrize("k", [3, 5])
def test_dtkp_long_group_disj_two_level_merge(cuda, k):
    """Groups long enough to be split (48 records per item) and to need the two-level merge
    (> 8 partial lists): bit-exact against the oracle, with exact key ties included, on
    both the dynamic and the static schedule."""
    S = sg()
    from oracle import algebra as A
    from paper_2410_03348_b200 import ops

    rng = np.random.default_rng(40 + k)
    reg = S.InputRegistry()
    prov = S.DtkpAm(k)
    n, B = 24, 37
    p = np.round(rng.uniform(0.05, 0.95, size=(B, n)), 1).astype(np.float32).astype(np.float64)
    base = prov.input_tags(reg, [("x", i) for i in range(n)], torch.tensor(p))
    obase = A.dtkp_input_tags(0, n, n, B, k)
    perm = list(rng.permutation(n))
    pair = prov.conj(prov.gather(base, list(range(n))), prov.gather(base, perm))
    opair = A.dtkp_conj(A.dtkp_gather(obase, list(range(n))), A.dtkp_gather(obase, perm), p, k)
    pair = prov.concat_syms([pair] * 60)  # 1440 rows
    opair = A.dtkp_concat([opair] * 60)
    groups = [list(rng.integers(0, 1440, size=int(m))) for m in (1000, 433, 385, 49, 1, 700)]
    for dynamic in (True, False):
        ops.DTKP_DYNAMIC = dynamic
        try:
            got = prov.group_disj(pair, groups)
        finally:
            ops.DTKP_DYNAMIC = True
        ref = A.dtkp_group_disj(opair, groups, p, k)
        np.testing.assert_array_equal(got.member, ref[0])
        np.testing.assert_array_equal(got.present, ref[1])


@pytest.mark.parametrize("n_digits,B", [(15, 4096), (6, 77), (3, 1)])
def test_chain_nll_fused_backward_bit_identical(cuda, n_digits, B):
    """loss_nll straight on a fused chain's output runs ONE fused backward
    (sg_chain_bwd_nll, the loss gradient generated in the kernel); it must equal the
    separate sg_nll_bwd + sg_chain_bwd launches bit for bit, loss and gradients, with
    None targets and a second consumer of the same probabilities."""
    S = sg()
    from paper_2410_03348_b200 import ops
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.learn import loss_nll

    rng = np.random.default_rng(n_digits * 31 + B)
    xs = [G.rows(rng, B, 10) for _ in range(n_digits)]
    t = rng.integers(-1, 9 * n_digits + 1, size=B)

    def run(fuse, second):
        old = ops.FUSE_CHAIN_NLL
        ops.FUSE_CHAIN_NLL = fuse
        try:
            ctx = S.ProgramContext(S.Damp())
            leaves = [torch.tensor(x, device=cuda, dtype=torch.float32, requires_grad=True) for x in xs]
            probs = S.get_probs(P.sum_n(ctx, [S.make_distribution(ctx, lf, range(10)) for lf in leaves]))
            loss = loss_nll(probs, torch.as_tensor(t, device=cuda))
            total = loss * 3.0 + (probs[:, :3].double().sum() if second else 0.0)
            total.backward()
            return float(loss), [lf.grad.double().cpu().numpy() for lf in leaves]
        finally:
            ops.FUSE_CHAIN_NLL = old

    l1, g1 = run(True, False)
    l0, g0 = run(False, False)
    assert l1 == l0
    for a, b in zip(g1, g0):
        np.testing.assert_array_equal(a, b)
    # a second consumer of the probabilities: its gradient flows through the chain's own
    # backward and is added by autograd (summed after, not before, the chain backward)
    _, g1 = run(True, True)
    _, g0 = run(False, True)
    for a, b in zip(g1, g0):
        assert_close_rel(a, b, 1e-5, 1e-6)
