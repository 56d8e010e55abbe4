"""The fused conj -> group_disj DTKP launch (sg_dtkp_apply_desc.inner_*): an arity-1 apply
over a pending binary apply — HWF's eval over its last concat step — must equal the two
separate launches bit for bit (membership, row order, probabilities, gradients), and both
must equal the reference (tests/golden)."""

import numpy as np
import pytest

import golden_cases as G
from runners import load_golden, run_gpu

pytestmark = pytest.mark.gpu


def _run(name, inputs, fuse):
    import paper_2410_03348_b200 as sg

    old = sg.DtkpAm.fuse_conj_group  # default off; both paths must agree
    sg.DtkpAm.fuse_conj_group = fuse
    try:
        return run_gpu(name, inputs)
    finally:
        sg.DtkpAm.fuse_conj_group = old


@pytest.mark.parametrize("name", ["dtkp_hwf3", "dtkp_hwf5", "dtkp_hwf7", "dtkp_hwf3_k1", "dtkp_hwf3_k7"])
def test_fused_equals_unfused_and_reference(cuda, name):
    gold = load_golden(name)
    inputs = [gold[f"in{i}"] for i in range(int(gold["n_inputs"]))]
    fused = _run(name, inputs, True)
    plain = _run(name, inputs, False)
    np.testing.assert_array_equal(fused["member"], plain["member"])
    np.testing.assert_array_equal(fused["present"], plain["present"])
    np.testing.assert_array_equal(fused["probs"], plain["probs"])
    for a, b in zip(fused["grads"], plain["grads"]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(fused["member"], gold["member"])
    np.testing.assert_array_equal(fused["present"], gold["present"])


def test_fused_launch_is_used_for_hwf(cuda):
    """The eval apply consumes the pending concat apply: one fewer launch, no materialised
    208767-symbol tag at HWF-7 (here HWF-5: 10045 intermediate symbols)."""
    from paper_2410_03348_b200 import _native as N

    prov, k, prog, syms_fn, make, seed = G.CASES["dtkp_hwf5"]
    inputs = make(np.random.default_rng(5))
    _run("dtkp_hwf5", inputs, True)  # warm plans
    c0 = N.launch_count()
    _run("dtkp_hwf5", inputs, True)
    fused = N.launch_count() - c0
    c0 = N.launch_count()
    _run("dtkp_hwf5", inputs, False)
    plain = N.launch_count() - c0
    assert fused < plain


def test_pending_conj_materialises_for_other_consumers(cuda):
    """A pending binary apply read by anything but an arity-1 apply (get_probs, filter,
    union, a second binary apply) is materialised with the plain kernel."""
    import torch

    import paper_2410_03348_b200 as sg

    old = sg.DtkpAm.fuse_conj_group
    sg.DtkpAm.fuse_conj_group = True
    try:
        _pending_case(cuda, sg)
    finally:
        sg.DtkpAm.fuse_conj_group = old


def _pending_case(cuda, sg):
    import torch

    ctx = sg.ProgramContext(sg.DtkpAm(3), device=cuda)
    rng = np.random.default_rng(3)
    a = sg.make_distribution(ctx, torch.tensor(G.rows(rng, 4, 5), device=cuda), range(5))
    b = sg.make_distribution(ctx, torch.tensor(G.rows(rng, 4, 4), device=cuda), range(4))
    s = sg.apply(lambda x, y: x + y, a, b)
    assert s.tags.pending is not None
    f = s.filter(lambda v: v % 2 == 0)
    assert s.tags.pending is None and f.tags.pending is None
    p = sg.get_probs(sg.union(f, s))
    assert torch.isfinite(p).all()


@pytest.mark.parametrize("name", ["dtkp_hwf7", "dtkp_clutrr_e5_r20_k5", "dtkp_path_k5", "dtkp_sum4_k5"])
def test_ranked_early_exit_and_packing_are_exact(cuda, name):
    """The streaming kernels' ranked-rows early exit (sg_dtkp_apply_desc.rows_ranked) and
    the packed work items change no retained proof and no row order."""
    from paper_2410_03348_b200 import ops, plan

    gold = load_golden(name)
    inputs = [gold[f"in{i}"] for i in range(int(gold["n_inputs"]))]
    fast = run_gpu(name, inputs)
    old = (ops.DTKP_RANKED, plan.DTKP_PACK)
    try:
        ops.DTKP_RANKED, plan.DTKP_PACK = False, False
        plain = run_gpu(name, inputs)
    finally:
        ops.DTKP_RANKED, plan.DTKP_PACK = old
    np.testing.assert_array_equal(fast["member"], plain["member"])
    np.testing.assert_array_equal(fast["present"], plain["present"])
    np.testing.assert_array_equal(fast["probs"], plain["probs"])
    np.testing.assert_array_equal(fast["member"], gold["member"])
