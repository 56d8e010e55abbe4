"""Device-resident fixpoint driver (programs.py:177-196).

CPU: the host-only iteration count of a closure equals the reference loop's.  GPU: a
CUDA-graph-captured CLUTRR closure (5 entities x 20 relations, DTKP k=5 — BASELINE
configs[3]) replays bit-identically to the eager closure and matches the reference's
own outputs (tests/golden/dtkp_clutrr_e5_r20_k5.npz) and the oracle on fresh inputs.
"""

import numpy as np
import pytest

import golden_cases as G
from runners import assert_close_rel, load_golden, run_oracle


def _reference_loop_iterations(f, cond, facts, undefined):
    """programs.py:177-196 on symbols alone (oracle map/shuffle)."""
    from oracle.algebra import map_shuffle

    derived = tuple(facts)
    it = 0
    while True:
        new, _, _ = map_shuffle(f, cond, [derived, tuple(facts)], undefined)
        merged = derived + tuple(s for s in new if s not in set(derived))
        it += 1
        if set(merged) == set(derived):
            return it
        derived = merged


@pytest.mark.parametrize("n_entities", [3, 4, 5])
def test_closure_iterations_match_reference_loop(n_entities):
    from paper_2410_03348_b200 import UNDEFINED
    from paper_2410_03348_b200.fixpoint import closure_iterations
    from paper_2410_03348_b200.programs import _chain_link, kinship_compose

    facts = G.clutrr_facts(n_entities)
    assert closure_iterations(kinship_compose, _chain_link, facts) == _reference_loop_iterations(
        kinship_compose, _chain_link, facts, UNDEFINED)


def _graphed(cuda, x, w=None):
    import torch

    import paper_2410_03348_b200 as sg
    from paper_2410_03348_b200.programs import _chain_link, kinship_compose

    facts = G.clutrr_facts(5)
    loss_fn = None
    if w is not None:
        wt = torch.as_tensor(w, device=cuda)

        def loss_fn(p):
            return (p.double() * wt).sum()

    gc = sg.GraphedClosure(kinship_compose, _chain_link, facts, lambda: sg.DtkpAm(5),
                           torch.tensor(x, device=cuda, dtype=torch.float32), loss_fn=loss_fn)
    return gc


@pytest.mark.gpu
def test_graphed_clutrr_closure_matches_eager_and_reference(cuda):
    import torch

    from runners import run_gpu

    name = "dtkp_clutrr_e5_r20_k5"
    gold = load_golden(name)
    x = gold["in0"]
    eager = run_gpu(name, [x])
    gc = _graphed(cuda, x, w=gold["w"])
    loss, g = gc(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    assert [repr(s) for s in gc.symbols] == gold["symbols"]
    np.testing.assert_array_equal(g.double().cpu().numpy(), eager["grads"][0])
    assert_close_rel(g.double().cpu().numpy(), gold["grad0"], 1e-5, floor_frac=1e-6, what="graphed grad")
    assert float(loss.detach()) == pytest.approx(float((gold["probs"] * gold["w"]).sum()), rel=1e-5)
    gp = _graphed(cuda, x)
    probs = gp(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(probs.double().cpu().numpy(), eager["probs"])


@pytest.mark.gpu
def test_graphed_closure_replays_on_new_inputs(cuda):
    import torch

    from runners import run_gpu

    name = "dtkp_clutrr_e5_r20_k5"
    rng = np.random.default_rng(99)
    x0 = rng.uniform(0.05, 0.95, size=(6, 80)).astype(np.float32).astype(np.float64)
    gp = _graphed(cuda, x0)
    for seed in (1, 2, 3):
        x = np.random.default_rng(seed).uniform(0.05, 0.95, size=(6, 80)).astype(np.float32).astype(np.float64)
        probs = gp(torch.tensor(x, device=cuda, dtype=torch.float32)).double().cpu().numpy()
        eager = run_gpu(name, [x])
        ref = run_oracle(name, [x])
        np.testing.assert_array_equal(probs, eager["probs"])
        assert_close_rel(probs, ref["probs"], 1e-5, floor_frac=1e-7, what="graphed vs oracle")
        np.testing.assert_array_equal(eager["member"], ref["member"])
