"""GPU parity: every golden workload through the public API on the sm_100a kernels.

Symbols (the host plan) and DTKP proof membership + row order are bit-exact; fp32
probabilities and gradients are within 1e-5 relative of the reference (BASELINE.json
north star), with an absolute floor of 1e-6 * max|ref| for gradients (SURVEY §8c:
DAMP backward sums signed weights and can cancel).
"""

import numpy as np
import pytest

import golden_cases as G
from runners import assert_close_rel, load_golden, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.mark.parametrize("name", sorted(G.CASES))
def test_gpu_matches_reference_golden(cuda, name):
    gold = load_golden(name)
    got = run_gpu(name)
    assert got["symbols"] == gold["symbols"]
    assert_close_rel(got["probs"], gold["probs"], RTOL, floor_frac=1e-7, what=f"{name} probs")
    for i in range(int(gold["n_inputs"])):
        assert_close_rel(got["grads"][i], gold[f"grad{i}"], RTOL, floor_frac=1e-6, what=f"{name} grad{i}")
    if "member" in gold:
        np.testing.assert_array_equal(got["member"], gold["member"])
        np.testing.assert_array_equal(got["present"], gold["present"])


@pytest.mark.parametrize("name", ["damp_sum15", "dtkp_hwf5", "dtkp_path_k5", "damp_mod_cond_a2", "max_sum4",
                                  "max_mod_cond_a2", "max_path", "max_bcast_reuse"])
def test_gpu_matches_oracle_fresh_inputs(cuda, name):
    """Same programs on new seeded inputs: CUDA path vs the CPU oracle."""
    prov, k, prog, syms_fn, make, seed = G.CASES[name]
    inputs = make(np.random.default_rng(777 + seed))
    ref = run_oracle(name, inputs)
    got = run_gpu(name, inputs)
    assert got["symbols"] == ref["symbols"]
    assert_close_rel(got["probs"], ref["probs"], RTOL, floor_frac=1e-7, what="probs")
    for g, r in zip(got["grads"], ref["grads"]):
        assert_close_rel(g, r, RTOL, floor_frac=1e-6, what="grad")
    if "member" in ref:
        np.testing.assert_array_equal(got["member"], ref["member"])
        np.testing.assert_array_equal(got["present"], ref["present"])


@pytest.mark.parametrize("name", ["dtkp_hwf5", "dtkp_path_k5"])
def test_dtkp_dynamic_and_static_schedules_agree(cuda, name):
    """The apply's dynamic item schedule (per-column work counters) and the static block
    partition produce the same proofs bit for bit; the counters are left zeroed."""
    import torch

    from paper_2410_03348_b200 import ops

    prov, k, prog, syms_fn, make, seed = G.CASES[name]
    inputs = make(np.random.default_rng(4242 + seed))
    try:
        ops.DTKP_DYNAMIC = False
        static = run_gpu(name, inputs)
    finally:
        ops.DTKP_DYNAMIC = True
    dynamic = run_gpu(name, inputs)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dynamic["member"], static["member"])
    np.testing.assert_array_equal(dynamic["present"], static["present"])
    np.testing.assert_array_equal(dynamic["probs"], static["probs"])
    assert ops._SCHED and all(int(t.abs().sum()) == 0 for t in ops._SCHED.values())
