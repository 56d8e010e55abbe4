"""CPU: pin the oracle restatement against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

import golden_cases as G
from runners import load_golden, run_oracle


@pytest.mark.parametrize("name", sorted(G.CASES))
def test_oracle_matches_reference_golden(name):
    gold = load_golden(name)
    got = run_oracle(name)
    assert got["symbols"] == gold["symbols"], "output symbol order differs from the reference"
    np.testing.assert_allclose(got["probs"], gold["probs"], rtol=1e-9, atol=1e-12)
    for i in range(int(gold["n_inputs"])):
        np.testing.assert_allclose(got["grads"][i], gold[f"grad{i}"], rtol=1e-8, atol=1e-10)
    if "member" in gold:
        np.testing.assert_array_equal(got["member"], gold["member"])
        np.testing.assert_array_equal(got["present"], gold["present"])


def test_oracle_dedup_topk_matches_compiled_reference_fuzz():
    from oracle.algebra import dedup_topk

    z = np.load(load_golden.__globals__["GOLDEN"] / "dedup_topk_fuzz.npz")
    for c in range(int(z["n_cases"])):
        om, op = dedup_topk(z[f"c{c}_member"], z[f"c{c}_present"], z[f"c{c}_p"], int(z[f"c{c}_k"]))
        np.testing.assert_array_equal(om, z[f"c{c}_om"])
        np.testing.assert_array_equal(op, z[f"c{c}_op"])


def _ref_dtkpcore():
    try:
        import importlib.util
        from pathlib import Path

        so = sorted((Path(__file__).resolve().parents[1] / "oracle" / "_ref").glob("_dtkpcore*.so"))
        if not so:
            return None
        spec = importlib.util.spec_from_file_location("_dtkpcore", so[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    except Exception:  # noqa: BLE001 - optional checker
        return None


def test_oracle_c_restatement_matches_oracle_ref_build():
    """The C restatement vs the reference's _dtkpcore compiled from its source (oracle/_ref)."""
    ref = _ref_dtkpcore()
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    from oracle.algebra import dedup_topk

    rng = np.random.default_rng(7)
    for _ in range(200):
        M, R, I, k = int(rng.integers(1, 5)), int(rng.integers(1, 14)), int(rng.integers(0, 140)), int(rng.integers(1, 8))
        member = (rng.uniform(size=(M, R, I)) < 0.35).astype(np.uint8)
        present = (rng.uniform(size=(M, R)) < 0.8).astype(np.uint8)
        p = np.round(rng.uniform(0.0, 1.0, size=(M, I)), 1)
        om, op = dedup_topk(member, present, p, k)
        rm, rp = ref.dedup_topk(member, present, p, k)
        np.testing.assert_array_equal(om, rm)
        np.testing.assert_array_equal(op, rp)


def test_dedup_topk_semantics_examples():
    """The reference's hand-written dedup_topk cases (test_kernels.py:31-84) on the oracle."""
    from oracle.algebra import dedup_topk

    m, pr = dedup_topk(np.array([[[1, 0], [0, 1], [0, 0]]], np.uint8), np.array([[1, 1, 1]], np.uint8),
                       np.array([[0.2, 0.8]]), 3)
    np.testing.assert_array_equal(m[0], [[0, 0], [0, 1], [1, 0]])
    m, pr = dedup_topk(np.array([[[1, 0], [1, 0], [0, 1]]], np.uint8), np.array([[1, 1, 1]], np.uint8),
                       np.array([[0.5, 0.5]]), 3)
    assert pr[0].tolist() == [1, 1, 0]
    m, _ = dedup_topk(np.array([[[0, 1], [1, 0]]], np.uint8), np.array([[1, 1]], np.uint8), np.array([[0.5, 0.5]]), 1)
    np.testing.assert_array_equal(m[0, 0], [0, 1])
    m, pr = dedup_topk(np.zeros((1, 3, 0), np.uint8), np.ones((1, 3), np.uint8), np.zeros((1, 0)), 2)
    assert pr[0].tolist() == [1, 0]
