"""loss_nll (learn.py:92-119), the step right after the path.

CPU: the oracle restatement and the product's target contract against the reference's
own outputs (tests/golden/loss_nll.npz, tools/make_golden.py) and its error cases
(test_learn.py:66-106).  GPU: the fused sg_nll_fwd/bwd kernels against the same fixture.
"""

import numpy as np
import pytest
import torch

from runners import GOLDEN

from paper_2410_03348_b200.learn import loss_nll


def _cases():
    z = np.load(GOLDEN / "loss_nll.npz")
    return [(z[f"c{c}_probs"], z[f"c{c}_targets"], float(z[f"c{c}_loss"]), z[f"c{c}_grad"])
            for c in range(int(z["n_cases"]))]


def test_oracle_loss_matches_reference_fixture():
    from oracle.algebra import loss_nll as oracle_loss

    for probs, targets, loss, grad in _cases():
        got, g = oracle_loss(probs, targets)
        assert got == pytest.approx(loss, rel=1e-12)
        np.testing.assert_allclose(g, grad, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("bad", [[0, 1], [0, 1, 2, 0]])
def test_target_count_mismatch_raises_value_error(bad):
    with pytest.raises(ValueError):
        loss_nll(torch.full((3, 4), 0.25), bad)
    with pytest.raises(ValueError):
        loss_nll(torch.full((3, 4), 0.25), torch.tensor(bad))


@pytest.mark.parametrize("bad", [[0, 4, 1], [0, -1, 1], [7, 0, 0]])
def test_target_out_of_range_raises_index_error(bad):
    """learn.py:108-109 (test_learn.py:99-101); -1 is the device encoding of None, so the
    list form rejects it exactly like the reference."""
    with pytest.raises(IndexError):
        loss_nll(torch.full((3, 4), 0.25), bad)


def test_tensor_targets_out_of_range_raise_index_error():
    with pytest.raises(IndexError):
        loss_nll(torch.full((3, 4), 0.25), torch.tensor([0, 4, 1]))
    with pytest.raises(IndexError):
        loss_nll(torch.full((3, 4), 0.25), torch.tensor([0, -2, 1]))


@pytest.mark.gpu
def test_fused_loss_matches_reference_fixture(cuda):
    for probs, targets, loss, grad in _cases():
        x = torch.tensor(probs, device=cuda, dtype=torch.float32, requires_grad=True)
        tl = [None if t < 0 else int(t) for t in targets]
        for tgt in (tl, torch.tensor(targets, device=cuda)):
            x.grad = None
            out = loss_nll(x, tgt)
            out.backward()
            assert float(out) == pytest.approx(loss, rel=1e-9)
            g = x.grad.double().cpu().numpy()
            # the kernel computes in fp64 and stores fp32 gradients
            np.testing.assert_allclose(g, grad, rtol=1e-5, atol=1e-6 * np.abs(grad).max())


@pytest.mark.gpu
def test_device_targets_checked_and_kernel_guard(cuda):
    x = torch.full((4, 5), 0.2, device=cuda, requires_grad=True)
    with pytest.raises(IndexError):
        loss_nll(x, torch.tensor([0, 5, 1, 1], device=cuda))
    # past the host check (as inside a captured graph) the kernel never reads out of
    # bounds: the bad sample turns the loss and its gradient row NaN
    from paper_2410_03348_b200 import ops

    t = torch.tensor([0, 5, 1, -1], device=cuda)
    out = ops.NllLoss.apply(x.t(), t)
    out.backward()
    torch.cuda.synchronize()
    assert np.isnan(float(out))
    g = x.grad.cpu().numpy()
    assert np.isnan(g[1]).all() and np.isfinite(g[[0, 2, 3]]).all()
