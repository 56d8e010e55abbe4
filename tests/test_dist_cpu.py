"""CPU, world_size 2 over gloo: the data-parallel host logic of the N > 1 path.

* every rank builds bit-identical symbol plans (no plan broadcast needed);
* batch sharding covers the global batch exactly once;
* DDP over the per-rank shards reproduces the single-process global-batch gradient of the
  perception parameters (loss_nll is a batch mean).  The symbolic layer runs on the CPU
  oracle here (test infrastructure; the product path is CUDA-only).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _symbolic_loss_and_grad(probs_np, targets, n_digits):
    """Oracle Sum-N forward + loss_nll gradient w.r.t. the digit probabilities."""
    from oracle import programs as OP
    from paper_2410_03348_b200.plan import UNDEFINED

    ctx = OP.OContext("damp", None, undefined=UNDEFINED)
    dists = [OP.make_distribution(ctx, probs_np[i], list(range(10))) for i in range(n_digits)]
    out = OP.sum_n(dists)
    p = OP.get_probs(out)
    B = p.shape[0]
    s = p.sum(axis=1) + 1e-8
    pt = p[np.arange(B), targets]
    picked = np.maximum(np.maximum(pt / s, 1e-12), 1e-12)
    loss = -np.log(picked).mean()
    g = np.zeros_like(p)
    coef = -(1.0 / B) / picked
    g += (coef * (-pt / s**2))[:, None]
    g[np.arange(B), targets] += coef / s
    return loss, OP.grad_inputs(out, g)


class _SymbolicLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, probs, targets):
        loss, grads = _symbolic_loss_and_grad(probs.detach().double().numpy(), targets.numpy(), probs.shape[0])
        ctx.grads = torch.tensor(np.stack(grads), dtype=probs.dtype)
        return torch.tensor(loss, dtype=probs.dtype)

    @staticmethod
    def backward(ctx, g):
        return ctx.grads * g, None


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(16, 10), torch.nn.Softmax(dim=-1)).double()


def _data(global_batch=12, n_digits=3):
    rng = np.random.default_rng(0)
    x = torch.tensor(rng.normal(size=(n_digits, global_batch, 16)))
    t = torch.tensor(rng.integers(0, 9 * n_digits + 1, size=global_batch))
    return x, t


def _grads_single(global_batch=12, n_digits=3):
    model = _model()
    x, t = _data(global_batch, n_digits)
    loss = _SymbolicLoss.apply(model(x), t)
    loss.backward()
    return [p.grad.clone() for p in model.parameters()]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_03348_b200.dp import assert_plans_replicated, max_over_ranks, shard_range
        from paper_2410_03348_b200.plan import build_plan
        from paper_2410_03348_b200.programs import _add

        digits = tuple(range(10))
        plans = [build_plan(_add, None, [digits if i == 1 else tuple(range(9 * (i - 1) + 10)), digits])
                 for i in range(1, 6)]
        fps = assert_plans_replicated(plans)
        x, t = _data()
        lo, hi = shard_range(t.numel(), rank, world)
        model = torch.nn.parallel.DistributedDataParallel(_model())
        loss = _SymbolicLoss.apply(model(x[:, lo:hi]), t[lo:hi])
        loss.backward()
        grads = [p.grad.clone() for p in model.parameters()]
        worst = max_over_ranks(float(rank + 1))
        # the bench's train step: grads as views of one flat buffer, ONE all_reduce
        from paper_2410_03348_b200.dp import FlatGradReducer

        m2 = _model().float()
        red = FlatGradReducer(m2.parameters())
        red.zero_()
        loss2 = _SymbolicLoss.apply(m2(x[:, lo:hi].float()), t[lo:hi])
        loss2.backward()
        red.all_reduce_()
        flat = [p.grad.detach().double().clone().numpy() for p in m2.parameters()]
        q.put((rank, fps, (lo, hi), [g.numpy() for g in grads], worst, flat))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2410_03348_b200.dp import shard_range

    for B in (1, 7, 16, 16384, 16385):
        for world in (1, 2, 3, 8):
            spans = [shard_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_ddp_gloo_world2_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    (_, fp0, span0, g0, w0, f0), (_, fp1, span1, g1, w1, f1) = results
    assert fp0 == fp1
    assert span0 == (0, 6) and span1 == (6, 12)
    assert w0 == w1 == 2.0
    ref = _grads_single()
    for a, b, r in zip(g0, g1, ref):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)  # DDP leaves identical grads
        np.testing.assert_allclose(a, r.numpy(), rtol=1e-9, atol=1e-12)  # == global-batch gradient
    for a, b, r in zip(f0, f1, ref):  # flat-buffer all_reduce == DDP == global batch (fp32)
        np.testing.assert_array_equal(a, b)
        np.testing.assert_allclose(a, r.numpy(), rtol=2e-5, atol=1e-6)
