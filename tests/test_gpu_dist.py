"""Two ranks on ONE B200 over gloo (this pool has one GPU per box): the data-parallel train
step of the bench — CUDA symbolic path (fused Sum-N chain + fused loss) per rank shard,
perception gradients averaged by ONE all_reduce of the flat buffer (dp.FlatGradReducer) —
reproduces the single-process global-batch gradient.  The NCCL launch of bench.py runs the
same code with one rank per GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B_GLOBAL, N_DIGITS = 256, 4


def _data():
    rng = np.random.default_rng(3)
    labels = rng.integers(0, 10, size=(N_DIGITS, B_GLOBAL))
    centers = rng.normal(size=(10, 784))
    feats = (centers[labels] * (5.0 / 28) + rng.normal(size=(N_DIGITS, B_GLOBAL, 784))).astype(np.float32)
    return feats, labels.sum(axis=0)


def _grads(feats, targets, dev, world=1):
    import paper_2410_03348_b200 as sg
    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.dp import FlatGradReducer
    from paper_2410_03348_b200.learn import Mlp, loss_nll

    model = Mlp(seed=0).to(dev)
    red = FlatGradReducer(model.parameters())
    red.zero_()
    x = torch.tensor(feats, device=dev)
    probs = model(x.view(-1, 784)).view(N_DIGITS, -1, 10)
    ctx = sg.ProgramContext(sg.Damp(), device=dev)
    out = P.sum_n(ctx, [sg.make_distribution(ctx, probs[i], range(10)) for i in range(N_DIGITS)])
    loss = loss_nll(sg.get_probs(out), torch.tensor(targets, device=dev))
    loss.backward()
    red.all_reduce_()
    return [p.grad.detach().double().cpu().numpy() for p in model.parameters()]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_03348_b200.dp import shard_range

        feats, targets = _data()
        lo, hi = shard_range(B_GLOBAL, rank, world)
        q.put((rank, _grads(feats[:, lo:hi], targets[lo:hi], torch.device("cuda", 0), world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_on_one_gpu_match_single_process(cuda):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    feats, targets = _data()
    ref = _grads(feats, targets, cuda)
    for a, b, r in zip(res[0], res[1], ref):
        np.testing.assert_array_equal(a, b)  # one all_reduce -> identical on both ranks
        np.testing.assert_allclose(a, r, rtol=2e-4, atol=1e-6 * np.abs(r).max())
