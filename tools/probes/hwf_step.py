"""One warmed-up eager HWF-7 DTKP step (fwd + loss + bwd), for ncu launch lists:
    ncu --metrics gpu__time_duration.sum ... python tools/probes/hwf_step.py"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2410_03348_b200 as sg  # noqa: E402
from paper_2410_03348_b200 import programs as P  # noqa: E402
from paper_2410_03348_b200.learn import loss_nll  # noqa: E402
from bench_configs import rows  # noqa: E402

DEV = torch.device("cuda", 0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(1)
xs = [torch.tensor(rows(rng, B, 14), device=DEV, requires_grad=True) for _ in range(7)]


def step():
    c = sg.ProgramContext(sg.DtkpAm(3), device=DEV)
    o = P.hwf(c, [sg.make_distribution(c, x, P.TOKEN_ALPHABET) for x in xs], 7)
    t = torch.zeros(B, dtype=torch.int64, device=DEV)
    loss = loss_nll(sg.get_probs(o), t)
    return torch.autograd.grad(loss, xs)


for _ in range(2):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
