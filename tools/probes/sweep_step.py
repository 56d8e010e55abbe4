"""One warmed-up sweep step (apply f=sum, fwd + bwd with upstream weights), inside an NVTX
range "step", for ncu launch lists:
    ncu --nvtx --nvtx-include "step/" ... python tools/probes/sweep_step.py ARITY SIZE B [damp|max]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2410_03348_b200 as sg  # noqa: E402
from bench_configs import rows  # noqa: E402

arity, size, B = (int(v) for v in sys.argv[1:4])
prov = sg.Damp if (len(sys.argv) < 5 or sys.argv[4] == "damp") else sg.DampMax
DEV = torch.device("cuda", 0)
rng = np.random.default_rng(0)
xs = [torch.tensor(rows(rng, B, size), device=DEV, requires_grad=True) for _ in range(arity)]
f = (lambda a, b: a + b) if arity == 2 else (lambda a, b, c: a + b + c)
n_out = arity * (size - 1) + 1
w = torch.tensor(rng.uniform(-1, 1, size=(B, n_out)).astype(np.float32), device=DEV)


def step():
    c = sg.ProgramContext(prov(), device=DEV)
    p = sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, list(range(size))) for x in xs]))
    return torch.autograd.grad(p, xs, grad_outputs=w)


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
