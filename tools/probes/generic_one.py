"""One generic apply (f = x*y, |S|=10, B=262144) forward + backward, for ncu launch lists."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import bench_configs as BC  # noqa: E402

import paper_2410_03348_b200 as sg  # noqa: E402

B, size = 262144, 10
f = lambda a, b: a * b  # noqa: E731
rng = np.random.default_rng(0)
xs = [torch.tensor(BC.rows(rng, B, size), device=BC.DEV, requires_grad=True) for _ in range(2)]
n_out = len(sg.plan.build_plan(f, None, [tuple(range(size))] * 2).out_symbols)
w = torch.rand((B, n_out), device=BC.DEV)
for _ in range(3):
    c = sg.ProgramContext(sg.Damp(), device=BC.DEV)
    p = sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, range(size)) for x in xs]))
    torch.autograd.grad(p, xs, grad_outputs=w)
torch.cuda.synchronize()
