"""One warmed-up Sum-15 step under the max/DAMP variant (fused max chain + loss), fwd+bwd,
for ncu launch lists (no NVTX filter: the backward runs on autograd's device thread):
    ncu ... --launch-skip N python tools/probes/max15_step.py [B]"""
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

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
DEV = torch.device("cuda", 0)
rng = np.random.default_rng(0)
xs = [torch.tensor(rows(rng, B, 10), device=DEV, requires_grad=True) for _ in range(15)]
t = torch.tensor(rng.integers(0, 136, size=B), device=DEV)


def step():
    c = sg.ProgramContext(sg.DampMax(), device=DEV)
    o = P.sum_n(c, [sg.make_distribution(c, x, list(range(10))) for x in xs])
    return torch.autograd.grad(loss_nll(sg.get_probs(o), t), xs)


for _ in range(4):
    step()
torch.cuda.synchronize()
