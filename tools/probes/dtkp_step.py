"""One warmed-up eager DTKP step (fwd + loss + bwd) of HWF-7 (B=64) or the CLUTRR-style
closure (B=4096), inside an NVTX range "step", for ncu launch lists:
    ncu --nvtx --nvtx-include "step/" ... python tools/probes/dtkp_step.py hwf|clutrr"""
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
MODE = sys.argv[1] if len(sys.argv) > 1 else "hwf"
rng = np.random.default_rng(1)
if MODE == "hwf":
    B = 64
    xs = [torch.tensor(rows(rng, B, 14), device=DEV, requires_grad=True) for _ in range(7)]

    def program(c):
        return P.hwf(c, [sg.make_distribution(c, x, P.TOKEN_ALPHABET) for x in xs], 7), 3
else:
    sys.path.insert(0, str(ROOT / "tests"))
    from golden_cases import clutrr_facts  # noqa: E402

    B = 4096
    facts = clutrr_facts(5)
    xs = [torch.tensor(rng.uniform(0.05, 0.95, size=(B, len(facts))).astype(np.float32), device=DEV,
                       requires_grad=True)]

    def program(c):
        return P.clutrr_closure(c, sg.make_distribution(c, xs[0], facts)), 5


def step():
    c = sg.ProgramContext(sg.DtkpAm(3 if MODE == "hwf" else 5), device=DEV)
    o, _ = program(c)
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
