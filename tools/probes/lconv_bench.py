"""fwd / fwd+bwd time of one long-Toeplitz apply (f = sum, two lists of |S| symbols)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import bench_configs as BC  # noqa: E402

import paper_2410_03348_b200 as sg  # noqa: E402

for size, B in ((1000, 16384), (100, 65536)):
    rng = np.random.default_rng(0)
    xs = [torch.tensor(BC.rows(rng, B, size), device=BC.DEV, requires_grad=True) for _ in range(2)]
    w = torch.rand((B, 2 * size - 1), device=BC.DEV)

    def fwd():
        c = sg.ProgramContext(sg.Damp(), device=BC.DEV)
        return sg.get_probs(sg.apply(lambda a, b: a + b, *[sg.make_distribution(c, x, range(size)) for x in xs]))

    ms_f, _ = BC.timed(fwd, 10)
    ms, _ = BC.timed(lambda: torch.autograd.grad(fwd(), xs, grad_outputs=w), 10)
    fl = B * size * size
    print(f"|S|={size} B={B}: fwd {ms_f:.3f} ms ({fl / ms_f / 1e9:.0f} GFMA/s)  fwd+bwd {ms:.3f} ms "
          f"({3 * fl / ms / 1e9:.0f} GFMA/s)")
