"""Generic (non-Toeplitz) DAMP apply: fwd and fwd+bwd time and HBM fraction on
HBM-bound shapes (arity 2, |S|=10, f = x*y / (x + 3y) % 17)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import bench_configs as BC  # noqa: E402

import paper_2410_03348_b200 as sg  # noqa: E402

for name, f, size in (("x*y", lambda a, b: a * b, 10), ("(x+3y)%17", lambda a, b: (a + 3 * b) % 17, 10),
                      ("x*y", lambda a, b: a * b, 30)):
    for B in (16384, 65536, 262144):
        rng = np.random.default_rng(0)
        xs = [torch.tensor(BC.rows(rng, B, size), device=BC.DEV, requires_grad=True) for _ in range(2)]
        n_out = len(sg.plan.build_plan(f, None, [tuple(range(size))] * 2).out_symbols)
        w = torch.rand((B, n_out), device=BC.DEV)

        def fwd():
            c = sg.ProgramContext(sg.Damp(), device=BC.DEV)
            return sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, range(size)) for x in xs]))

        ms_f, _ = BC.timed(fwd, 20)
        ms, _ = BC.timed(lambda: torch.autograd.grad(fwd(), xs, grad_outputs=w), 20)
        C = size * size
        fb = 4 * B * (2 * size + n_out) + 4 * C
        bb = 4 * B * (n_out + 4 * size) + 4 * C
        print(json.dumps({"f": name, "S": size, "B": B, "n_out": n_out, "fwd_us": round(ms_f * 1e3, 2),
                          "fwd_frac": round(fb / (ms_f * 1e-3) / 1e9 / BC.HBM, 3),
                          "bwd_us": round((ms - ms_f) * 1e3, 2),
                          "bwd_frac": round(bb / ((ms - ms_f) * 1e-3) / 1e9 / BC.HBM, 3)}))
