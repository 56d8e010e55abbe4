"""Host-side profile of the eager Sum-15 step (Python/API overhead per step)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2410_03348_b200 as sg  # noqa: E402

dev = torch.device("cuda", 0)
x_h, t_h = bench.make_inputs(torch, 16384, dev, 0)
x = [x_h[i].to(dev).requires_grad_(True) for i in range(bench.N_DIGITS)]
t = t_h.to(dev)
step = bench.build_step(torch, sg, dev)
for _ in range(5):
    step(x, t)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    step(x, t)
torch.cuda.synchronize()
print(f"eager step: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms (host+device, 50 steps)")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step(x, t)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
