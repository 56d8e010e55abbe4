"""Which torch kernels does one eager Sum-15 step launch besides ours (with stacks)?"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2410_03348_b200 as sg  # noqa: E402

dev = torch.device("cuda", 0)
x_h, t_h = bench.make_inputs(torch, 1024, dev, 0)
x = [x_h[i].to(dev).requires_grad_(True) for i in range(bench.N_DIGITS)]
t = t_h.to(dev)
step = bench.build_step(torch, sg, dev)
for _ in range(3):
    step(x, t)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    step(x, t)
    torch.cuda.synchronize()
for ev in prof.events():
    if ev.device_type.name == "CUDA" or "Fill" in ev.name or "fill" in ev.name:
        print(ev.name[:80])
for ev in prof.events():
    if ev.name in ("aten::fill_", "aten::ones_like", "aten::zeros", "aten::zero_", "aten::ones", "aten::full"):
        print("==", ev.name, [s for s in ev.stack if "paper_2410" in s or "bench" in s or "autograd" in s][:6])
