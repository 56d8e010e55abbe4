"""Eager runs of the DTKP CLUTRR closure with a loss + backward and the golden cases, for
compute-sanitizer memcheck with PYTORCH_NO_CUDA_MEMORY_CACHING=1 (every tensor its own
allocation, so an out-of-bounds write into a neighbouring tensor is visible)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_cases as G  # noqa: E402
from runners import load_golden, run_gpu  # noqa: E402
import paper_2410_03348_b200 as sg  # noqa: E402
from paper_2410_03348_b200.programs import _chain_link, kinship_compose  # noqa: E402

cuda = torch.device("cuda", 0)
names = sys.argv[1:] or sorted(G.CASES)
for n in names:
    run_gpu(n)
gold = load_golden("dtkp_clutrr_e5_r20_k5")
x = torch.tensor(gold["in0"], device=cuda, dtype=torch.float32, requires_grad=True)
wt = torch.as_tensor(gold["w"], device=cuda)
ctx = sg.ProgramContext(sg.DtkpAm(5), device=cuda)
out = sg.closure(kinship_compose, _chain_link, sg.make_distribution(ctx, x, G.clutrr_facts(5)))
loss = (sg.get_probs(out).double() * wt).sum()
loss.backward()
torch.cuda.synchronize()
print("oob cases done", float(loss.detach()))
