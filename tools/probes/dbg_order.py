"""Diagnostic: does running golden cases first change the graph-captured CLUTRR closure?"""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_cases as G
from runners import load_golden, run_gpu
import paper_2410_03348_b200 as sg
from paper_2410_03348_b200.programs import _chain_link, kinship_compose
cuda = torch.device("cuda", 0)
pre = sys.argv[1:]  # golden case names to run first
for name in pre:
    if name in ("ALL", "ALLC", "DAMP", "MAX"):
        for n in sorted(G.CASES):
            kind = G.CASES[n][0]
            if name == "ALLC" or (name == "ALL" and kind == "dtkp") or (name == "DAMP" and kind == "damp") \
                    or (name == "MAX" and kind == "max"):
                run_gpu(n)
    else:
        run_gpu(name)
gold = load_golden("dtkp_clutrr_e5_r20_k5"); x = gold["in0"]
eager = run_gpu("dtkp_clutrr_e5_r20_k5", [x])
facts = G.clutrr_facts(5)
wt = torch.as_tensor(gold["w"], device=cuda)
gc = sg.GraphedClosure(kinship_compose, _chain_link, facts, lambda: sg.DtkpAm(5),
                       torch.tensor(x, device=cuda, dtype=torch.float32), loss_fn=lambda p: (p.double() * wt).sum())
loss, g = gc(torch.tensor(x, device=cuda, dtype=torch.float32)); torch.cuda.synchronize()
print(pre, "graphed loss", float(loss.detach()), "eager", float((eager["probs"] * gold["w"]).sum()),
      "grad err", float(np.abs(g.double().cpu().numpy() - eager["grads"][0]).max()))
