"""Probe (copied into tests/ on the GPU box): which module cache, cleared before the
capture, makes the graphed CLUTRR closure match eager after the golden cases ran."""
import os

import numpy as np
import pytest

from runners import load_golden, run_gpu
from test_fixpoint import _graphed


@pytest.mark.gpu
def test_zz_order(cuda):
    import torch

    from paper_2410_03348_b200 import distribution as D
    from paper_2410_03348_b200 import ops
    from paper_2410_03348_b200 import plan as PL
    from paper_2410_03348_b200 import provenance as PV

    what = os.environ.get("ZZ_CLEAR", "")
    if "words" in what:
        PV._WORDS_CACHE.clear()
    if "union" in what:
        D._UNION_CACHE.clear()
    if "map" in what:
        ops._MAP_CACHE.clear()
        ops._GATHER_CACHE.clear()
    if "sched" in what:
        ops._SCHED.clear()
    if "plan" in what:
        PL.plan_cache_clear()
    if "prov" in what:
        for n in ("_GROUPS", "_COLWISE", "_PAIRMAX"):
            getattr(PV, n).clear()
    if "filter" in what:
        D._FILTER_CACHE.clear()
    name = "dtkp_clutrr_e5_r20_k5"
    gold = load_golden(name)
    x = gold["in0"]
    eager = run_gpu(name, [x])
    if os.environ.get("ZZ_AFTER"):  # clear after the eager run, right before the capture
        PV._WORDS_CACHE.clear()
    wu = int(os.environ.get("ZZ_WARMUP", "3"))
    if os.environ.get("ZZ_WARMUP"):
        import paper_2410_03348_b200 as sg
        from paper_2410_03348_b200.programs import _chain_link, kinship_compose
        import golden_cases as G
        wt = torch.as_tensor(gold["w"], device=cuda)
        gc = sg.GraphedClosure(kinship_compose, _chain_link, G.clutrr_facts(5), lambda: sg.DtkpAm(5),
                               torch.tensor(x, device=cuda, dtype=torch.float32),
                               loss_fn=lambda p: (p.double() * wt).sum(), warmup=wu)
    else:
        gc = _graphed(cuda, x, w=gold["w"])
    loss, g = gc(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    err = float(np.abs(g.double().cpu().numpy() - eager["grads"][0]).max())
    print(f"ZZ {what!r} grad err {err} loss {float(loss.detach())} eager loss {float((eager['probs'] * gold['w']).sum())}")
    loss2, g2 = gc(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    print("ZZ replay 2 grad err", float(np.abs(g2.double().cpu().numpy() - eager["grads"][0]).max()), float(loss2.detach()))
    gp = _graphed(cuda, x)
    pr = gp(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    print("ZZ no-loss graph probs err", float(np.abs(pr.double().cpu().numpy() - eager["probs"]).max()))
    gc3 = _graphed(cuda, x, w=gold["w"])
    l3, g3 = gc3(torch.tensor(x, device=cuda, dtype=torch.float32))
    torch.cuda.synchronize()
    print("ZZ second loss graph grad err", float(np.abs(g3.double().cpu().numpy() - eager["grads"][0]).max()), float(l3.detach()))
    assert err == 0.0
