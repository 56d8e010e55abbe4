"""Debug: find the first op that breaks CUDA-graph capture of an HWF step."""
import sys, traceback
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2410_03348_b200 as sg
from paper_2410_03348_b200 import programs as P
from paper_2410_03348_b200.learn import loss_nll
DEV = torch.device("cuda", 0)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
B = 64
rng = np.random.default_rng(1)
xs = [torch.tensor(rng.uniform(0.05, 1, size=(B, 14)).astype(np.float32), device=DEV, requires_grad=True) for _ in range(L)]
def step():
    c = sg.ProgramContext(sg.DtkpAm(3), device=DEV)
    o = P.hwf(c, [sg.make_distribution(c, x, P.TOKEN_ALPHABET) for x in xs], L)
    t = torch.zeros(B, dtype=torch.int64, device=DEV)
    loss = loss_nll(sg.get_probs(o), t)
    return torch.autograd.grad(loss, xs)
s = torch.cuda.Stream(DEV); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3): step()
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
for mode in ("thread_local", "relaxed"):
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, capture_error_mode=mode):
            step()
        g.replay(); torch.cuda.synchronize(); print(mode, "capture OK")
    except Exception:
        print(mode, "FAILED"); traceback.print_exc(limit=12)
        torch.cuda.synchronize()
