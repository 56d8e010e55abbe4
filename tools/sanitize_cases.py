"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) over the
kernels with cross-thread protocols: the DTKP apply (shared probability tile, dynamic
per-column work counters reset by the last CTA, two-level merge of split segments), the
fused loss (last-CTA ticket), the chain kernels and the generic segmented apply.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from runners import run_gpu  # noqa: E402

import paper_2410_03348_b200 as sg  # noqa: E402
from paper_2410_03348_b200 import ops  # noqa: E402
from paper_2410_03348_b200.learn import loss_nll  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    # DTKP: HWF-5 (split segments + merges), CLUTRR closure (k=5, unions), dynamic and static
    # (round 2: HWF-7 for the keyed conj's continuation / pruning / first fill and the
    # adaptive piece size; the benchmarked CLUTRR closure for k = 5)
    for name in ("dtkp_hwf5", "dtkp_hwf7", "dtkp_clutrr_k5", "dtkp_clutrr_e5_r20_k5", "dtkp_stack_k3"):
        run_gpu(name)
    ops.DTKP_DYNAMIC = False
    run_gpu("dtkp_hwf3")
    ops.DTKP_DYNAMIC = True
    # fused loss: one-pass, chunked (many symbols, small batch) and given-rowsum paths
    rng = np.random.default_rng(0)
    for B, n in ((40, 2500), (1000, 20), (64, 300)):
        x = torch.tensor(rng.uniform(0.01, 1, size=(B, n)).astype(np.float32), device=dev, requires_grad=True)
        loss_nll(x, torch.tensor(rng.integers(0, n, size=B), device=dev)).backward()
    # DAMP chain (fused fwd/bwd) + loss on the rowsum path, generic segmented apply
    # (damp_sum15 at B = 4 runs the 16-row-group chain variant; the sweep case the
    # sample-pair Toeplitz kernels; max_sum4 the fused max chain with 4 lanes per sample)
    for name in ("damp_sum15", "damp_sweep_a2_s10", "damp_mod_cond_a2", "damp_mod_a3", "damp_union_filter",
                 "max_sum4"):
        run_gpu(name)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
