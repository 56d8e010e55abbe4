"""Kernel microbenchmark: per-launch time of the DAMP apply kernels on Sum-15 step shapes.

Each measurement replays a CUDA graph of ``reps`` launches that rotate over enough
input/output buffer sets to exceed L2 (so every launch streams from HBM), and reports
µs per launch, algorithmic GB/s and the fraction of MEASURED_PEAKS.json hbm_gbs.  A
torch device-to-device copy of the same byte count is timed the same way as a practical
ceiling for a kernel of that size.

    python tools/microbench.py [--batch 16384] [--steps 1,7,14] [--reps 64]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2410_03348_b200 import _native as N  # noqa: E402
from paper_2410_03348_b200.plan import build_plan  # noqa: E402
from paper_2410_03348_b200.programs import _add  # noqa: E402


def graph_time(fn, reps, dev):
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        t = e0.elapsed_time(e1) * 1e3 / reps
        best = t if best is None else min(best, t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--steps", default="1,4,7,10,14")
    ap.add_argument("--reps", type=int, default=64)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    lib = N.load()
    B = args.batch
    digits = tuple(range(10))
    results = []
    for i in [int(x) for x in args.steps.split(",")]:
        left = digits if i == 1 else tuple(range(9 * (i - 1) + 10))
        kp = build_plan(_add, None, [left, digits]).kernel_plan()
        s1, s2 = kp.sizes
        per_set = 4 * B * (s1 + s2 + 2 * kp.n_out + s1 + s2)
        nsets = max(2, int(400e6 // per_set) + 1)
        sets = []
        for _ in range(nsets):
            a = torch.rand((s1, B), device=dev)
            b = torch.rand((s2, B), device=dev)
            sets.append((a, b, torch.empty((kp.n_out, B), device=dev), torch.rand((kp.n_out, B), device=dev),
                         torch.empty_like(a), torch.empty_like(b)))
        st = kp.device(dev).damp_struct(B)

        def fwd(j):
            a, b, out, g, ga, gb = sets[j % nsets]
            N.check(lib.sg_damp_apply_fwd(ctypes.byref(st), N.rows_array([a, b]), B, out.data_ptr(), None,
                                          torch.cuda.current_stream(dev).cuda_stream), "fwd")

        def bwd(j):
            a, b, out, g, ga, gb = sets[j % nsets]
            N.check(lib.sg_damp_apply_bwd(ctypes.byref(st), N.rows_array([a, b]), N.rows(g), B,
                                          N.rows_array([ga, gb]), None, torch.cuda.current_stream(dev).cuda_stream),
                    "bwd")

        fb = 4 * B * (s1 + s2 + kp.n_out)
        bb = 4 * B * (kp.n_out + 2 * (s1 + s2))
        # a copy of fb/2 bytes moves fb bytes (read + write): same traffic as the forward
        csrc = [torch.rand(fb // 8, device=dev) for _ in range(max(2, int(400e6 // fb) + 1))]
        cdst = [torch.empty_like(c) for c in csrc]

        def copy(j):
            cdst[j % len(csrc)].copy_(csrc[j % len(csrc)])

        tf = graph_time(fwd, args.reps, dev)
        tb = graph_time(bwd, args.reps, dev)
        tc = graph_time(copy, args.reps, dev)
        row = {"step": i, "S1": s1, "n_out": kp.n_out, "fwd_us": tf, "fwd_gbs": fb / tf / 1e3, "fwd_frac": fb / tf / 1e3 / hbm,
               "bwd_us": tb, "bwd_gbs": bb / tb / 1e3, "bwd_frac": bb / tb / 1e3 / hbm,
               "copy_us_same_traffic_as_fwd": tc, "copy_frac": fb / tc / 1e3 / hbm}
        results.append(row)
        print(json.dumps(row), flush=True)
        del sets, csrc, cdst
        torch.cuda.empty_cache()
    tot_f = sum(r["fwd_us"] for r in results)
    print(json.dumps({"summary": "per-launch, HBM-streamed (rotating buffers > L2)", "fwd_us_total": tot_f,
                      "bwd_us_total": sum(r["bwd_us"] for r in results)}))


if __name__ == "__main__":
    main()
