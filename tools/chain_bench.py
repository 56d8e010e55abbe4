"""Per-launch time of the fused Sum-15 chain kernels (bench.kernel_roofline) at a few
batch sizes: python tools/chain_bench.py [--batch 16384,65536]"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", default="16384")
args = ap.parse_args()
hbm = bench.peaks()[0]["hbm_gbs"]
dev = torch.device("cuda", 0)
for B in [int(x) for x in args.batch.split(",")]:
    r = bench.kernel_roofline(torch, dev, B, hbm)
    print(json.dumps({"B": B, **{k: {"us": round(v["avg_us"], 2), "frac": round(v["frac"], 3)} for k, v in r.items()}}))
