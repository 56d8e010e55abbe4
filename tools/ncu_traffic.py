"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels
in one `ncu --set full` report -> profiles/traffic.json (bench.py's roofline.traffic) and
a markdown summary of the key metrics.

    python tools/ncu_traffic.py gpurun_out/chain2.ncu-rep --batch 16384 --out profiles/r02_ncu_chain.md
"""

import argparse
import csv
import io
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("sm__warps_active.avg.pct_of_peak_sustained_active",
                                                  "achieved occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("launch__registers_per_thread", "registers"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("smsp__inst_executed.sum", "warp instructions")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    tr_path = ROOT / "profiles" / "traffic.json"
    traffic = json.loads(tr_path.read_text()) if tr_path.exists() else {}
    lines = [f"# ncu --set full: {Path(args.report).name} (B={args.batch})", "",
             "| kernel | " + " | ".join(n for _, n in KEYS) + " |", "|---" * (len(KEYS) + 1) + "|"]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        base = re.sub(r"<.*", "", name.replace("void ", "")).split("(")[0].split("::")[-1]
        vals = []
        for k, _ in KEYS:
            v = r[h.index(k)] if k in h else ""
            vals.append(v)
        lines.append(f"| `{name[:60]}` | " + " | ".join(vals) + " |")
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * SCALE.get(units[h.index("dram__bytes_read.sum")], 1)
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * SCALE.get(units[h.index("dram__bytes_write.sum")], 1)
        traffic[base] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "batch": args.batch,
                         "source": f"{args.out} (ncu --set full, {Path(args.report).name})"}
    tr_path.write_text(json.dumps(traffic, indent=1) + "\n")
    Path(args.out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
