"""Issue-ceiling summary of DTKP kernels from `ncu --set full` captures -> profiles/issue.json.

The DTKP apply is instruction-issue bound, not HBM bound: per candidate proof
it ORs W words, multiplies the fp64 registry probabilities of the set bits in ascending
column order and inserts into a dedup-aware top-K.  Its ceiling is the SM issue rate (4 warp
instructions per cycle per SM); the fraction reported is sm__inst_executed per active
cycle / 4 (= smsp__issue_active), with the fp64 pipe share and the executed instructions
per ranked candidate row beside it.

    python tools/ncu_issue.py <report.ncu-rep> <label> [--launch N] [--candidates C]
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles" / "issue.json"

rep, label = sys.argv[1], sys.argv[2]
launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
cand = float(sys.argv[sys.argv.index("--candidates") + 1]) if "--candidates" in sys.argv else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, r = rows[0], rows[2 + launch]


def g(name):
    return float(r[h.index(name)].replace(",", ""))


ent = {
    "kernel": r[h.index("Kernel Name")],
    "duration_us": g("gpu__time_duration.sum") * {"ms": 1e3, "msecond": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3,
                                                  "nsecond": 1e-3}.get(rows[1][h.index("gpu__time_duration.sum")], 1.0),
    "issue_active_frac": g("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
    "ipc_per_sm": g("sm__inst_executed.avg.per_cycle_active"),
    "ipc_peak": 4.0,
    "warp_instructions": g("smsp__inst_executed.sum"),
    "fp64_pipe_frac": g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active") / 100,
    "warps_active_frac": g("sm__warps_active.avg.pct_of_peak_sustained_active") / 100,
    "dram_bytes": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) * 1e6,
    "registers": g("launch__registers_per_thread"),
    "source": str(Path(rep).name),
}
if cand:
    ent["warp_instructions_per_candidate_row"] = ent["warp_instructions"] * 32 / cand
d = json.loads(OUT.read_text()) if OUT.exists() else {}
d[label] = ent
OUT.write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps({label: ent}, indent=1))
