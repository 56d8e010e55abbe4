"""Summarise ncu captures (gpurun_out/) into committed markdown under profiles/.

    python tools/ncu_summary.py --tag r01
Reads ``<tag>_step_launches.csv`` (launch list of the captured Sum-15 step) and every
``<tag>_full_*.ncu-rep`` (``ncu --set full`` of one launch) and writes
``profiles/<tag>_ncu_summary.md``.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__waves_per_multiprocessor", "waves/SM"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", None),
]


def launch_table(path: Path):
    rows = list(csv.reader(path.open()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    L = list(launches.values())
    # the last complete captured step: from the last loss-forward launch back to the previous one
    idx = [i for i, l in enumerate(L) if "k_nll_fwd" in l["name"]]
    if len(idx) >= 2:
        a, b = idx[-2], idx[-1]
        step = L[a + 1: b + 1]
    else:
        step = L
    agg = collections.OrderedDict()
    step = [l for l in step if not ("FillFunctor" in l["name"] and l.get("dram__bytes_write.sum", 0) > 4e8)]
    for l in step:  # (the 512 MB L2-flush memset between timed steps is excluded above)
        name = l["name"].split("(")[0].replace("void ", "")[:48]
        e = agg.setdefault(name, [0, 0.0, 0.0])
        e[0] += 1
        e[1] += l.get("gpu__time_duration.sum", 0.0)
        e[2] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    return step, agg


def raw_metrics(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        res.append((d, u))
    return res


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
          "msecond": 1e-3, "second": 1.0}


def to_si(v, unit):
    """Value in bytes or seconds (None when the unit is not a size/time)."""
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return None
    return x * _SCALE[unit] if unit in _SCALE else None


def fmt(v, unit):
    si = to_si(v, unit)
    if si is not None and "byte" in unit:
        return f"{si / 1e6:.2f} MB"
    if si is not None:
        return f"{si * 1e6:.2f} us"
    try:
        return f"{float(str(v).replace(',', '')):g} {unit}".strip()
    except ValueError:
        return str(v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    args = ap.parse_args()
    lines = [f"# ncu evidence — round {args.tag}", "",
             "Captured on 1x B200 with `tools/ncu_round.sh` (ncu 2025, `--clock-control none`). ",
             "Peak for fractions: MEASURED_PEAKS.json hbm_gbs = %.1f GB/s (measured)." % PEAK, ""]
    ll = OUT / f"{args.tag}_step_launches.csv"
    if ll.exists():
        step, agg = launch_table(ll)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list of one captured Sum-15 step (B=16384, `--cache-control none`: warm L2 as in the run)",
                  "", "ncu serialises launches and adds per-launch overhead: compare **shares**, not absolutes.", "",
                  "| kernel | launches | time (us) | share | DRAM bytes (MB) | DRAM GB/s |", "|---|---|---|---|---|---|"]
        for name, (n, t, byts) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{name}` | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% | {byts / 1e6:.2f} | "
                         f"{byts / max(t, 1e-9):.0f} |")
        lines += ["", f"Total {tot / 1e3:.1f} us over {len(step)} launches.", ""]
    for rep in sorted(OUT.glob(f"{args.tag}_full_*.ncu-rep")):
        kern = rep.stem.replace(f"{args.tag}_full_", "")
        lines += [f"## `ncu --set full`: {kern}", ""]
        for d, u in raw_metrics(rep):
            lines.append(f"Launch `{d.get('Kernel Name', '?')[:90]}`")
            lines += ["", "| metric | value |", "|---|---|"]
            for key, label in METRICS:
                if key in d:
                    lines.append(f"| {label or key} (`{key}`) | {fmt(d[key], u.get(key, ''))} |")
            t = to_si(d.get("gpu__time_duration.sum", ""), u.get("gpu__time_duration.sum", ""))
            br = to_si(d.get("dram__bytes_read.sum", ""), u.get("dram__bytes_read.sum", ""))
            bw = to_si(d.get("dram__bytes_write.sum", ""), u.get("dram__bytes_write.sum", ""))
            if t and br is not None and bw is not None:
                lines.append(f"| traffic = DRAM read + write | {(br + bw) / 1e6:.2f} MB |")
                lines.append(f"| traffic / duration | {(br + bw) / t / 1e9:.0f} GB/s "
                             f"({100 * (br + bw) / t / 1e9 / PEAK:.1f}% of measured peak) |")
            lines.append("")
    # per-launch DRAM traffic of the captured kernels -> profiles/traffic.json (bench.py's
    # roofline.traffic for the dominant kernel)
    traffic = {}
    for rep in sorted(OUT.glob(f"{args.tag}_full_*.ncu-rep")):
        kern = rep.stem.replace(f"{args.tag}_full_", "")
        for d, u in raw_metrics(rep)[:1]:
            br = to_si(d.get("dram__bytes_read.sum", ""), u.get("dram__bytes_read.sum", ""))
            bw = to_si(d.get("dram__bytes_write.sum", ""), u.get("dram__bytes_write.sum", ""))
            if br is not None and bw is not None:
                traffic[kern] = {"bytes_per_launch": br + bw, "read": br, "write": bw,
                                 "batch": 16384 if kern.startswith(("k_chain", "k_nll")) else None,
                                 "source": f"profiles/{args.tag}_ncu_summary.md (ncu --set full, {rep.name})"}
    if traffic:
        (ROOT / "profiles" / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    dst = ROOT / "profiles" / f"{args.tag}_ncu_summary.md"
    dst.parent.mkdir(exist_ok=True)
    dst.write_text("\n".join(lines) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
