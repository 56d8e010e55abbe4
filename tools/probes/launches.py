"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]):
    python tools/probes/launches.py gpurun_out/x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
k = defaultdict(dict)
for r in rows:
    k[(int(r["ID"]), r["Kernel Name"][:60])][r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])


def val(m, name):
    v, u = m.get(name, ("0", ""))
    v = float(v.replace(",", ""))
    return v * {"ms": 1e6, "us": 1e3, "usecond": 1e3, "msecond": 1e6}.get(u, 1.0)


tot = sum(val(m, "gpu__time_duration.sum") for m in k.values())
print(f"{len(k)} launches, {tot / 1e3:.1f} us")
for (i, n), m in sorted(k.items()):
    t = val(m, "gpu__time_duration.sum")
    if t > 0.01 * tot:
        by = val(m, "dram__bytes_read.sum") + val(m, "dram__bytes_write.sum")
        print(f"{i:4d} {n:60s} {t / 1e3:9.1f} us {t / tot:6.1%} regs={m.get('launch__registers_per_thread', ('', ''))[0]}"
              f" grid={m.get('launch__grid_size', ('', ''))[0]} dram={by / 1e6:.1f}MB")
