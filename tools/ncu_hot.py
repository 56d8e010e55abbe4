"""Hottest SASS instructions (warp-stall samples) of one kernel from an ncu report:
    python tools/ncu_hot.py <report.ncu-rep> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
# --launch N: the N-th captured launch of the kernel (0-based; default the first)
want = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
data = []
seen = 0
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        seen += 1
        if seen > want:
            break
        continue
    if seen == want and len(r) == len(h) and r[0] != "Address":
        data.append(dict(zip(h, r)))
stall_cols = [c for c in h if c.startswith("stall_")]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
agg = {c: sum(float(d[c] or 0) for d in data) for c in stall_cols}
print(f"total samples {tot:.0f}; by reason:",
      ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
data.sort(key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    reasons = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{d['Address']:>6} {s / tot:6.1%} {d['Source'][:60]:60s} " + " ".join(f"{n}={v:.0f}" for v, n in reasons))

if "--exec" in sys.argv:
    # executed-instruction weight per contiguous address block (loop bodies)
    data.sort(key=lambda d: int(d["Address"], 16))
    tot_ex = sum(float(d["Instructions Executed"] or 0) for d in data)
    print(f"executed warp-instructions: {tot_ex:.0f}")
    run, start, acc = None, None, 0.0
    for d in data:
        ex = float(d["Instructions Executed"] or 0)
        if run is None or ex != run:
            if run is not None and acc / tot_ex > 0.01:
                print(f"  {start}..  x{run:.0f}  {acc / tot_ex:5.1%}  ({acc / run:.0f} instrs)")
            run, start, acc = ex, d["Address"], 0.0
        acc += ex
    if run and acc / tot_ex > 0.01:
        print(f"  {start}..  x{run:.0f}  {acc / tot_ex:5.1%}  ({acc / run:.0f} instrs)")
