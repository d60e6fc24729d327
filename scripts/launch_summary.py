"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
a markdown table: kernel, grid, launches, avg us, share.
    python scripts/launch_summary.py gpurun_out/launches.csv [steps] > profiles/x.md"""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
    name = r["Kernel Name"]
    if len(name) > 60:
        name = name[:57] + "..."
    k = (name, r.get("Grid Size", ""))
    agg[k][0] += 1
    agg[k][1] += us
total = sum(v[1] for v in agg.values())
print("| kernel | grid | launches | avg us | share |\n|---|---|---|---|---|")
for (name, grid), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name}` | {grid} | {n} | {t / n:.2f} | {100 * t / total:.1f}% |")
if steps:
    print(f"\nSerialised kernel time per step: {total / steps:.1f} us over {steps} steps")
