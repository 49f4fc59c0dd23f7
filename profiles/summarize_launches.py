"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per engine kernel, launches / total / share of engine time."""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"], float(r["Metric Value"]), r.get("Metric Unit", "")))
agg = defaultdict(lambda: [0, 0.0])
for name, v, unit in rows:
    if not ("dqtg" in name or "kernel" in name.split("(")[0]):
        continue
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    key = name.split("(")[0].replace("void ", "").strip()
    agg[key][0] += 1
    agg[key][1] += v * scale
eng = {k: v for k, v in agg.items() if "dqtg::" in k}
tot = sum(v[1] for v in eng.values())
print("| kernel | launches | total us | share of engine time |")
print("|---|---|---|---|")
for k, (n, us) in sorted(eng.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
