"""Per-CUDA-line warp-stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
cur = None
agg = {}
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < 6 or r[0] in ("Line No",):
        continue
    if r[0]:  # cuda line row
        cur = (fname, r[0], r[1][:90])
        try:
            agg[cur] = agg.get(cur, 0) + float(r[4] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[1]) if len(sys.argv) > 1 else 25]:
    print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:>5}  {k[2]}")
