"""Per-CUDA-line executed warp instructions (mixed cuda,sass source page), in line order.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k K | python profiles/line_insts.py [min_pct]"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr, cur, inst, fname = None, None, {}, ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:75])
        continue
    try:
        n = float(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    inst[cur] = inst.get(cur, 0) + n
tot = sum(inst.values()) or 1
lim = float(sys.argv[1]) if len(sys.argv) > 1 else 0.4
print(f"total {tot:.3e}")
for k, v in sorted(inst.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if 100 * v / tot >= lim:
        print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
