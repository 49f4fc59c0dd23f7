"""Per-CUDA-line hotspots from `ncu -i rep --page source --csv --print-source cuda,sass -k <k>`.

In the mixed view each CUDA line row ("Line No", "Source") is followed by its SASS rows
("", "", address, sass, metrics...).  SASS metrics are summed onto the preceding CUDA
line.  Prints the top lines by warp-stall samples with executed warp instructions.

usage: ncu ... | python profiles/src_hotspots.py [top]"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
fname, cur, hdr = "", None, None
samp, inst = {}, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0]:  # CUDA line
        cur = (fname, r[0], r[1].strip()[:80])
        continue
    if cur is None:
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = float(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    samp[cur] = samp.get(cur, 0) + s
    inst[cur] = inst.get(cur, 0) + n
ts = sum(samp.values()) or 1
ti = sum(inst.values()) or 1
print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
for k, v in sorted(samp.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / ts:5.1f}% stall {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]:>5}  {k[2]}")
