"""Summarise an `ncu --set full` report: per kernel duration, DRAM traffic, achieved
DRAM GB/s, issue/occupancy and top stall reasons (markdown), plus
profiles/ncu_traffic.json (dram read+write bytes per launch) for bench.py's roofline.
usage: python profiles/ncu_summary.py report.ncu-rep out.md"""
import csv
import io
import json
import os
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
col = {k: i for i, k in enumerate(h)}


def val(r, k):
    try:
        return float(r[col[k]])
    except (KeyError, ValueError):
        return float("nan")


lines = ["| kernel | time us | DRAM read MB | DRAM write MB | DRAM GB/s | issue active % | "
         "warps active % | regs | top stalls (cycles per issue) |", "|---" * 9 + "|"]
traffic = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("dqtg::", "")
    base = name.split("<")[0]
    t = val(r, "gpu__time_duration.sum")  # us
    units = rows[1]  # per-metric units (Kbyte / Mbyte / Gbyte, ns / us / ms)

    def mb(k):
        u = units[col[k]].lower()
        return val(r, k) * {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1.0, "gbyte": 1e3}.get(u, 1.0)

    tu = units[col["gpu__time_duration.sum"]].lower()
    t_us = t * {"msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}.get(tu, 1.0)
    rd_mb, wr_mb = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    gbs = (rd_mb + wr_mb) * 1e6 / (t_us * 1e-6) / 1e9 if t_us else float("nan")
    st = sorted(((val(r, k), k) for k in h if k.startswith("smsp__average_warps_issue_stalled")
                 and k.endswith("per_issue_active.ratio")), reverse=True)[:3]
    sts = ", ".join(f"{k.split('stalled_')[1].replace('_per_issue_active.ratio', '')} {v:.1f}"
                    for v, k in st)
    lines.append(f"| {name} | {t_us:.1f} | {rd_mb:.1f} | {wr_mb:.1f} | {gbs:.0f} | "
                 f"{val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{val(r, 'launch__registers_per_thread'):.0f} | {sts} |")
    traffic[base] = int((rd_mb + wr_mb) * 1e6)
with open(out, "w") as f:
    f.write(f"# ncu --set full summary ({os.path.basename(rep)})\n\n" + "\n".join(lines) + "\n")
with open(os.path.join(os.path.dirname(out), "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
print("\n".join(lines))
