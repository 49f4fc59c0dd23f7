"""Largest host gaps (DQTG_SYNC_TRACE) inside each pipelined run of a bench log
(DQTG_PIPE_TRACE blocks delimit the runs: a run's syncs precede its trace block).
usage: python profiles/pipe_stalls.py bench.err"""
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
blocks, start = [], None
for i, ln in enumerate(lines):
    if ln.startswith("pipe k="):
        if start is None:
            start = i
    elif start is not None:
        blocks.append((start, i))
        start = None
prev_end = 0
for b0, b1 in blocks:
    ends = [float(re.search(r"encoded ([\d.]+)", ln).group(1)) for ln in lines[b0:b1]]
    worst = []
    for ln in lines[prev_end:b0]:
        if ln.startswith("sync ") or ln.startswith("tp "):
            m = re.search(r"host\s+([\d.]+)", ln) if ln.startswith("sync") else re.match(r"tp \d+ ([\d.-]+)", ln)
            v = float(m.group(1)) if m else 0.0
            worst.append((v, ln.strip()[:90]))
    worst.sort(reverse=True)
    print(f"run lines {b0}-{b1}: {max(ends):8.1f} ms  top host gaps: {[round(w[0] / 1e3, 1) for w in worst[:3]]} ms")
    for w in worst[:2]:
        if w[0] > 20000:
            print("    ", w[1])
    prev_end = b1
