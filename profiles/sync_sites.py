"""Average host gap / blocked time per sync call site from a DQTG_SYNC_TRACE log.
usage: python profiles/sync_sites.py trace.txt [skip_first_n]"""
import collections
import sys

skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lines = open(sys.argv[1]).read().split("\n")
if any(ln.startswith("MARK") for ln in lines):  # only between the first MARK pair
    i0 = next(i for i, ln in enumerate(lines) if ln.startswith("MARK"))
    i1 = next(i for i, ln in enumerate(lines) if ln.startswith("MARK") and i > i0)
    lines = lines[i0:i1]
rows = [ln.split() for ln in lines if ln.startswith("sync ")]
rows = rows[skip:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    # sync <fn> :<line> host <us> us blocked <us> us   (fn and :line may be fused)
    site = " ".join(r[1:r.index("host")])
    h, b = float(r[r.index("host") + 1]), float(r[r.index("blocked") + 1])
    a = agg[site]
    a[0] += 1
    a[1] += h
    a[2] += b
    a[3] = max(a[3], h)
tot_h = sum(a[1] for a in agg.values())
tot_b = sum(a[2] for a in agg.values())
print(f"{len(rows)} syncs, host {tot_h / 1e3:.2f} ms, blocked {tot_b / 1e3:.2f} ms")
for s, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {s:40s} n {a[0]:5d} host avg {a[1] / a[0]:8.1f} max {a[3]:9.1f} us  blocked avg {a[2] / a[0]:8.1f} us")

tps = collections.defaultdict(list)
for ln in lines:
    if ln.startswith("tp "):
        p = ln.split()
        tps[int(p[1])].append(float(p[2]))
for k in sorted(tps):
    v = tps[k]
    print(f"  tp line {k:5d} n {len(v):4d} avg {sum(v) / len(v):8.1f} max {max(v):9.1f} us")
