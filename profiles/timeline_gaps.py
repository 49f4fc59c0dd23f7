"""Coverage of a DQTG_TIMELINE dump (profiles/pipe_timeline.py stderr): for the last
repetition, wall span, union of kernel spans (GPU busy with >=1 engine kernel),
idle gaps and per-kernel summed span time.  usage: python profiles/timeline_gaps.py timeline.txt"""
import collections
import sys

lines = open(sys.argv[1]).read().split("--- rep")
blocks = [b for b in lines if "timeline" in b]
spans = []
for ln in blocks[-1].splitlines():
    p = ln.split()
    if len(p) >= 6 and p[0] == "timeline":
        spans.append((float(p[1]), float(p[2]), p[4], p[5]))
spans.sort()
t0, t1 = spans[0][0], max(s[1] for s in spans)
busy, cur_a, cur_b, gaps = 0.0, None, None, []
for a, b, _, _ in spans:
    if cur_b is None or a > cur_b:
        if cur_b is not None:
            busy += cur_b - cur_a
            gaps.append((a - cur_b, cur_b))
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
busy += cur_b - cur_a
print(f"wall {t1 - t0:.3f} ms, busy {busy:.3f} ms ({100 * busy / (t1 - t0):.1f}%), "
      f"{len(gaps)} gaps, largest {sorted(gaps)[-5:]}")
per = collections.defaultdict(float)
cnt = collections.Counter()
for a, b, _, n in spans:
    per[n] += b - a
    cnt[n] += 1
for n, v in sorted(per.items(), key=lambda kv: -kv[1])[:16]:
    print(f"  {n:28s} {cnt[n]:4d} x  {v:8.3f} ms  ({v / cnt[n]:.3f} each)")
