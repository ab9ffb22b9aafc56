"""Per-warp time breakdown of a tools/wtc_trace.py timeline (transition -> total cycles)."""
import re
import sys
from collections import defaultdict

ev = []
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.txt"):
    m = re.match(r"\s*(\d+) w(\d+) (.*?) g=(\d+)", line)
    if m:
        ev.append((int(m.group(1)), int(m.group(2)), m.group(3), int(m.group(4))))
for W in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,2,4")]:
    e = [x for x in ev if x[1] == W]
    if len(e) < 2:
        continue
    cat, cnt = defaultdict(int), defaultdict(int)
    for a, b in zip(e, e[1:]):
        k = (a[2], b[2])
        cat[k] += b[0] - a[0]
        cnt[k] += 1
    span = e[-1][0] - e[0][0]
    print("warp", W, "span", span)
    for k, v in sorted(cat.items(), key=lambda x: -x[1]):
        print(f"   {v:8d} {100 * v / span:5.1f}% n={cnt[k]:4d} avg={v / cnt[k]:7.0f}  {k[0]} -> {k[1]}")
