"""Timeline of one group-mode CTA of the LongNet tcgen05 kernel (debug build with
-DGA_LNET_TRACE at abtest/libga_ltrace.so): per chunk, when the stage landed, S was issued /
ready, P arrived, P V's WAR wait ended; gaps in cycles."""
import ctypes
import os
import sys
from collections import defaultdict

os.environ["GA_LIB"] = os.path.abspath("abtest/libga_ltrace.so")
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2502_01659_b200 as ga  # noqa: E402

WL, WM = int(os.environ.get("LT_LOADER", "4")), int(os.environ.get("LT_MMA", "5"))  # loader / MMA warp

L = 1 << 22
q, k, v = ga.qkv_device(1, L, 1, 64, torch.bfloat16)
m = ga.LongNet(2048, 2)
lib = ga._abi.lib()
N = 8192
buf = (ctypes.c_ulonglong * N)()
for _ in range(2):
    ga.attention(q, k, v, m, kernel="tc")
torch.cuda.synchronize()
lib.ga_lnet_trace_read(buf, N)
ga.attention(q, k, v, m, kernel="tc")
torch.cuda.synchronize()
lib.ga_lnet_trace_read(buf, N)
ev = sorted(((b & 0xffffffffff), (b >> 48) & 0xff, (b >> 40) & 0xff, b >> 56) for b in buf if b)
names = {0: "start", 1: "mma: stage landed", 3: "mma: P arrived", 7: "mma: PV done (WAR)", 10: "smx: wait S",
         12: "smx: S ready", 14: "smx: P arrive", 20: "ldr: stage free", 99: "end"}
print(len(ev), "events; span", ev[-1][0] - ev[0][0], "cycles")
per = defaultdict(dict)
for t, e, w, c in ev:
    per[(e, w)].setdefault(c, t)
end = max(t for t, e, w, c in ev if e == 99)
print("end of CTA at", end)
for e, nm in ((30, "TMEM + barriers ready"), (31, "pieces ready"), (32, "Q loads issued (loader)")):
    ts = sorted(t for t, ev, w, c in ev_all if ev == e) if False else sorted(t for t, ev, w, c in ev if ev == e)
    if ts: print(f"{nm}: first {ts[0]} last {ts[-1]}")
for c in range(0, 48):
    row = []
    for (e, w) in [(20, WL), (1, WM), (10, 0), (12, 0), (14, 0), (12, 3), (14, 3), (3, WM), (7, WM)]:
        row.append(per.get((e, w), {}).get(c, -1))
    if all(x < 0 for x in row):
        break
    print(f"c={c:2d} " + " ".join(f"{names[e][:14]:>14s}={x:7d}" for (e, w), x in
                               zip([(20, WL), (1, WM), (10, 0), (12, 0), (14, 0), (12, 3), (14, 3), (3, WM), (7, WM)], row)))
# softmax busy vs waiting
w0 = [(t, e, c) for t, e, w, c in ev if w == 0 and e in (10, 12, 14)]
wait = sum(per[(12, 0)][c] - per[(10, 0)][c] for c in per[(12, 0)] if c in per[(10, 0)])
busy = sum(per[(14, 0)][c] - per[(12, 0)][c] for c in per[(14, 0)] if c in per[(12, 0)])
print("softmax warp 0: waiting for S", wait, "cycles; working", busy, "cycles; chunks", len(per[(14, 0)]))
print("per chunk: P arrive of softmax warps 0-3 and the MMA warp's P-arrived time")
for c in range(0, 48):
    xs = [per.get((14, w), {}).get(c, -1) for w in range(4)] + [per.get((3, 5), {}).get(c, -1)]
    ss = [per.get((12, w), {}).get(c, -1) for w in range(4)]
    if all(x < 0 for x in xs):
        break
    print(f"c={c:2d} S ready " + " ".join(f"{x:7d}" for x in ss) + " | P arrive " + " ".join(f"{x:7d}" for x in xs[:4]) +
          f" | mma sees {xs[4]:7d} (+{xs[4] - max(xs[:4]):5d})")
