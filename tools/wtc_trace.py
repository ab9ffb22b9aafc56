"""Timeline of CTA 0 of the tcgen05 window kernel (debug build with -DGA_WTC_TRACE at
abtest/libga_trace.so): per event type, count and mean gap to the previous event of the
same warp; plus the first events in order."""
import ctypes
import os
import sys
from collections import defaultdict

os.environ["GA_LIB"] = os.path.abspath("abtest/libga_trace.so")
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2502_01659_b200 as ga  # noqa: E402

L, H, w, r = (int(x) for x in os.environ.get("WTC_SHAPE", "65536,8,256,2").split(","))
q, k, v = ga.qkv_device(1, L, H, 64, torch.bfloat16)
m = ga.Window(w, r)
lib = ga._abi.lib()
N = 16384
buf = (ctypes.c_ulonglong * N)()
for _ in range(3):
    ga.attention(q, k, v, m, kernel="tc")
torch.cuda.synchronize()
lib.ga_wtc_trace_read(buf, N)
ga.attention(q, k, v, m, kernel="tc")
torch.cuda.synchronize()
n = lib.ga_wtc_trace_read(buf, N)
ev = sorted(((b & 0xffffffffff), (b >> 48) & 0xff, (b >> 40) & 0xff, b >> 56) for b in buf[:n] if b)
names = {3: "mma: P arrived", 6: "mma: S issued", 10: "smx A: wait S start", 11: "smx B: wait S start", 12: "smx A: S ready",
         13: "smx B: S ready", 14: "smx A: P arrive", 15: "smx B: P arrive", 18: "epi: A tile ready", 19: "epi: B tile ready",
         20: "loader: fill issued", 16: "smx A: tile end", 17: "smx B: tile end", 22: "smx A: OFREE ok", 23: "smx B: OFREE ok", 24: "smx A: S loaded", 25: "smx B: S loaded", 26: "smx A: max+vote done", 27: "smx B: max+vote done", 28: "smx A: exps+st issued", 29: "smx B: exps+st issued", 30: "smx A: st done", 31: "smx B: st done", 21: "loader: wants slot"}
print(f"{n} events, span {ev[-1][0] - ev[0][0]} cycles")
last = {}
gaps = defaultdict(list)
for t, e, wp, gv in ev:
    key = (wp,)
    if key in last:
        gaps[(e, wp)].append(t - last[key][0])
    last[key] = (t, e)
for (e, wp), g in sorted(gaps.items()):
    print(f"{names.get(e, e):24s} warp {wp}: n={len(g):5d} mean gap since previous event of the warp {sum(g) / len(g):8.1f}")
for t, e, wp, gv in ev[:int(sys.argv[1]) if len(sys.argv) > 1 else 120]:
    print(f"{t:10d} w{wp} {names.get(e, e)} g={gv}")
