"""Band-kernel phase timing (experimental build with -DGA_BAND_PROF at abtest/libga_prof.so):
sum over warps of clock64 cycles per phase, as fractions of the warps' total lifetime."""
import ctypes
import os
import sys

os.environ["GA_LIB"] = os.path.abspath("abtest/libga_prof.so")
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2502_01659_b200 as ga  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
L, H, w, r = {"cfg2": (65536, 8, 256, 2), "cfg5": (16_000_000, 1, 128, 1)}[cfg]
q, k, v = ga.qkv_device(1, L, H, 64, torch.bfloat16)
m = ga.Window(w, r)
lib = ga._abi.lib()
buf = (ctypes.c_ulonglong * 8)()
for _ in range(3):
    ga.attention(q, k, v, m)
torch.cuda.synchronize()
lib.ga_band_prof_read(buf)
ga.attention(q, k, v, m)
torch.cuda.synchronize()
lib.ga_band_prof_read(buf)
names = ["load wait (stage 0)", "CUDA-core triangles + hand-off", "wait dense rows", "MMA phase", "epilogue", "total"]
tot = buf[5]
for i, n in enumerate(names):
    print(f"{n:32s} {buf[i]:16d}  {100 * buf[i] / max(tot, 1):6.1f}%")
