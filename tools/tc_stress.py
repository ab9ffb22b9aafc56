"""Stress the tcgen05 window kernel: many launches over assorted shapes (hang / nondeterminism check)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_2502_01659_b200 as ga

shapes = [(65536, 256, 2, 8), (3000, 128, 1, 2), (20000, 256, 2, 3), (131072, 129, 1, 1), (50000, 400, 4, 2)]
t0 = time.time()
for L, w, r, H in shapes:
    q, k, v = ga.qkv_device(11, L, H, 64, torch.bfloat16)
    ref = ga.attention(q, k, v, ga.Window(w, r), kernel="tc")
    for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
        out = ga.attention(q, k, v, ga.Window(w, r), kernel="tc")
        if i % 50 == 0:
            torch.cuda.synchronize()
            assert torch.equal(out, ref), (L, w, r, H, i)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    print(f"L={L} w={w} r={r} H={H} ok {time.time() - t0:.1f}s", flush=True)
