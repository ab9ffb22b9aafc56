"""Compare the tcgen05 window kernel with the band kernel on several shapes (debug aid):
max |diff| and the first differing rows."""
import sys
import os
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_01659_b200 as ga

cases = [(3000, 65, 1, 2), (3000, 128, 1, 2), (3000, 256, 2, 2), (20000, 256, 2, 2), (65536, 256, 2, 8)]
for L, w, r, H in cases:
    q, k, v = ga.qkv_device(5, L, H, 64, torch.bfloat16)
    a = ga.attention(q, k, v, ga.Window(w, r), kernel="tc").float()
    b = ga.attention(q, k, v, ga.Window(w, r), kernel="window").float()
    d = (a - b).abs().amax(dim=(1, 2))
    bad = torch.nonzero(d > 2e-2).flatten()
    print(f"L={L} w={w} r={r} H={H}: max {d.max().item():.3e}, bad rows {bad.numel()}", bad[:20].tolist(),
          "cls", sorted(set(((bad.cpu() // r) % 128).tolist()))[:20] if bad.numel() else "")
