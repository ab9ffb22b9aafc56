"""Repeat the LongNet tcgen05 kernels with the TMA lattice loader and compare each output
with the cp.async loader's (bitwise): reports which rows differ and their valuations."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_01659_b200 as ga  # noqa: E402

L, w0, alpha, H, d = 65536, 2048, 2, 2, 64
q, k, v = ga.qkv_device(L + 3, L, H, d, torch.bfloat16)
m = ga.LongNet(w0, alpha)
os.environ["GA_LNET_CPASYNC"] = "1"
ref = ga.attention(q, k, v, m, kernel="tc")
r0 = (L // 3 // w0) * w0
ref_part = ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc")
os.environ.pop("GA_LNET_CPASYNC")
nbad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    a = ga.attention(q, k, v, m, kernel="tc")
    part = ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc")
    torch.cuda.synchronize()
    for name, x, y, off in (("full", a, ref, 0), ("part", part, ref_part, r0)):
        if not torch.equal(x, y):
            nbad += 1
            diff = (x.float() - y.float()).abs().amax(dim=(1, 2))
            rows = (diff > 0).nonzero().flatten()
            rr = (rows + off).tolist()
            nu = [(r & -r).bit_length() - 1 if r else 99 for r in rr[:12]]
            print(it, name, "rows differing", len(rr), "first", rr[:12], "valuations", nu,
                  "max diff", diff.max().item())
print("bad runs", nbad)
