"""A/B of the LongNet tcgen05 loaders (TMA lattice boxes vs cp.async) on the same inputs:
bitwise comparison of full and query-sub-range outputs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_01659_b200 as ga  # noqa: E402

for (L, w0, alpha) in [(65536, 2048, 2), (5000, 300, 2), (8192, 256, 2)]:
    H, d = 2, 64
    q, k, v = ga.qkv_device(L + 3, L, H, d, torch.bfloat16)
    m = ga.LongNet(w0, alpha)
    r0 = (L // 3 // w0) * w0
    res = {}
    for mode in ("tma", "cpa"):
        if mode == "cpa":
            os.environ["GA_LNET_CPASYNC"] = "1"
        else:
            os.environ.pop("GA_LNET_CPASYNC", None)
        a = ga.attention(q, k, v, m, kernel="tc")
        part = ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc")
        torch.cuda.synchronize()
        res[mode] = (a, part)
    a_t, p_t = res["tma"]
    a_c, p_c = res["cpa"]
    diff = (a_t.float() - a_c.float()).abs()
    print(L, w0, "tma==cpa full:", torch.equal(a_t, a_c), "max diff", diff.max().item(),
          "rows differing", int((diff.amax(dim=(1, 2)) > 0).sum()),
          "| part==full tma:", torch.equal(p_t, a_t[r0:]), "cpa:", torch.equal(p_c, a_c[r0:]))
    if not torch.equal(a_t, a_c):
        bad = (diff.amax(dim=(1, 2)) > 0).nonzero().flatten()[:10].tolist()
        print("  first differing rows", bad)
