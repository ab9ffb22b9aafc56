"""Hang guard / smoke for the LongNet tcgen05 kernel: one small call, checked against the edge kernel."""
import sys; sys.path.insert(0, '.')
import torch, paper_2502_01659_b200 as ga
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
q, k, v = ga.qkv_device(1, L, 1, 64, torch.bfloat16)
m = ga.LongNet(2048, 2)
o = ga.attention(q, k, v, m)
e = ga.attention(q, k, v, m, kernel="edge")
torch.cuda.synchronize()
print("ok", L, float((o.float() - e.float()).abs().max()))
