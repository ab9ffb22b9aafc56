import sys, os; sys.path.insert(0, '.')
import torch, paper_2502_01659_b200 as ga
L, H = int(sys.argv[1]), int(sys.argv[2])
q, k, v = ga.qkv_device(1, L, H, 64, torch.bfloat16)
o = ga.attention(q, k, v, ga.Window(256, 2), kernel="tc")
torch.cuda.synchronize()
print("ok", L, H, float(o.float().abs().sum()))
