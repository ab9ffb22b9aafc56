import torch, paper_2502_01659_b200 as ga
L, H, d = 10000, 2, 64
q, k, v = ga.qkv_device(31, L, H, d, torch.bfloat16)
mask = ga.LongNet(256, 2)
ref = ga.attention(q, k, v, mask, kernel="tc")
for it in range(4):
    if it % 2: ga.attention(q * 7.0, k * -3.0, v, ga.Window(300, 3))
    again = ga.attention(q, k, v, mask, kernel="tc")
    bad = (again != ref).any(-1).nonzero()
    print(it, "mismatch (row,head)", bad.shape[0], bad[:12].tolist(), (again.float() - ref.float()).abs().max().item())
al = ga.query_alignment(mask, L, d, torch.bfloat16)
r0 = (L // 3 // al) * al
part = ga.attention(q[r0:].contiguous(), k, v, mask, L=L, q_begin=r0, kv_begin=0, kernel="tc")
bad = (part != ref[r0:]).any(-1).nonzero()
print("al", al, "r0", r0, "sub mismatch", bad.shape[0], (bad[:12] + torch.tensor([r0, 0], device='cuda')).tolist())
