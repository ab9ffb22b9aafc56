"""Time ga.attention_backward on cfg2's shape (CUDA events, median of 20, L2 not flushed)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2502_01659_b200 as ga

L, H, d = 65536, 8, 64
q, k, v = ga.qkv_device(2, L, H, d, torch.bfloat16)
g = ga.qkv_device(9, L, H, d, torch.bfloat16, shift=-0.5)[0]
m = ga.Window(256, 2)
o = ga.attention(q, k, v, m)
for _ in range(3):
    ga.attention_backward(q, k, v, o, g, m)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ga.attention_backward(q, k, v, o, g, m)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"backward cfg2 {ts[len(ts) // 2]:.4f} ms")
