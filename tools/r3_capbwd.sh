cat > /tmp/bwd_once.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2502_01659_b200 as ga
L, H, d = 65536, 8, 64
q, k, v = ga.qkv_device(2, L, H, d, torch.bfloat16)
g = ga.qkv_device(9, L, H, d, torch.bfloat16, shift=-0.5)[0]
m = ga.Window(256, 2)
o = ga.attention(q, k, v, m)
for _ in range(2): ga.attention_backward(q, k, v, o, g, m)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:row_kernel|col_kernel" -s 2 -c 2 -f -o gpurun_out/full_cfg2_bwd python /tmp/bwd_once.py > /dev/null 2>&1
ls -la gpurun_out/full_cfg2_bwd.ncu-rep
