python -c "import __graft_entry__ as g; g.build()" > /dev/null
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
timeout 900 ncu --set full --import-source on --clock-control none -k regex:row_kernel -s 1 -c 1 -o gpurun_out/full_bwd_row python /tmp/bwd_once.py > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:col_kernel -s 1 -c 1 -o gpurun_out/full_bwd_col python /tmp/bwd_once.py >> gpurun_out/ncu_bwd.log 2>&1
tail -3 gpurun_out/ncu_bwd.log; ls -la gpurun_out/full_bwd*
