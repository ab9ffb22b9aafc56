python -c "import __graft_entry__ as g; g.build()" > /dev/null
cat > /tmp/bwd_t.py <<'PY'
import sys, time; sys.path.insert(0, '.')
import torch, paper_2502_01659_b200 as ga
L, H, d = 65536, 8, 64
q, k, v = ga.qkv_device(2, L, H, d, torch.bfloat16)
g = ga.qkv_device(9, L, H, d, torch.bfloat16, shift=-0.5)[0]
m = ga.Window(256, 2)
o = ga.attention(q, k, v, m)
for _ in range(3): ga.attention_backward(q, k, v, o, g, m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ga.attention_backward(q, k, v, o, g, m)
e1.record(); torch.cuda.synchronize(); print(sys.argv[1], e0.elapsed_time(e1) / 10)
PY
for i in 1 2; do python /tmp/bwd_t.py u2; GA_LIB=$PWD/abtest/libga_u3.so python /tmp/bwd_t.py u3; GA_LIB=$PWD/abtest/libga_u4.so python /tmp/bwd_t.py u4; done
timeout 600 python -m pytest tests/test_gpu_backward.py -q -x -p no:cacheprovider -k "band or window or dilated" 2>&1 | tail -2
