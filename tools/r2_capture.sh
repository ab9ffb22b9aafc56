# round-2 profile capture: launch lists (time + DRAM bytes) for every config, --set full of the
# dominant kernels, and the backward kernels at cfg2
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CFGS="cfg1 cfg2 cfg3 cfg3i cfg4 cfg5" NO_FULL=1 bash tools/capture_profiles.sh > /dev/null 2>&1
out=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
full="ncu --set full --import-source on --clock-control none"
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg2_wtc $B --config cfg2 > /dev/null 2>&1
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg5_wtc $B --config cfg5 > /dev/null 2>&1
timeout 900 $full -k regex:csr_tma -s 1 -c 1 -o $out/full_cfg3_csrtma $B --config cfg3 > /dev/null 2>&1
timeout 900 $full -k regex:extras -s 1 -c 1 -o $out/full_cfg3i_extras $B --config cfg3i > /dev/null 2>&1
timeout 900 $full -k regex:longnet_umma -s 6 -c 1 -o $out/full_cfg4_umma $B --config cfg4 > /dev/null 2>&1
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
timeout 900 $full -k "regex:row_kernel|col_kernel" -s 2 -c 2 -o $out/full_cfg2_bwd python /tmp/bwd_once.py > /dev/null 2>&1
ls -la $out/*.ncu-rep $out/launches_*.csv
