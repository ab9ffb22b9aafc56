python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -x -p no:cacheprovider -k "longnet or LongNet" > gpurun_out/t_ln.log 2>&1; tail -n 2 gpurun_out/t_ln.log
for i in 1 2; do for lib in abtest/libga_sepp.so paper_2502_01659_b200/libga.so abtest/libga_k5v4.so abtest/libga_k5v5.so abtest/libga_k4v4l3.so abtest/libga_k6v4.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3))"
done; done
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tools/sanitize_cases.py longnet_umma > gpurun_out/san_ln.log 2>&1; tail -n 2 gpurun_out/san_ln.log
