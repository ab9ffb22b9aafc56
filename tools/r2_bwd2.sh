python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_variants.py -q -x -p no:cacheprovider > gpurun_out/t_bwd.log 2>&1; tail -n 15 gpurun_out/t_bwd.log
timeout 600 python bench.py --config cfg2 --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['per_config']['cfg2_backward']; print('bwd', round(b['ms_per_step'],3), b['roofline'])"
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/sanitize_cases.py backward > gpurun_out/san_bwd.log 2>&1; tail -n 2 gpurun_out/san_bwd.log
