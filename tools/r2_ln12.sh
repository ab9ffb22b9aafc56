python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -x -p no:cacheprovider -k "longnet or LongNet" > gpurun_out/t_ln.log 2>&1; tail -n 3 gpurun_out/t_ln.log
timeout 300 python bench.py --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['ms_per_step'],3))"
