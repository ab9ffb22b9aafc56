timeout 150 python tools/ln_tiny.py 65536 || { echo "LongNet tiny case failed/hung"; exit 1; }
timeout 200 python tools/ln_tiny.py 1048576 || { echo "LongNet 1M case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_contracts.py -q -x -p no:cacheprovider -k "longnet or LongNet or lnet" > gpurun_out/t_ln.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/t_ln.log
for i in 1 2; do timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', round(d['ms_per_step'],4), d.get('roofline',{}).get('frac'))"; done
