# window_tc: hang guard on a tiny case, then the window-related GPU tests, then bench
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
timeout 150 python tools/wtc_tiny.py 65536 8 || { echo "cfg2 case failed/hung"; exit 1; }
timeout 300 python -m pytest tests/test_gpu_edgesets.py -q -x -p no:cacheprovider -k "window_tc" > gpurun_out/t_edge.log 2>&1; echo "edge rc=$?"; tail -n 3 gpurun_out/t_edge.log
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_bigbird.py tests/test_gpu_dist.py -q -x -p no:cacheprovider -k "window or Window or tc or host or alias or state or bigbird or shard" > gpurun_out/t_wtc.log 2>&1; echo "tests rc=$?"; tail -n 5 gpurun_out/t_wtc.log
for c in cfg5 cfg2 cfg3i; do timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), d.get('roofline',{}).get('frac'))"; done
