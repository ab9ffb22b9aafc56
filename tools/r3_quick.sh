# hang guard + edge-set tests + cfg5/cfg2 bench + trace
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
timeout 300 python -m pytest tests/test_gpu_edgesets.py -q -x -p no:cacheprovider -k "window_tc" 2>&1 | tail -n 2
for c in cfg5 cfg2; do timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), d.get('roofline',{}).get('frac'))"; done
[ -n "$TRACE" ] && bash tools/r3_trace.sh > /dev/null 2>&1 && cat gpurun_out/trace5_sum.txt | head -60
true
