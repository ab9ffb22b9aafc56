python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_synccheck.log 2>&1
echo "== synccheck rc=$?"; grep -E "OK|FAIL|SUMMARY|Barrier" gpurun_out/san_synccheck.log | sort | uniq -c | head
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "longnet" > gpurun_out/t_ln.log 2>&1; tail -n 3 gpurun_out/t_ln.log
timeout 300 python bench.py --steps 10 --no-per-config --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 ms', d['ms_per_step'])"
