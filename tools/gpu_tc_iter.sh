timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "window_tc or cfg2_shape or sharded_offsets or repeat_launches or cfg2_full" > gpurun_out/tc1.log 2>&1; echo rc=$?; tail -2 gpurun_out/tc1.log
python bench.py --kernel tc --steps 20 > gpurun_out/bench_tc.log 2>&1; tail -1 gpurun_out/bench_tc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'kernel_ms', d['roofline']['kernel_ms_median'])"
python tools/wtc_trace.py 20000 > gpurun_out/trace.txt 2>&1
