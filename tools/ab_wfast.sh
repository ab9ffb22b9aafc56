for cfg in cfg2 cfg5; do for i in 1 2 3; do for lib in abtest/libga_wbase.so abtest/libga_wfast.so; do
GA_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $lib', d['ms_per_step'])"
done; done; done
python tools/lib_bitwise.py abtest/libga_wbase.so abtest/libga_wfast.so window
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window or band or cfg2 or cfg5" > gpurun_out/pytest_w.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_w.log
python tools/wtc_race.py 100 | tail -1
