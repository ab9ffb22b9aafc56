# LongNet check: parity tests, cfg4 bench, launch list + ncu of the group-mode tcgen05 kernel
timeout 900 python -m pytest tests -m gpu -x -q -k "longnet or LongNet or sharded or repeat or families or multiset" > gpurun_out/pytest_ln.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_ln.log
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; tail -1 gpurun_out/bench_cfg4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["roofline"]["frac"])'
CFGS=cfg4 NO_FULL=1 bash tools/capture_profiles.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:longnet_umma -s 6 -c 1 -o gpurun_out/full_cfg4_umma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --config cfg4 > /dev/null 2>&1
ls gpurun_out | head -40
GA_LNET_CPASYNC=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_cpa.log 2>&1; echo "cpasync $(tail -1 gpurun_out/bench_cfg4_cpa.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
