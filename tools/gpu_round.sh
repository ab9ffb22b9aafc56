set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log; done
bash tools/capture_profiles.sh
