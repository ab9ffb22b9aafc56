./tools/tmem_bench > gpurun_out/tmem_bench.txt 2>&1
for c in cfg5 cfg2; do timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/base_$c.json; done
cat gpurun_out/tmem_bench.txt; cat gpurun_out/base_*.json | cut -c1-300
