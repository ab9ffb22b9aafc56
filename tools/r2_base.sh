set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
for c in cfg4 cfg3 cfg5 cfg2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget 8 > gpurun_out/base_$c.json 2> gpurun_out/base_$c.err; done
timeout 600 python bench.py --max-context > gpurun_out/base_maxctx.json 2> gpurun_out/base_maxctx.err
tail -c 3000 gpurun_out/base_*.json
