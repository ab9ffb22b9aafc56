python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_bigbird.py -q -x -p no:cacheprovider > gpurun_out/t_bb.log 2>&1; tail -n 3 gpurun_out/t_bb.log
for i in 1 2; do
  timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3i', round(d['ms_per_step'],3))"
done
