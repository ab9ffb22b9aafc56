python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_bigbird.py -q -x -p no:cacheprovider > gpurun_out/t3.log 2>&1
tail -n 30 gpurun_out/t3.log
timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline > gpurun_out/b_cfg3i.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3i.csv \
    python bench.py --config cfg3i --steps 2 --warmup 3 --no-per-config --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/b_cfg3i.json').read().strip().splitlines()[-1]); print('cfg3i ms', d['ms_per_step'])
PY
grep extras gpurun_out/launches_cfg3i.csv | tail -2
