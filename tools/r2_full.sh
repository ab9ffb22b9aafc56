python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_full.log 2>&1; tail -n 5 gpurun_out/t_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 400 gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print('headline', d['config']['workload'], round(d['ms_per_step'],3), d['value'], d['roofline']['bound'], d['roofline']['frac'])
for k,v in d['per_config'].items(): print(k, round(v['ms_per_step'],4), '%.3e'%v['value'], v['roofline']['bound'], v['roofline']['frac'])
print('e2e', d['e2e']['ms_per_step'], 'cpu', d['cpu_baseline']['value'], d['clocks'])
PY
