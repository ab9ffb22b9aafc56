# end-of-session refresh: default bench line + backward ncu capture
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print('headline', round(d['ms_per_step'],3), '%.3e' % d['value'], d['roofline']['bound'], d['roofline']['frac'], d['clocks'])
for k,v in d['per_config'].items(): print(k, round(v['ms_per_step'],4), '%.3e'%v['value'], v['roofline']['bound'], v['roofline']['frac'])
PY
bash tools/r3_capbwd.sh
