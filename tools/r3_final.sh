# evidence refresh: GPU tests, smoke, default bench line, max context, launch lists + full captures
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_full.log 2>&1; tail -n 3 gpurun_out/t_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print('headline', round(d['ms_per_step'],3), '%.3e' % d['value'], d['roofline']['bound'], d['roofline']['frac'], d['clocks'])
for k,v in d['per_config'].items(): print(k, round(v['ms_per_step'],4), '%.3e'%v['value'], v['roofline']['bound'], v['roofline']['frac'])
PY
timeout 900 python bench.py --max-context > gpurun_out/max_context.json 2> gpurun_out/max_context.err; tail -c 600 gpurun_out/max_context.json
bash tools/r2_capture.sh > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | wc -l
