# headline refresh after a LongNet change: default bench line, cfg4 launch list + full capture
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 120 python tools/ln_tiny.py 65536 || { echo "tiny failed"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "longnet or LongNet or cfg4 or edgeset or smoke" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print('headline', round(d['ms_per_step'],3), '%.3e' % d['value'], d['roofline']['bound'], d['roofline']['frac'], d['clocks'])
for k,v in d['per_config'].items(): print(k, round(v['ms_per_step'],4), '%.3e'%v['value'], v['roofline']['bound'], v['roofline']['frac'])
PY
CFGS=cfg4 NO_FULL=1 bash tools/capture_profiles.sh > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:longnet_umma -s 6 -c 1 -o gpurun_out/full_cfg4_umma -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --config cfg4 > /dev/null 2>&1
ls gpurun_out/full_cfg4_umma.ncu-rep gpurun_out/launches_cfg4.csv
