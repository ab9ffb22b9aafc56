# one default bench line (cfg4 headline + per_config) and the ncu launch list of the same step
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 600 gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-per-config --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3i.csv \
    python bench.py --config cfg3i --steps 2 --warmup 3 --no-per-config --no-e2e --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/bench_default.json
