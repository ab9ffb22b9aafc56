python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_bigbird.py tests/test_gpu_dist.py -q -x -p no:cacheprovider -k "bigbird or BigBird" > gpurun_out/t_bb.log 2>&1; tail -n 3 gpurun_out/t_bb.log
for i in 1 2; do for v in 0 1; do
  env $([ $v = 1 ] && echo GA_BB_NOCSR=1) timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nocsr=$v', round(d['ms_per_step'],3))"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3i_v3.csv python bench.py --config cfg3i --steps 1 --warmup 3 --no-per-config --no-e2e --no-cpu-baseline > /dev/null 2>&1
grep -E "bb::|csr_|window_tc|full_|scan" gpurun_out/launches_cfg3i_v3.csv | tail -12 | awk -F'","' '{print $5, $NF}'
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/sanitize_cases.py bigbird_implicit > gpurun_out/san_bb.log 2>&1; tail -n 2 gpurun_out/san_bb.log
