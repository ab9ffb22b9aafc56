# window_tc with one MMA issuer per warpgroup: hang-trapping build first, then parity, A/B, synccheck
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/build_variant.py spin "-DGA_MBAR_SPIN_LIMIT=50000000" window_tc.cu > /dev/null
python tools/build_variant.py single "-DGA_WTC_DUAL=0" window_tc.cu > /dev/null
GA_LIB=$PWD/abtest/libga_spin.so timeout 600 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -x -p no:cacheprovider -k "window or Window or tc" > gpurun_out/t_dual_spin.log 2>&1; echo "spin rc=$?"; tail -n 2 gpurun_out/t_dual_spin.log
if grep -q " passed" gpurun_out/t_dual_spin.log && ! grep -q "failed\|error" gpurun_out/t_dual_spin.log; then
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_bigbird.py tests/test_gpu_dist.py tests/test_gpu_variants.py -q -x -p no:cacheprovider -k "window or Window or tc or host or alias or state or bigbird or ring or shard" > gpurun_out/t_dual.log 2>&1; tail -n 2 gpurun_out/t_dual.log
for c in cfg2 cfg5; do for i in 1 2; do for lib in abtest/libga_single.so paper_2502_01659_b200/libga.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $lib', round(d['ms_per_step'],4), d['roofline']['frac'])"
done; done; done
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tools/sanitize_cases.py window_tc > gpurun_out/san_dual.log 2>&1; tail -n 2 gpurun_out/san_dual.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tools/sanitize_cases.py window_tc > gpurun_out/san_dual_race.log 2>&1; tail -n 2 gpurun_out/san_dual_race.log
fi
