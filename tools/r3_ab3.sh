timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_bigbird.py -q -x -p no:cacheprovider -k "csr or CSR or bigbird or BigBird" 2>&1 | tail -n 1
for rep in 1 2; do for c in cfg3 cfg3i; do for lib in abtest/libga_prev.so paper_2502_01659_b200/libga.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $lib', round(d['ms_per_step'],4))"
done; done; done
