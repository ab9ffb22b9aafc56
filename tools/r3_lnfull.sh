timeout 150 python tools/ln_tiny.py 65536 || { echo "LongNet tiny case failed/hung"; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -n 2
for rep in 1 2; do for lib in abtest/libga_prev.so paper_2502_01659_b200/libga.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $lib', round(d['ms_per_step'],4))"
done; done
