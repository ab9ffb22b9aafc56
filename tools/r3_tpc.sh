# LongNet tiles-per-CTA A/B: hang guard, LongNet GPU tests, cfg4 timing (same box)
timeout 120 python tools/ln_tiny.py 65536 || { echo "TPC2 tiny failed/hung"; exit 1; }
GA_LIB=$PWD/abtest/libga_tpc1.so timeout 120 python tools/ln_tiny.py 65536 > /dev/null || { echo "tpc1 hung"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "longnet or LongNet or dilated or cfg4 or edgeset or block" 2>&1 | tail -5
for rep in 1 2 3; do for n in base tpc1; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
