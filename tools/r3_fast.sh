# K7 fast exponential path A/B (fast0 = max first every chunk): hang guard, window GPU tests on the new default, cfg5/cfg2 timing
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "base tiny failed"; exit 1; }
GA_LIB=$PWD/abtest/libga_fast0.so timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "fast0 tiny failed/hung"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "window or Window or wtc or window_tc or edgeset or cfg2 or cfg5 or dilated" 2>&1 | tail -3
for rep in 1 2; do for c in cfg5 cfg2; do for n in base fast0; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $n', round(d['ms_per_step'],4))"
done; done; done
