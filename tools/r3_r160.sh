# K7 setmaxnreg 160/104/88 (spill-free) vs 168/104/72: window GPU tests on the variant, cfg5/cfg2 timing
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "base tiny failed"; exit 1; }
GA_LIB=$PWD/abtest/libga_r160.so timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "r160 tiny failed/hung"; exit 1; }
GA_LIB=$PWD/abtest/libga_r160.so timeout 900 python -m pytest tests -m gpu -x -q -k "window or Window or wtc or window_tc or edgeset or cfg2 or cfg5 or dilated" 2>&1 | tail -3
for rep in 1 2; do for c in cfg5 cfg2; do for n in base r160; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $n', round(d['ms_per_step'],4))"
done; done; done
