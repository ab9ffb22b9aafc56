# LongNet ring depth 5 vs 4 (current code), cfg4; plus the BigBird tests on the default build
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bigbird or BigBird" 2>&1 | tail -1
GA_LIB=$PWD/abtest/libga_st5.so timeout 120 python tools/ln_tiny.py 65536 || { echo "st5 failed"; exit 1; }
for rep in 1 2 3; do for n in base st5; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
