timeout 120 python tools/ln_tiny.py 65536 || { echo "base tiny failed"; exit 1; }
GA_LIB=$PWD/abtest/libga_pair2.so timeout 120 python tools/ln_tiny.py 65536 || { echo "pair tiny failed/hung"; exit 1; }
for rep in 1 2; do for n in base pair2; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
