# LongNet: share of the exponentials on the FMA pipe (1/16, 1/8, 1/4 of the pairs), cfg4 A/B
timeout 120 python tools/ln_tiny.py 65536 || { echo "base tiny failed"; exit 1; }
for n in p116 p18 p14; do GA_LIB=$PWD/abtest/libga_$n.so timeout 120 python tools/ln_tiny.py 65536 || { echo "$n failed/hung"; exit 1; }; done
for rep in 1 2; do for n in base p116 p18 p14; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
