# BigBird extras kernel register target: 4 CTAs/SM (64 regs) vs 5, 6 (more warps, more spills); 3 and 1 measured slower
GA_LIB=$PWD/abtest/libga_mb5.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bigbird or BigBird" 2>&1 | tail -2
for rep in 1 2 3; do for n in base mb5 mb6; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3i $n', round(d['ms_per_step'],4))"
done; done
