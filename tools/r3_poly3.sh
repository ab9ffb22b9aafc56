# exp2 share on the FMA pipe: K7 1 of 16 pairs per half (cfg5, cfg2); K5 1 of 32 pairs (cfg4) vs the 1/16 default
for rep in 1 2; do
for n in base wpoly1; do lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  for c in cfg5 cfg2; do GA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $n', round(d['ms_per_step'],4))"; done; done
for n in base p132; do lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"; done
done
