# LongNet 1/16 of the exp2 pairs on the FMA pipe: LongNet GPU tests on the variant + cfg4 A/B
GA_LIB=$PWD/abtest/libga_p116.so timeout 900 python -m pytest tests -m gpu -x -q -k "longnet or LongNet or cfg4 or edgeset" 2>&1 | tail -3
for rep in 1 2 3; do for n in base p116; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
