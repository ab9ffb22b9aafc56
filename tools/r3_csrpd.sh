# CSR index pairs staged ahead in shared memory: 5 (default) vs 3, 7 at cfg3
GA_LIB=$PWD/abtest/libga_pd7.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "csr or CSR or cfg3 or bigbird" 2>&1 | tail -1
for rep in 1 2 3; do for n in base pd3 pd7; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg3 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 $n', round(d['ms_per_step'],4))"
done; done
