for rep in 1 2; do for lib in paper_2502_01659_b200/libga.so abtest/libga_contig.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $lib', round(d['ms_per_step'],4))"
done; done
