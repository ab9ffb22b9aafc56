python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2; do for lib in paper_2502_01659_b200/libga.so abtest/libga_s5.so abtest/libga_s3.so; do
  GA_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3))"
done; done
