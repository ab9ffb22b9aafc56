for i in 1 2 3; do for lib in abtest/libga_pre.so abtest/libga_exact2.so; do
GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'])"
done; done
python tools/lib_bitwise.py abtest/libga_pre.so abtest/libga_exact2.so longnet
timeout 900 python -m pytest tests -m gpu -x -q -k "longnet or LongNet or multiset or lattice or sharded" > gpurun_out/pytest_ln.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_ln.log
