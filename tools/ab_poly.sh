# A/B of GA_LNET_POLY (exp2 pairs per 4 on the FMA pipe) on cfg4, plus LongNet parity with the default build
for i in 1 2; do for n in 0 1 2; do
GA_LIB=$PWD/abtest/libga_poly$n.so timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('poly$n', d['ms_per_step'])"
done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "longnet or LongNet or multiset" > gpurun_out/pytest_ln.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_ln.log
python tools/lnet_stress.py 30 | tail -1
