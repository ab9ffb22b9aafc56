for i in 1 2 3; do for lib in abtest/libga_csrbase.so abtest/libga_fm.so; do
GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'])"
done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "csr or bigbird or coo or multiset or preset or paper_protocol" > gpurun_out/pytest_csr.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_csr.log
