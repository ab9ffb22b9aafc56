# CSR path check: parity tests touching CSR (default cp.async ring, and the TMA gather4 variant),
# cfg3 bench A/B (cp.async / gather4 / LDG), cfg3 launch list + ncu of the default light kernel
K="csr or bigbird or paper_protocol or empty_rows or preset or state or host_entry or sharded or repeat"
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_csr.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_csr.log
GA_CSR_CPASYNC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "csr" > gpurun_out/pytest_csr_cpa.log 2>&1; echo pytest cpasync rc=$?; tail -1 gpurun_out/pytest_csr_cpa.log
for v in "" GA_CSR_CPASYNC=1 GA_CSR_LDG=1; do env $v timeout 600 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_ab.log 2>&1; echo "$v $(tail -1 gpurun_out/bench_cfg3_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"; done
timeout 600 python bench.py --config cfg3 > gpurun_out/bench_cfg3.log 2>&1; tail -1 gpurun_out/bench_cfg3.log | cut -c1-200
CFGS=cfg3 NO_FULL=1 bash tools/capture_profiles.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_tma -s 1 -c 1 -o gpurun_out/full_cfg3_csrtma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --config cfg3 > /dev/null 2>&1
ls gpurun_out
