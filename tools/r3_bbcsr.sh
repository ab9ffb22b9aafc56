timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bigbird.py tests/test_gpu_edgesets.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bigbird or BigBird" > gpurun_out/t_bb.log 2>&1; echo "bb tests rc=$?"; tail -n 3 gpurun_out/t_bb.log
GA_BB_CSR=0 timeout 900 python -m pytest tests/test_gpu_bigbird.py -q -x -p no:cacheprovider 2>&1 | tail -n 1
for rep in 1 2; do for e in 0 1; do
  GA_BB_CSR=$e timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3i GA_BB_CSR=$e', round(d['ms_per_step'],4))"
done; done
