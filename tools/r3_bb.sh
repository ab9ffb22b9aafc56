timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bigbird.py -q -x -p no:cacheprovider > gpurun_out/t_bb.log 2>&1; echo "bb tests rc=$?"; tail -n 2 gpurun_out/t_bb.log
for np in 1 2 4 6 8 12; do GA_BB_PASSES=$np timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3i passes=$np', round(d['ms_per_step'],4))"; done
timeout 300 python bench.py --config cfg3i --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3i default', round(d['ms_per_step'],4))"
