# full GPU suite + default bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_full.log 2>&1; echo "gpu tests rc=$?"; tail -n 3 gpurun_out/t_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_default.json
