python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edgesets.py -q -x -p no:cacheprovider -k "window_tc" > gpurun_out/t_edge.log 2>&1; echo "edge rc=$?"; tail -n 2 gpurun_out/t_edge.log
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
full="ncu --set full --import-source on --clock-control none"
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o gpurun_out/full_cfg2_wtc $B --config cfg2 > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o gpurun_out/full_cfg5_wtc $B --config cfg5 > /dev/null 2>&1; echo "ncu5 rc=$?"
CFGS="cfg2 cfg5 cfg3i" NO_FULL=1 bash tools/capture_profiles.sh > /dev/null 2>&1; echo "launches rc=$?"
bash tools/r3_trace.sh > /dev/null 2>&1; echo "trace rc=$?"
ls gpurun_out
