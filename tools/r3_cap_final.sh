# final captures for the kernels changed late in the round: launch lists cfg2 cfg3 cfg5, --set full of window_tc (cfg2, cfg5) and csr_tma (cfg3)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CFGS="cfg2 cfg3 cfg5" NO_FULL=1 bash tools/capture_profiles.sh > /dev/null 2>&1
out=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
full="ncu --set full --import-source on --clock-control none -f"
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg2_wtc $B --config cfg2 > /dev/null 2>&1
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg5_wtc $B --config cfg5 > /dev/null 2>&1
timeout 900 $full -k regex:csr_tma -s 1 -c 1 -o $out/full_cfg3_csrtma $B --config cfg3 > /dev/null 2>&1
ls -la $out/full_cfg2_wtc.ncu-rep $out/full_cfg5_wtc.ncu-rep $out/full_cfg3_csrtma.ncu-rep $out/launches_cfg2.csv $out/launches_cfg3.csv $out/launches_cfg5.csv
