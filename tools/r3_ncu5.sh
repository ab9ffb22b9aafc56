B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:window_tc -s 3 -c 1 -o gpurun_out/r3b_cfg5_wtc $B --config cfg5 > gpurun_out/r3_ncu5.log 2>&1
ncu -i gpurun_out/r3b_cfg5_wtc.ncu-rep --page source --csv --print-source=sass > gpurun_out/r3b_cfg5_sass.csv 2>&1
ls -la gpurun_out
