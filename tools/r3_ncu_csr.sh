B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_tma -s 1 -c 1 -o gpurun_out/full_cfg3_csrtma $B --config cfg3 > gpurun_out/ncu_csr.log 2>&1
ncu -i gpurun_out/full_cfg3_csrtma.ncu-rep --page source --csv --print-source=sass > gpurun_out/cfg3_csr_sass.csv 2>&1
ls -la gpurun_out | tail -3
