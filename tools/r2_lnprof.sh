python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python tools/lnet_trace.py > gpurun_out/lnet_trace.txt 2>&1; tail -n 60 gpurun_out/lnet_trace.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:longnet_umma -s 6 -c 1 -o gpurun_out/full_cfg4_umma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --config cfg4 > /dev/null 2>&1
ls -la gpurun_out/full_cfg4_umma.ncu-rep
