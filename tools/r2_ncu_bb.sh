python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/t_dist.log 2>&1
tail -n 30 gpurun_out/t_dist.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:extras_kernel -s 1 -c 1 -o gpurun_out/full_cfg3i_extras python bench.py --config cfg3i --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
