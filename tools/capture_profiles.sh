#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   launch lists (time + DRAM bytes per launch, cold caches, serialised) for cfg1-cfg5 and
#   one `ncu --set full` report of each config's dominant kernel(s), into gpurun_out/.
set -u
out=gpurun_out
mkdir -p $out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg3i cfg4 cfg5}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $out/launches_$c.csv $B --config $c > $out/launches_$c.log 2>&1
done
[ -n "${NO_FULL:-}" ] && exit 0
full="ncu --set full --import-source on --clock-control none"
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg2_wtc $B --config cfg2 > /dev/null 2>&1
timeout 900 $full -k regex:csr_tma -s 1 -c 1 -o $out/full_cfg3_csrtma $B --config cfg3 > /dev/null 2>&1
timeout 900 $full -k regex:longnet_umma -s 6 -c 2 -o $out/full_cfg4_umma $B --config cfg4 > /dev/null 2>&1
timeout 900 $full -k regex:window_tc -s 3 -c 1 -o $out/full_cfg5_wtc $B --config cfg5 > /dev/null 2>&1
ls -la $out
