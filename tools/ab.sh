#!/bin/bash
# A/B timing of two libga builds on the same box: tools/ab.sh CONFIG [reps]
# (old build at abtest/libga_old.so, new = in-tree build); prints ms/step per run.
cfg=$1; reps=${2:-3}
for i in $(seq $reps); do
  for lib in abtest/libga_old.so paper_2502_01659_b200/libga.so; do
    GA_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['roofline']['kernel_ms_median'])"
  done
done
