# backward: batched D / lse loads — backward GPU tests + timing A/B vs the previous build
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "backward or grad or autograd" 2>&1 | tail -2
for rep in 1 2 3; do for n in base bwdprev; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  echo -n "$n: "; GA_LIB=$PWD/$lib timeout 300 python tools/bwd_time.py
done; done
GA_LIB= timeout 300 python bench.py --config cfg2 --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['per_config']['cfg2_backward']; print('bench cfg2_backward', round(b['ms_per_step'],4), b['roofline']['frac'])"
