for cfg in cfg2 cfg5; do for i in 1 2 3; do for lib in abtest/libga_old.so abtest/libga_war.so; do
GA_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $lib', d['ms_per_step'])"
done; done; done
GA_LIB=$PWD/abtest/libga_war.so python tools/wtc_race.py 100 | tail -1
