# A/B of LongNet build variants: VARIANTS="name:flags;name:flags"
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do n=${v%%:*}; f=${v#*:}; python tools/build_variant.py $n "$f" longnet_umma.cu > /dev/null 2>&1; done
timeout 150 python tools/ln_tiny.py 65536 || { echo "LongNet tiny case failed/hung"; exit 1; }
for v in "${VS[@]}"; do n=${v%%:*}; GA_LIB=$PWD/abtest/libga_$n.so timeout 150 python tools/ln_tiny.py 65536 > /dev/null || { echo "$n hung"; exit 1; }; done
for rep in 1 2; do for v in base "${VS[@]}"; do n=${v%%:*}
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg4 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $n', round(d['ms_per_step'],4))"
done; done
