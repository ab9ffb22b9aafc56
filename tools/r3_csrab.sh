# A/B of CSR kernel variants: VARIANTS="name:flags;..."
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do n=${v%%:*}; f=${v#*:}; python tools/build_variant.py $n "$f" csr_mma.cu > /dev/null 2>&1; done
timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
for rep in 1 2; do for v in base "${VS[@]}"; do n=${v%%:*}
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  GA_LIB=$PWD/$lib timeout 300 python bench.py --config cfg3 --steps 10 --no-per-config --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 $n', round(d['ms_per_step'],4))"
done; done
