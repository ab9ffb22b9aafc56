for rep in 1 2; do for n in base u3 u4; do
  lib=paper_2502_01659_b200/libga.so; [ "$n" != base ] && lib=abtest/libga_$n.so
  echo -n "$n: "; GA_LIB=$PWD/$lib timeout 300 python tools/bwd_time.py
done; done
