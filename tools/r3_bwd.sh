timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_backward.py -q -x -p no:cacheprovider > gpurun_out/t_bwd.log 2>&1; echo "bwd tests rc=$?"; tail -n 2 gpurun_out/t_bwd.log
for rep in 1 2 3; do for lib in abtest/libga_prev.so paper_2502_01659_b200/libga.so; do
  echo -n "$lib: "; GA_LIB=$PWD/$lib timeout 300 python tools/bwd_time.py
done; done
