S=/usr/local/cuda/bin/compute-sanitizer
timeout 150 python tools/wtc_tiny.py 2048 1 || { echo "tiny case failed/hung"; exit 1; }
GA_WTC_GRID=3 timeout 150 python tools/sanitize_cases.py window_tc_run || { echo "run case failed"; exit 1; }
for tool in memcheck synccheck racecheck; do
  timeout 1200 $S --tool $tool --print-limit 20 python tools/sanitize_cases.py ${CASES:-window_tc window_tc_run bigbird_implicit} > gpurun_out/san3_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -n 6 gpurun_out/san3_$tool.log
done
