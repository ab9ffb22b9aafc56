python -c "import __graft_entry__ as g; g.build()" > /dev/null
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $S --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -n 25 gpurun_out/san_$tool.log
done
