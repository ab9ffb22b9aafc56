python tools/build_variant.py trace "-DGA_WTC_TRACE" window_tc.cu > /dev/null 2>&1
WTC_SHAPE=16777216,1,128,1 python tools/wtc_trace.py 6000 > gpurun_out/trace5.txt 2>&1
python tools/wtc_trace_summary.py gpurun_out/trace5.txt 0,2,4 > gpurun_out/trace5_sum.txt
head -40 gpurun_out/trace5.txt; cat gpurun_out/trace5_sum.txt | head -120
