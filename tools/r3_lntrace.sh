python tools/build_variant.py ltrace "-DGA_LNET_TRACE" longnet_umma.cu > /dev/null 2>&1
timeout 300 python tools/lnet_trace.py > gpurun_out/ln_trace.txt 2>&1; echo "trace rc=$?"
head -12 gpurun_out/ln_trace.txt; tail -12 gpurun_out/ln_trace.txt
